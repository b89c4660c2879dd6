# A/B of two builds on one box: libfreekv_A.so vs libfreekv_B.so (built locally, travel in-tree)
for r in 1 2 3; do
  for v in A B; do
    FREEKV_LIB_SUFFIX=_$v timeout 300 python tools/kbench.py --layers 32 --steps 10 --warmup 5 --graph --no-profile > gpurun_out/ab_${v}_$r.json 2>&1
  done
done
