# c4 (48K context) correction-threshold sweep (bench.py --config c4 --tau T)
for t in 0.0 0.5 0.8 0.9 0.95 1.0; do
  timeout 300 python bench.py --config c4 --tau $t --steps 64 --warmup 4 --no-cpu-baseline > gpurun_out/c4_tau${t}.json 2> gpurun_out/c4_tau${t}.err
done
