python -c "import __graft_entry__ as g; g.build()"
: > gpurun_out/f3_perf.txt
for r in 1 2; do
for p in 0 1 2 3 4 5; do
  out=$(timeout 300 python tools/kbench.py --layers 32 --steps 10 --warmup 5 --graph --no-profile --pool $p 2>/dev/null | tail -1)
  echo "pool=$p $out" >> gpurun_out/f3_perf.txt
done
out=$(timeout 300 python tools/kbench.py --layers 32 --steps 10 --warmup 5 --graph --no-profile --corr_pool 1 2>/dev/null | tail -1)
echo "corr_pool=1 $out" >> gpurun_out/f3_perf.txt
done
