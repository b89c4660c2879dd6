# build, bench lines for $CFGS (no GPU test suite), the graph trace of c2
python -c "import __graft_entry__ as g; g.build()"
for c in ${CFGS:-c2 c3}; do
  timeout 300 python bench.py --config $c --steps 128 --no-cpu-baseline > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
done
timeout 300 python tools/trace_step.py --graph > gpurun_out/${TAG}_trace.json 2>&1
