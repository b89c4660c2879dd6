# build, GPU parity suite, smoke, then c2/c3 bench lines (round 2 iteration check)
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -q -x --timeout 300 ${PYTEST_K:+-k "$PYTEST_K"} > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
for c in ${CFGS:-c2 c3}; do
  timeout 300 python bench.py --config $c --steps 128 --no-cpu-baseline > gpurun_out/${TAG}_bench_$c.json 2> gpurun_out/${TAG}_bench_$c.err
done
