python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest77.log 2>&1; echo "rc=$?" >> gpurun_out/pytest77.log
timeout 900 python bench.py --config c1 --steps 64 --no-cpu-baseline > gpurun_out/bench77_c1.json 2> gpurun_out/bench77_c1.err
timeout 900 python bench.py --config c3 --steps 32 --no-cpu-baseline > gpurun_out/bench77_c3.json 2> gpurun_out/bench77_c3.err
