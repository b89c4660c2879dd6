python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest10.log 2>&1; echo "rc=$?" >> gpurun_out/pytest10.log
timeout 300 python tools/kbench.py --layers 4 --steps 20 --warmup 5 --graph > gpurun_out/kb10_graph.json 2>&1
timeout 900 python bench.py --steps 16 --warmup 3 --profile-steps 4 --no-cpu-baseline > gpurun_out/bench10.json 2> gpurun_out/bench10.err
