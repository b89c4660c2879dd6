python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest20.log 2>&1; echo "rc=$?" >> gpurun_out/pytest20.log
timeout 600 python tools/trace_step.py > gpurun_out/trace20.json 2> gpurun_out/trace20.err
timeout 300 python tools/kbench.py --layers 4 --steps 20 --warmup 5 --graph --no-profile > gpurun_out/kb20_graph_noprof.json 2>&1
