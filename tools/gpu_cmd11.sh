python -c "import __graft_entry__ as g; g.build()"
timeout 300 python tools/kbench.py --layers 4 --steps 20 --warmup 5 --graph > gpurun_out/kb11_graph.json 2>&1
timeout 300 python tools/kbench.py --layers 4 --steps 20 --warmup 5 --graph --no-profile > gpurun_out/kb11_graph_noprof.json 2>&1
timeout 900 python bench.py --steps 16 --warmup 3 --profile-steps 4 --no-cpu-baseline > gpurun_out/bench11.json 2> gpurun_out/bench11.err
