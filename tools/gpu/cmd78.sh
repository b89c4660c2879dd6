python -c "import __graft_entry__ as g; g.build()"
timeout 900 python bench.py > gpurun_out/bench78.json 2> gpurun_out/bench78.err
bash tools/gpu/ablation.sh
