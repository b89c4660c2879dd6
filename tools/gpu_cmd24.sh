python -c "import __graft_entry__ as g; g.build()"
timeout 600 python tools/trace_step.py --graph > gpurun_out/trace24.json 2> gpurun_out/trace24.err
timeout 900 python bench.py --steps 128 --warmup 4 --profile-steps 4 --cpu-sample-s 12 > gpurun_out/bench24.json 2> gpurun_out/bench24.err
