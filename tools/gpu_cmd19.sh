python -c "import __graft_entry__ as g; g.build()"
timeout 600 python tools/trace_step.py > gpurun_out/trace19.json 2> gpurun_out/trace19.err
