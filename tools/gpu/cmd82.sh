python -c "import __graft_entry__ as g; g.build()"
FREEKV_TRACE=1 timeout 600 python tools/trace_step.py --graph --dump > gpurun_out/trace82.json 2> gpurun_out/trace82.err
