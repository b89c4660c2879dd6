python -c "import __graft_entry__ as g; g.build()"
FREEKV_TRACE=1 timeout 600 python tools/trace_step.py --graph > gpurun_out/trace51.json 2> gpurun_out/trace51.err
FREEKV_DEBUG_EXP=1 FREEKV_TRACE=1 timeout 600 python tools/trace_step.py --graph > gpurun_out/trace51x.json 2> gpurun_out/trace51x.err
