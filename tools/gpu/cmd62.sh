FREEKV_TRACE=1 timeout 600 python tools/trace_step.py --graph --dump > gpurun_out/trace62.json 2> gpurun_out/trace62.err
