python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest64.log 2>&1; echo "rc=$?" >> gpurun_out/pytest64.log
FREEKV_TRACE=1 timeout 600 python tools/trace_step.py --graph > gpurun_out/trace64.json 2> gpurun_out/trace64.err
FREEKV_DEBUG_EXP=4 FREEKV_TRACE=1 timeout 600 python tools/trace_step.py --graph > gpurun_out/trace64x.json 2> gpurun_out/trace64x.err
timeout 300 python tools/kbench.py --layers 32 --steps 10 --warmup 5 --graph --no-profile > gpurun_out/kb64.json 2>&1
