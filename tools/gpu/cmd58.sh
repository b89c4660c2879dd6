python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest58.log 2>&1; echo "rc=$?" >> gpurun_out/pytest58.log
FREEKV_TRACE=1 timeout 600 python tools/trace_step.py --graph > gpurun_out/trace58.json 2> gpurun_out/trace58.err
timeout 310 python tools/kbench.py --layers 32 --steps 10 --warmup 5 --graph --no-profile > gpurun_out/kb58.json 2>&1
