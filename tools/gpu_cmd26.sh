python -c "import __graft_entry__ as g; g.build()"
timeout 300 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "llama_shape or full_refresh" > gpurun_out/pytest26a.log 2>&1; echo "rc=$?" >> gpurun_out/pytest26a.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest26.log 2>&1; echo "rc=$?" >> gpurun_out/pytest26.log
FREEKV_TRACE=1 timeout 600 python tools/trace_step.py --graph > gpurun_out/trace26.json 2> gpurun_out/trace26.err
timeout 300 python tools/kbench.py --layers 4 --steps 20 --warmup 5 --graph --no-profile > gpurun_out/kb26.json 2>&1
FREEKV_CORR=recall timeout 300 python tools/kbench.py --layers 4 --steps 20 --warmup 5 --graph --no-profile > gpurun_out/kb26r.json 2>&1
