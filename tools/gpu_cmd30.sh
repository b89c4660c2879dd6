python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest30.log 2>&1; echo "rc=$?" >> gpurun_out/pytest30.log
FREEKV_TRACE=1 timeout 600 python tools/trace_step.py --graph > gpurun_out/trace30.json 2> gpurun_out/trace30.err
timeout 300 python tools/kbench.py --layers 4 --steps 20 --warmup 5 --graph --no-profile > gpurun_out/kb30.json 2>&1
FREEKV_PIPELINE=0 timeout 300 python tools/kbench.py --layers 4 --steps 20 --warmup 5 --graph --no-profile > gpurun_out/kb30np.json 2>&1
timeout 300 python tools/kbench.py --layers 32 --steps 10 --warmup 5 --graph --no-profile > gpurun_out/kb30_32.json 2>&1
FREEKV_ATTN_CTAS_PER_SM=2 timeout 300 python tools/kbench.py --layers 32 --steps 10 --warmup 5 --graph --no-profile > gpurun_out/kb30_32_c2.json 2>&1
