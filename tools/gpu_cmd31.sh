python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest31.log 2>&1; echo "rc=$?" >> gpurun_out/pytest31.log
FREEKV_TRACE=1 timeout 600 python tools/trace_step.py --graph > gpurun_out/trace31.json 2> gpurun_out/trace31.err
timeout 310 python tools/kbench.py --layers 4 --steps 20 --warmup 5 --graph --no-profile > gpurun_out/kb31.json 2>&1
FREEKV_PIPELINE=0 timeout 310 python tools/kbench.py --layers 4 --steps 20 --warmup 5 --graph --no-profile > gpurun_out/kb31np.json 2>&1
timeout 310 python tools/kbench.py --layers 32 --steps 10 --warmup 5 --graph --no-profile > gpurun_out/kb31_32.json 2>&1
FREEKV_ATTN_CTAS_PER_SM=2 timeout 310 python tools/kbench.py --layers 32 --steps 10 --warmup 5 --graph --no-profile > gpurun_out/kb31_32_c2.json 2>&1
