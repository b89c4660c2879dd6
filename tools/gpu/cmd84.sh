python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest84.log 2>&1; echo "rc=$?" >> gpurun_out/pytest84.log
for r in 1 2; do timeout 300 python tools/kbench.py --layers 32 --steps 10 --warmup 5 --graph --no-profile > gpurun_out/kb84_$r.json 2>&1; done
FREEKV_TRACE=1 timeout 600 python tools/trace_step.py --graph --dump > gpurun_out/trace84.json 2> gpurun_out/trace84.err
