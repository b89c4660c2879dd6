python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest22.log 2>&1; echo "rc=$?" >> gpurun_out/pytest22.log
timeout 600 python tools/trace_step.py > gpurun_out/trace22.json 2> gpurun_out/trace22.err
timeout 300 python tools/kbench.py --layers 4 --steps 20 --warmup 5 --graph --no-profile > gpurun_out/kb22_fused.json 2>&1
FREEKV_SELECT=split timeout 300 python tools/kbench.py --layers 4 --steps 20 --warmup 5 --graph --no-profile > gpurun_out/kb22_split.json 2>&1
