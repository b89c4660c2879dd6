python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest27.log 2>&1; echo "rc=$?" >> gpurun_out/pytest27.log
FREEKV_TRACE=1 timeout 600 python tools/trace_step.py --graph > gpurun_out/trace27.json 2> gpurun_out/trace27.err
for mp in 1 2 4; do
FREEKV_ATTN_MIN_PAGES=$mp timeout 300 python tools/kbench.py --layers 4 --steps 20 --warmup 5 --graph --no-profile > gpurun_out/kb27_$mp.json 2>&1
done
