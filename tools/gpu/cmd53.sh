python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest53.log 2>&1; echo "rc=$?" >> gpurun_out/pytest53.log
for t in 256 512 1024; do
FREEKV_SELECT_THREADS=$t timeout 310 python tools/kbench.py --layers 32 --steps 10 --warmup 5 --graph --no-profile > gpurun_out/kb53_$t.json 2>&1
done
FREEKV_SELECT_THREADS=256 FREEKV_TRACE=1 timeout 600 python tools/trace_step.py --graph > gpurun_out/trace53.json 2> gpurun_out/trace53.err
