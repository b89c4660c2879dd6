python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest55.log 2>&1; echo "rc=$?" >> gpurun_out/pytest55.log
FREEKV_PIPELINE=1 FREEKV_TRACE=1 timeout 600 python tools/trace_step.py --graph > gpurun_out/trace55.json 2> gpurun_out/trace55.err
for v in "FREEKV_PIPELINE=0" "FREEKV_PIPELINE=1"; do
env $v timeout 310 python tools/kbench.py --layers 32 --steps 10 --warmup 5 --graph --no-profile > "gpurun_out/kb55_${v}.json" 2>&1
done
