python -c "import __graft_entry__ as g; g.build()"
for v in 0 8 16 24; do
FREEKV_DEBUG_EXP=$v FREEKV_TRACE=1 timeout 600 python tools/trace_step.py --graph > gpurun_out/trace69_$v.json 2> gpurun_out/trace69_$v.err
done
