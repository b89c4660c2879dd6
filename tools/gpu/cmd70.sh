for v in "FREEKV_SERIAL_RECALL=0" "FREEKV_SERIAL_RECALL=1" "FREEKV_RECALL_MODE=ld" "FREEKV_RECALL_BG_CTAS=4"; do
env $v FREEKV_TRACE=1 timeout 600 python tools/trace_step.py --graph > "gpurun_out/trace70_${v}.json" 2> gpurun_out/trace70.err
done
