python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest21.log 2>&1; echo "rc=$?" >> gpurun_out/pytest21.log
timeout 600 python tools/trace_step.py > gpurun_out/trace21.json 2> gpurun_out/trace21.err
for cfg in "32 8" "16 4" "64 16" "148 148"; do set -- $cfg; FREEKV_RECALL_SYNC_CTAS=$1 FREEKV_RECALL_BG_CTAS=$2 timeout 300 python tools/kbench.py --layers 4 --steps 20 --warmup 5 --graph --no-profile > gpurun_out/kb21_$1_$2.json 2>&1; done
FREEKV_DEBUG_FULL_REFRESH=1 timeout 300 python tools/kbench.py --layers 4 --steps 10 --warmup 3 --graph > gpurun_out/kb21_genx.json 2>&1
