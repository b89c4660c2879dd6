python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -q -x > gpurun_out/pytest92.log 2>&1; echo "rc=$?" >> gpurun_out/pytest92.log
AB_A="FREEKV_DEBUG_EXP=0" AB_B="FREEKV_DEBUG_EXP=8" bash tools/gpu/ab.sh
