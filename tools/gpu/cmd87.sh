python -c "import __graft_entry__ as g; g.build()"
AB_A="FREEKV_ATTN_SPEC=0" AB_B="FREEKV_ATTN_SPEC=1" bash tools/gpu/ab.sh
FREEKV_ATTN_SPEC=1 FREEKV_TRACE=1 timeout 600 python tools/trace_step.py --graph --dump > gpurun_out/trace87.json 2> gpurun_out/trace87.err
