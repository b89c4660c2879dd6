# A/B of runtime knobs after the select-width change (bench.py --steps 64 --warmup 4)
run() { name=$1; cfg=$2; shift 2; env "$@" timeout 300 python bench.py --config $cfg --steps 64 --warmup 4 --no-cpu-baseline > gpurun_out/kn_${name}_${cfg}.json 2> gpurun_out/kn_${name}_${cfg}.err; }
for cfg in c2 c3; do
  run base $cfg X=1
  run st2 $cfg FREEKV_ATTN_STAGES=2
  run bg32 $cfg FREEKV_RECALL_BG_CTAS=32
  run bg8 $cfg FREEKV_RECALL_BG_CTAS=8
done
