# Design ablation on one box (c2 shape, 32 layers, whole-step graphs): µs per layer for each
# environment switch, two alternating rounds.  Output: gpurun_out/ablation.jsonl
python -c "import __graft_entry__ as g; g.build()"
: > gpurun_out/ablation.jsonl
for r in 1 2; do
for v in "BASE=1" "FREEKV_SELECT=split" "FREEKV_ATTN=split" "FREEKV_CORR=recall" "FREEKV_PIPELINE=1" "FREEKV_PDL=0" \
         "FREEKV_RECALL_BG_CTAS=148" "FREEKV_SELECT_THREADS=1024" "FREEKV_ATTN_SPEC=1" "FREEKV_RECALL_MODE=ld"; do
  out=$(env $v timeout 300 python tools/kbench.py --layers 32 --steps 10 --warmup 5 --graph --no-profile 2>/dev/null | tail -1)
  echo "{\"variant\": \"$v\", \"round\": $r, \"result\": $out}" >> gpurun_out/ablation.jsonl
done
done
