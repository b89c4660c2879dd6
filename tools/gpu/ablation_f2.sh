# B200 analog of the paper's efficiency ablation (fig:eff-abl).
#  HL (transfer unit): full-refresh synchronous recall (every unit re-fetches K pages per layer,
#     32 MiB per layer at c2) moving each 16 KiB page as one bulk copy vs 256-byte pieces (one
#     (token, head) row, i.e. an NHD host layout) vs 4 KiB pieces vs SM loads.
#  DB (overlap of the recall): background recall overlapped (own stream) vs serial.
#  SR (speculative retrieval): speculative (tau 0.8) vs correction every step (mode 1) vs the
#     paper's synchronous recall order, and no correction at all (mode 2).
python -c "import __graft_entry__ as g; g.build()"
: > gpurun_out/ablation_f2.jsonl
run() {  # label, env, kbench args
  out=$(env $2 timeout 300 python tools/kbench.py --graph --no-profile $3 2>/dev/null | tail -1)
  echo "{\"label\": \"$1\", \"env\": \"$2\", \"args\": \"$3\", \"result\": $out}" >> gpurun_out/ablation_f2.jsonl
}
FR="--layers 4 --steps 6 --warmup 3"
run "HL page 16KiB"      "FREEKV_CORR=recall FREEKV_DEBUG_FULL_REFRESH=1" "$FR"
run "HL frag 4KiB"       "FREEKV_CORR=recall FREEKV_DEBUG_FULL_REFRESH=1 FREEKV_RECALL_FRAG=4096" "$FR"
run "HL frag 256B (NHD)" "FREEKV_CORR=recall FREEKV_DEBUG_FULL_REFRESH=1 FREEKV_RECALL_FRAG=256" "$FR"
ST="--layers 32 --steps 10 --warmup 5"
for r in 1 2; do
run "SR speculative (default)" "BASE=1" "$ST"
run "SR correct every step"    "BASE=1" "$ST --mode 1"
run "SR never correct"         "BASE=1" "$ST --mode 2"
run "SR paper order (sync recall)" "FREEKV_CORR=recall" "$ST"
run "DB recall serial"         "FREEKV_SERIAL_RECALL=1" "$ST"
done
