python -c "import __graft_entry__ as g; g.build()"
FREEKV_FIN_THREADS=512 FREEKV_ATTN_SPEC=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "llama_shape or dense or ragged or modes" > gpurun_out/pytest88.log 2>&1; echo "rc=$?" >> gpurun_out/pytest88.log
for r in 1 2; do
for v in "FREEKV_ATTN_SPEC=0" "FREEKV_FIN_THREADS=512" "FREEKV_FIN_THREADS=512 FREEKV_ATTN_SPEC=1"; do
  out=$(env $v timeout 300 python tools/kbench.py --layers 32 --steps 10 --warmup 5 --graph --no-profile 2>/dev/null | tail -1)
  echo "$v $out" >> gpurun_out/ab88.txt
done; done
