python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest16.log 2>&1; echo "rc=$?" >> gpurun_out/pytest16.log
timeout 300 python tools/kbench.py --layers 4 --steps 20 --warmup 5 --graph --no-profile > gpurun_out/kb16_graph_noprof.json 2>&1
K2="python tools/kbench.py --layers 2 --steps 2 --warmup 5 --no-profile"
timeout 300 $K2 > gpurun_out/kb16_plain.log 2>&1 && \
timeout 600 ncu -k regex:fkv_ --cache-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_active.avg,sm__cycles_active.max --clock-control none -s 70 -c 28 --csv --log-file gpurun_out/kb16_launches.csv $K2 > gpurun_out/ncu16.log 2>&1 && \
timeout 600 ncu -k regex:"fkv_attn_split" --cache-control none --set full --import-source on --clock-control none -s 4 -c 1 -o gpurun_out/r16 $K2 > gpurun_out/ncu16b.log 2>&1
echo "rc=$?" >> gpurun_out/ncu16.log
