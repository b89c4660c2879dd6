python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest14.log 2>&1; echo "rc=$?" >> gpurun_out/pytest14.log
timeout 300 python tools/kbench.py --layers 4 --steps 20 --warmup 5 --graph > gpurun_out/kb14_graph.json 2>&1
timeout 300 python tools/kbench.py --layers 4 --steps 20 --warmup 5 --graph --no-profile > gpurun_out/kb14_graph_noprof.json 2>&1
K2="python tools/kbench.py --layers 2 --steps 2 --warmup 5 --no-profile"
timeout 300 $K2 > gpurun_out/kb14_plain.log 2>&1 && \
timeout 600 ncu -k regex:fkv_ --cache-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 70 -c 28 --csv --log-file gpurun_out/kb14_launches.csv $K2 > gpurun_out/ncu14.log 2>&1 && \
timeout 600 ncu -k regex:"fkv_attn_split|fkv_select_finalize" --cache-control none --set full --import-source on --clock-control none -s 10 -c 3 -o gpurun_out/r14 $K2 > gpurun_out/ncu14b.log 2>&1
echo "rc=$?" >> gpurun_out/ncu14.log
timeout 900 python bench.py --steps 16 --warmup 3 --profile-steps 4 --no-cpu-baseline > gpurun_out/bench14.json 2> gpurun_out/bench14.err
