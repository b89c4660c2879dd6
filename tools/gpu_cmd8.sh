python -c "import __graft_entry__ as g; g.build()"
timeout 120 python tools/launch_floor.py > gpurun_out/launch_floor.json 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest8.log 2>&1; echo "rc=$?" >> gpurun_out/pytest8.log
K="python tools/kbench.py --layers 2 --steps 20 --warmup 5"
timeout 300 $K > gpurun_out/kb8_par.json 2>&1
K2="python tools/kbench.py --layers 2 --steps 2 --warmup 5 --no-profile"
timeout 300 $K2 > gpurun_out/kb8_plain.log 2>&1 && \
timeout 600 ncu -k regex:fkv_ --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 80 -c 32 --csv --log-file gpurun_out/kb8_launches.csv $K2 > gpurun_out/ncu8.log 2>&1 && \
timeout 600 ncu -k regex:fkv_score --set full --import-source on --clock-control none -s 10 -c 1 -o gpurun_out/score_r1c $K2 > gpurun_out/ncu8b.log 2>&1 && \
timeout 600 ncu -k regex:fkv_attn_combine --set full --import-source on --clock-control none -s 10 -c 1 -o gpurun_out/comb_r1 $K2 > gpurun_out/ncu8c.log 2>&1 && \
timeout 600 ncu -k regex:fkv_append --set full --import-source on --clock-control none -s 10 -c 1 -o gpurun_out/app_r1 $K2 > gpurun_out/ncu8d.log 2>&1
echo "rc=$?" >> gpurun_out/ncu8.log
