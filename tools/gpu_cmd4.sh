python -c "import __graft_entry__ as g; g.build()"
K="python tools/kbench.py --layers 2 --steps 20 --warmup 5"
timeout 300 $K > gpurun_out/kb_par.json 2>&1
FREEKV_SERIAL_RECALL=1 timeout 300 $K > gpurun_out/kb_ser.json 2>&1
K2="python tools/kbench.py --layers 2 --steps 2 --warmup 5 --no-profile"
timeout 300 $K2 > gpurun_out/kb_plain.log 2>&1 && \
timeout 600 ncu -k regex:fkv_ --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 72 -c 28 --csv --log-file gpurun_out/kb_launches.csv $K2 > gpurun_out/ncu4a.log 2>&1 && \
timeout 600 ncu -k regex:fkv_attn_split --set full --import-source on --clock-control none -s 10 -c 1 -o gpurun_out/attn_r1 $K2 > gpurun_out/ncu4b.log 2>&1 && \
timeout 600 ncu -k regex:fkv_score --set full --import-source on --clock-control none -s 10 -c 1 -o gpurun_out/score_r1 $K2 > gpurun_out/ncu4c.log 2>&1
echo "rc=$?" >> gpurun_out/ncu4a.log
