python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest5.log 2>&1; echo "rc=$?" >> gpurun_out/pytest5.log
K="python tools/kbench.py --layers 2 --steps 20 --warmup 5"
timeout 300 $K > gpurun_out/kb5_par.json 2>&1
FREEKV_SERIAL_RECALL=1 timeout 300 $K > gpurun_out/kb5_ser.json 2>&1
K2="python tools/kbench.py --layers 2 --steps 2 --warmup 5 --no-profile"
timeout 300 $K2 > gpurun_out/kb5_plain.log 2>&1 && \
timeout 600 ncu -k regex:fkv_ --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -s 72 -c 28 --csv --log-file gpurun_out/kb5_launches.csv $K2 > gpurun_out/ncu5.log 2>&1
echo "rc=$?" >> gpurun_out/ncu5.log
