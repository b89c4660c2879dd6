python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest9.log 2>&1; echo "rc=$?" >> gpurun_out/pytest9.log
K="python tools/kbench.py --layers 2 --steps 20 --warmup 5"
timeout 300 $K > gpurun_out/kb9_par.json 2>&1
K2="python tools/kbench.py --layers 2 --steps 2 --warmup 5 --no-profile"
timeout 300 $K2 > gpurun_out/kb9_plain.log 2>&1 && \
timeout 600 ncu -k regex:fkv_ --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_active.max,gpc__cycles_elapsed.max --clock-control none -s 80 -c 32 --csv --log-file gpurun_out/kb9_launches.csv $K2 > gpurun_out/ncu9.log 2>&1 && \
timeout 600 ncu -k regex:fkv_score --set full --import-source on --clock-control none -s 10 -c 1 -o gpurun_out/score_r1d $K2 > gpurun_out/ncu9b.log 2>&1
echo "rc=$?" >> gpurun_out/ncu9.log
timeout 900 python bench.py --steps 16 --warmup 3 --profile-steps 4 --no-cpu-baseline > gpurun_out/bench9.json 2> gpurun_out/bench9.err
