python -c "import __graft_entry__ as g; g.build()"
timeout 900 python bench.py --steps 16 --warmup 3 --profile-steps 4 --no-cpu-baseline > gpurun_out/bench2.json 2> gpurun_out/bench2.err
B="python bench.py --steps 2 --warmup 3 --profile-steps 1 --no-cpu-baseline"
timeout 600 $B > gpurun_out/plain3.log 2>&1 && timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -s 704 -c 448 --csv --log-file gpurun_out/launches_r1.csv $B > gpurun_out/ncu3.log 2>&1
echo "rc=$?" >> gpurun_out/ncu3.log
