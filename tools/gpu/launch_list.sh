# ncu launch list of the bench command (cold, serialised per-launch times; see B200_PROFILING.md)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:fkv_ --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --profile-steps 1 --no-cpu-baseline \
  > gpurun_out/ncu_launches.log 2>&1
