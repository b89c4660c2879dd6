# one gpurun call: build, smoke, GPU tests, both bench arms, then the ncu launch list of the
# bench command (after the same command has exited 0 without ncu)
python -c "import __graft_entry__ as g; g.build()"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest.log 2>&1; echo "rc=$?" >> gpurun_out/pytest.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err
timeout 900 python bench.py --steps 2 --warmup 3 --profile-steps 1 --no-cpu-baseline > /dev/null 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:fkv_ --csv \
  --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 3 --profile-steps 1 --no-cpu-baseline \
  > gpurun_out/ncu.log 2>&1
