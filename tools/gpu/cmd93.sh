python -c "import __graft_entry__ as g; g.build()"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke93.log 2>&1; echo "rc=$?" >> gpurun_out/smoke93.log
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest93.log 2>&1; echo "rc=$?" >> gpurun_out/pytest93.log
timeout 900 python bench.py > gpurun_out/bench93.json 2> gpurun_out/bench93.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:fkv_ --csv --log-file gpurun_out/launches93.csv python bench.py --steps 2 --warmup 3 --profile-steps 1 --no-cpu-baseline > gpurun_out/ncu93.log 2>&1
