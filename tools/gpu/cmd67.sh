python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest67.log 2>&1; echo "rc=$?" >> gpurun_out/pytest67.log
timeout 900 python bench.py > gpurun_out/bench67.json 2> gpurun_out/bench67.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:fkv_ --csv --log-file gpurun_out/launches67.csv python bench.py --steps 2 --warmup 3 --profile-steps 1 --no-cpu-baseline > gpurun_out/ncu67.log 2>&1
