python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest83.log 2>&1; echo "rc=$?" >> gpurun_out/pytest83.log
timeout 900 python bench.py > gpurun_out/bench83.json 2> gpurun_out/bench83.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench83_ref.json 2> gpurun_out/bench83_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:fkv_ --csv --log-file gpurun_out/launches83.csv python bench.py --steps 2 --warmup 3 --profile-steps 1 --no-cpu-baseline > gpurun_out/ncu83.log 2>&1
