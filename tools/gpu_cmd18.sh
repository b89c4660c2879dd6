python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest18.log 2>&1; echo "rc=$?" >> gpurun_out/pytest18.log
timeout 900 python bench.py --steps 32 --warmup 4 --profile-steps 4 --cpu-sample-s 12 > gpurun_out/bench18.json 2> gpurun_out/bench18.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 --cpu-sample-s 10 > gpurun_out/bench18_ref.json 2> gpurun_out/bench18_ref.err
