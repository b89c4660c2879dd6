./tools/micro/kchain > gpurun_out/kchain.txt 2>&1
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python bench.py --steps 16 --warmup 3 --profile-steps 4 --no-cpu-baseline > gpurun_out/bench12.json 2> gpurun_out/bench12.err
