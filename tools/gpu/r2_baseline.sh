# round-2 baseline on one box: bench c2/c3 lines and per-kernel in-graph times
python -c "import __graft_entry__ as g; g.build()"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2b_smi.txt
timeout 300 python bench.py --config c2 --steps 128 --no-cpu-baseline > gpurun_out/r2b_c2.json 2> gpurun_out/r2b_c2.err
timeout 300 python bench.py --config c3 --steps 128 --no-cpu-baseline > gpurun_out/r2b_c3.json 2> gpurun_out/r2b_c3.err
timeout 300 python tools/kbench.py --layers 4 --steps 10 --warmup 5 --graph > gpurun_out/r2b_k_c2.json 2>&1
timeout 300 python tools/kbench.py --layers 4 --steps 10 --warmup 5 --graph --ctx 131072 --batch 4 --n_qo 28 --n_kv 4 > gpurun_out/r2b_k_c3.json 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:fkv_ --launch-skip 24 --launch-count 4 -o gpurun_out/r2b_c3 python tools/kbench.py --layers 2 --steps 3 --warmup 3 --ctx 131072 --batch 4 --n_qo 28 --n_kv 4 > gpurun_out/r2b_ncu_c3.log 2>&1
