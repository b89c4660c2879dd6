timeout 600 ncu --metrics gpu__time_duration.sum -k regex:fkv_ --launch-count 40 --csv python tools/kbench.py --layers 2 --steps 3 --warmup 3 --no-profile > gpurun_out/ncu57.log 2>&1
