python -c "import __graft_entry__ as g; g.build()"
for e in "FREEKV_OVERLAP=0" ; do
env $e timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:fkv_ --csv --log-file gpurun_out/${TAG}_launches.csv python tools/kbench.py --layers 4 --steps 3 --warmup 3 ${KB_ARGS} > gpurun_out/${TAG}_ncu.log 2>&1
done
