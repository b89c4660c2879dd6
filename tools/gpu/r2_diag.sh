# diagnostics: in-kernel globaltimer trace of one graph-replayed step (last layer), and the ncu
# launch list (serialised per-kernel durations) of a few c2 layers
python -c "import __graft_entry__ as g; g.build()"
timeout 300 python tools/trace_step.py --graph > gpurun_out/${TAG}_trace.json 2> gpurun_out/${TAG}_trace.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:fkv_ --csv --log-file gpurun_out/${TAG}_launches.csv python tools/kbench.py --layers 4 --steps 3 --warmup 3 ${KB_ARGS} > gpurun_out/${TAG}_ncu.log 2>&1
