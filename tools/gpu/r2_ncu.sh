# one ncu --set full capture of the score, select and attention kernels (c2 shape, eager kbench)
python -c "import __graft_entry__ as g; g.build()"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"fkv_(score|select|attn_cluster)" --launch-skip ${SKIP:-30} --launch-count ${COUNT:-3} -o gpurun_out/${TAG}_full python tools/kbench.py --layers 2 --steps 4 --warmup 4 ${KB_ARGS} > gpurun_out/${TAG}_ncufull.log 2>&1
