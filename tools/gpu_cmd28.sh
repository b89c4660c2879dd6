python -c "import __graft_entry__ as g; g.build()"
timeout 300 python tools/kbench.py --layers 4 --steps 20 --warmup 5 --graph --no-profile --event_rate 0 > gpurun_out/kb28_e0.json 2>&1
FKV_EVENT_RATE=0 FREEKV_TRACE=1 timeout 600 python tools/trace_step.py --graph > gpurun_out/trace28_e0.json 2> gpurun_out/trace28.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"fkv_(select_finalize|score|attn_split|attn_combine)" --launch-skip 24 --launch-count 4 -o gpurun_out/ncu28 -f python tools/kbench.py --layers 2 --steps 3 --warmup 2 --no-profile > gpurun_out/ncu28.log 2>&1
