python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest25.log 2>&1; echo "rc=$?" >> gpurun_out/pytest25.log
timeout 600 python tools/trace_step.py --graph > gpurun_out/trace25.json 2> gpurun_out/trace25.err
timeout 300 python tools/kbench.py --layers 4 --steps 20 --warmup 5 --graph --no-profile > gpurun_out/kb25.json 2>&1
