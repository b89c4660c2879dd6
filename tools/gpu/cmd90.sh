python -c "import __graft_entry__ as g; g.build()"
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest90.log 2>&1; echo "rc=$?" >> gpurun_out/pytest90.log
