# round-2 bench lines: headline (c2, default command), reference arm, c1/c3/c5, c4 tau sweep
python -c "import __graft_entry__ as g; g.build()"
timeout 900 python bench.py > gpurun_out/${TAG}_c2.json 2> gpurun_out/${TAG}_c2.err
timeout 600 python bench.py --impl reference > gpurun_out/${TAG}_reference.json 2> gpurun_out/${TAG}_reference.err
for c in c1 c3; do
  timeout 600 python bench.py --config $c --no-extras --no-cpu-baseline > gpurun_out/${TAG}_$c.json 2> gpurun_out/${TAG}_$c.err
done
timeout 900 python bench.py --config c5 --steps 64 --no-extras --no-cpu-baseline > gpurun_out/${TAG}_c5.json 2> gpurun_out/${TAG}_c5.err
for t in 0 0.8 0.9 1.0; do
  timeout 600 python bench.py --config c4 --tau $t --steps 128 --no-extras --no-cpu-baseline > gpurun_out/${TAG}_c4_tau$t.json 2> gpurun_out/${TAG}_c4_tau$t.err
done
