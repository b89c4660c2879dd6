# A/B on one box: alternate the variants, 3 rounds each (env strings in $AB_A / $AB_B)
python -c "import __graft_entry__ as g; g.build()"
for r in 1 2 3; do
  env $AB_A timeout 300 python tools/kbench.py --layers 32 --steps 10 --warmup 5 --graph --no-profile > gpurun_out/ab_A_$r.json 2>&1
  env $AB_B timeout 300 python tools/kbench.py --layers 32 --steps 10 --warmup 5 --graph --no-profile > gpurun_out/ab_B_$r.json 2>&1
done
