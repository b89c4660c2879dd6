# round-2 evidence: ncu launch lists of the bench command (c2, c3) and ncu --set full captures of the
# score + select (one select_pages) and the attention (one launch) per config, isolated (tools/iso_bench.py)
python -c "import __graft_entry__ as g; g.build()"
for c in ${CFGS:-c2 c3}; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:fkv_ --csv \
    --log-file gpurun_out/${TAG}_launches_$c.csv python bench.py --config $c --steps 2 --warmup 3 --profile-steps 1 \
    --no-cpu-baseline --no-extras > gpurun_out/${TAG}_launches_$c.log 2>&1
  timeout 900 ncu --set full --clock-control none -k regex:"fkv_(score|select)" \
    --launch-skip 8 --launch-count 2 -o gpurun_out/${TAG}_full_sel_$c python tools/iso_bench.py --config $c --reps 3 \
    > gpurun_out/${TAG}_full_sel_$c.log 2>&1
  timeout 900 ncu --set full --clock-control none -k regex:"fkv_attn_cluster" \
    --launch-skip 4 --launch-count 1 -o gpurun_out/${TAG}_full_attn_$c python tools/iso_bench.py --config $c --reps 3 \
    > gpurun_out/${TAG}_full_attn_$c.log 2>&1
done
# summaries on the box; the raw reports come back only while gpurun_out stays small
for f in gpurun_out/${TAG}_full_*.ncu-rep; do python tools/ncu_summary.py $f > ${f%.ncu-rep}.txt 2>&1; done
for f in gpurun_out/${TAG}_launches_*.csv; do python tools/launches_summary.py $f > ${f%.csv}_summary.txt 2>&1; gzip -f $f; done
du -sh gpurun_out/* > gpurun_out/${TAG}_sizes.txt
for f in gpurun_out/${TAG}_full_*.ncu-rep; do
  if [ $(du -sm gpurun_out | cut -f1) -gt 48 ]; then rm -f $f; fi
done
