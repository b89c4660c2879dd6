# ncu --set full of the kernels matching $KREGEX launched by tools/iso_bench.py (isolated, L2 flushed)
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"${KREGEX:-fkv_score}" --launch-skip ${SKIP:-6} --launch-count ${COUNT:-1} -o gpurun_out/${TAG}_iso python tools/iso_bench.py --config ${CFG:-c2} --reps 3 > gpurun_out/${TAG}_iso.log 2>&1
