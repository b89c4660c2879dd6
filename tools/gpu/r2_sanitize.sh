# compute-sanitizer over the default kernels (tools/sanitize_run.py), logs -> gpurun_out/${TAG}_san_*
for cfg in c1 c2s; do
  for tool in memcheck racecheck synccheck; do
    timeout 900 compute-sanitizer --tool $tool --error-exitcode 9 --print-limit 50 python tools/sanitize_run.py $cfg > gpurun_out/${TAG}_san_${tool}_${cfg}.log 2>&1
    echo "exit=$?" >> gpurun_out/${TAG}_san_${tool}_${cfg}.log
  done
done
