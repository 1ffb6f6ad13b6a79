# compute-sanitizer over the late round-2 kernels (scripts/sanitize_session3.py)
mkdir -p gpurun_out/san
for tool in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 python scripts/sanitize_session3.py \
    > gpurun_out/san/s3_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/san/s3_summary.txt
  tail -3 gpurun_out/san/s3_$tool.log >> gpurun_out/san/s3_summary.txt
done
