for v in I2 N I2 N; do
  cp scripts/ab/fusion_$v.cu paper_2511_21459_b200/csrc/fusion.cu
  (cd paper_2511_21459_b200/csrc && make -s -j8 > /dev/null 2>&1)
  timeout 600 python bench.py --workload room_fixed5mm --no-lidar --no-cpu-baseline > gpurun_out/abf_${v}_$RANDOM.json 2>/dev/null
done
