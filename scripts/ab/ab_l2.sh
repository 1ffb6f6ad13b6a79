for r in 1 2; do
  for p in 1 0; do
    TSDF_L2_PERSIST=$p timeout 600 python bench.py --workload room_fixed5mm --no-lidar --no-cpu-baseline > gpurun_out/abl2_fixed_p${p}_$r.json 2>/dev/null
    TSDF_L2_PERSIST=$p timeout 600 python bench.py --no-lidar --no-cpu-baseline > gpurun_out/abl2_room_p${p}_$r.json 2>/dev/null
  done
done
