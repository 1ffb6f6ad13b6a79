# LiDAR chunked mode: hot-segment threshold (rays per block) sweep, two runs each
for h in ${HOTS:-128 256 512}; do
  for r in 1 2; do
    TSDF_LIDAR_HOT=$h timeout 400 python bench.py --workload lidar --no-cpu-baseline --steps 5 \
      > gpurun_out/lidar_hot_${h}_${r}.json 2> /dev/null
  done
done
