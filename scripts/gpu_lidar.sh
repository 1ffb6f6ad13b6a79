# LiDAR iteration: LiDAR parity tests + the lidar workload bench
set -x
timeout 900 python -m pytest tests -m gpu -x -q -k "lidar or scan or config5" 2>&1 | tail -15 > gpurun_out/pytest_lidar.log
timeout 600 python bench.py --workload lidar ${BENCH_ARGS} > gpurun_out/bench_lidar.json 2> gpurun_out/bench_lidar.err
cat gpurun_out/pytest_lidar.log
