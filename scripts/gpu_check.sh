# round-2 iteration: GPU parity suite (or a subset via TESTS) + room and lidar bench lines
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi.txt
timeout 1200 python -m pytest ${TESTS:-tests} -m gpu -x -q -s 2>&1 | tail -40 > gpurun_out/pytest_gpu.log; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_room.json 2> gpurun_out/bench_room.err
timeout 900 python bench.py --workload lidar --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_lidar.json 2> gpurun_out/bench_lidar.err
tail -5 gpurun_out/pytest_gpu.log
