set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py > gpurun_out/bench_room.json 2> gpurun_out/bench_room.err
timeout 900 python bench.py --workload lidar --no-cpu-baseline > gpurun_out/bench_lidar.json 2> gpurun_out/bench_lidar.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_room.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_dda_walk -s 30 -c 1 -o gpurun_out/dda_walk python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_dda.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_depth_update -s 30 -c 1 -o gpurun_out/depth_update python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_du.log 2>&1
tail -3 gpurun_out/*.log
