# final-build lines for BASELINE configs 4 and 5 (depth part) and the N=2 path (gloo, ranks share the GPU)
timeout 900 python bench.py --workload room_fixed5mm --no-lidar > gpurun_out/bench_fixed5mm.json 2> gpurun_out/bench_fixed5mm.err
timeout 900 python bench.py --workload room1024 --no-lidar > gpurun_out/bench_room1024.json 2> gpurun_out/bench_room1024.err
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 \
  bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo --no-lidar > gpurun_out/bench_2rank.json 2> gpurun_out/bench_2rank.err
