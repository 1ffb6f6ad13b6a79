timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --dist-backend gloo > gpurun_out/bench_2rank.json 2> gpurun_out/bench_2rank.err
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_room.json 2> gpurun_out/bench_room.err
