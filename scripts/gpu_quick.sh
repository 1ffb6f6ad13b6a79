# quick GPU iteration: parity suite + room bench (diagnostics in the JSON line)
set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline ${BENCH_ARGS} > gpurun_out/bench_room.json 2> gpurun_out/bench_room.err
cat gpurun_out/pytest_gpu.log
