# ncu --set full capture of one launch of each named kernel (one GPU, serial)
# usage: KERNELS="k_depth_update k_depth_near" TAG=v3 bash scripts/gpu_ncu.sh
for k in ${KERNELS}; do
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:${k} -s 30 -c 1 \
    -o gpurun_out/${TAG}_${k} python bench.py --steps 1 --warmup 3 --no-cpu-baseline ${BENCH_ARGS} \
    > gpurun_out/${TAG}_${k}.log 2>&1
done
ls -la gpurun_out
