# ncu --set full of one launch per "kernel_regex:ENV=V,ENV=V" item in CAPS
# (one GPU, serial): gpurun_out/${TAG}_<kernel>.ncu-rep
for item in ${CAPS}; do
  k=${item%%:*}; envs=${item#*:}
  [ "$envs" = "$item" ] && envs=""
  env $(echo $envs | tr ',' ' ') timeout 900 ncu --set full --clock-control none --import-source on \
    -k regex:${k} -s ${SKIP:-30} -c 1 -o gpurun_out/${TAG}_${k} \
    python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-lidar ${BENCH_ARGS} \
    > gpurun_out/${TAG}_${k}.log 2>&1
done
