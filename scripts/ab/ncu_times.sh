# isolated per-kernel times (ncu launch list) for each fusion_<V>.cu variant
for v in ${VARIANTS}; do
  cp scripts/ab/fusion_$v.cu paper_2511_21459_b200/csrc/fusion.cu
  (cd paper_2511_21459_b200/csrc && make -s -j8 > /dev/null 2>&1)
  env ${ENVS} timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"${KREGEX}" \
    --csv --log-file gpurun_out/times_$v.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-lidar \
    > /dev/null 2>&1
done
