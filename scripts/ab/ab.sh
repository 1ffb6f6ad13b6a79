# A/B: bench each fusion_*.cu variant on the same box (rebuilds in place);
# every pass keeps its own output: gpurun_out/ab_<variant>_<pass><run>.json
p=0
for v in ${VARIANTS:-A B}; do
  p=$((p + 1))
  cp scripts/ab/fusion_$v.cu paper_2511_21459_b200/csrc/fusion.cu
  (cd paper_2511_21459_b200/csrc && make -s -j8 > /dev/null 2>&1)
  for r in 1 2; do
    python bench.py --no-cpu-baseline --steps 5 ${BENCH_ARGS} > gpurun_out/ab_${v}_${p}${r}.json 2>/dev/null
  done
done
