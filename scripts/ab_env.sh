# A/B over environment toggles on one box: every combination in COMBOS
# ("NAME:VAR=VAL,VAR=VAL ...") runs bench.py twice; outputs gpurun_out/abenv_<NAME>_<run>.json
for combo in ${COMBOS}; do
  name=${combo%%:*}; envs=${combo#*:}
  for r in 1 2; do
    env $(echo $envs | tr ',' ' ') timeout 300 python bench.py --no-cpu-baseline --no-lidar ${BENCH_ARGS} \
      > gpurun_out/abenv_${name}_${r}.json 2> gpurun_out/abenv_${name}_${r}.err
  done
done
