# One ncu --set full capture per main kernel of the current build (room and
# lidar workloads), for profiles/ncu_summary.json (scripts/ncu_build_summary.py)
set -x
mkdir -p gpurun_out/final
for k in k_dda_walk k_depth_frame k_depth_near k_depth_sub k_depth_micro k_depth_screen k_depth_exact k_block_stats k_merge_apply; do
  skip=30; case $k in k_block_stats|k_merge_apply) skip=3;; esac
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"^${k}" -s $skip -c 1 \
    -o gpurun_out/final/room_${k} python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-lidar \
    > gpurun_out/final/room_${k}.log 2>&1
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"k_mc" -s 0 -c 1 \
  -o gpurun_out/final/room_k_mc python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-lidar \
  > gpurun_out/final/room_k_mc.log 2>&1
for k in k_lidar_update k_lidar_hot_mask k_lidar_hot_partial k_lidar_hot_combine k_pair_resolve; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:"${k}" -s 20 -c 1 \
    -o gpurun_out/final/lidar_${k} python bench.py --workload lidar --steps 1 --warmup 3 --no-cpu-baseline \
    > gpurun_out/final/lidar_${k}.log 2>&1
done
timeout 900 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,dram__bytes_read.sum,dram__bytes_write.sum \
  --clock-control none --csv --log-file gpurun_out/final/room_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-lidar > /dev/null 2>&1
# summaries here (the reports are too big to bring back)
mkdir -p gpurun_out/final_md
for r in gpurun_out/final/*.ncu-rep; do
  python scripts/ncu_summary.py $r gpurun_out/final_md/$(basename $r .ncu-rep).md > /dev/null 2>&1
done
NCU_SUMMARY_OUT=gpurun_out/final_md/ncu_summary.json python scripts/ncu_build_summary.py \
  "ncu --set full --clock-control none, one launch per kernel of this build (scripts/gpu_final_ncu.sh): room workload (bench.py --steps 1 --warmup 3) and lidar workload (chunked mode)" \
  gpurun_out/final/*.ncu-rep > /dev/null 2>&1
cp gpurun_out/final/*.csv gpurun_out/final_md/ 2>/dev/null
rm -f gpurun_out/final/*.ncu-rep
ls -la gpurun_out/final_md
