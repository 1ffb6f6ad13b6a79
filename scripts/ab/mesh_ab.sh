# extraction time for each mesh_<V>.cu variant: bench extract ms (room) + mesh goldens
for v in ${VARIANTS}; do
  cp scripts/ab/mesh_$v.cu paper_2511_21459_b200/csrc/mesh.cu
  (cd paper_2511_21459_b200/csrc && make -s -j8 > /dev/null 2>&1)
  timeout 600 python -m pytest tests/test_gpu_mesh.py -m gpu -x -q 2>&1 | tail -1 > gpurun_out/mesh_test_$v.txt
  for r in 1 2; do
    timeout 300 python bench.py --no-cpu-baseline --no-lidar --steps 3 > gpurun_out/mesh_bench_${v}_$r.json 2>/dev/null
  done
done
