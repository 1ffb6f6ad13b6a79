for v in A D; do
  cp scripts/ab/fusion_$v.cu paper_2511_21459_b200/csrc/fusion.cu
  (cd paper_2511_21459_b200/csrc && make -s -j8 > /dev/null 2>&1)
  for c in 1 2 4; do echo "== $v cluster $c"; TSDF_WALK_CLUSTER=$c timeout 300 python scripts/ab/cl_diag.py 2>&1 | tail -3; done
done > gpurun_out/cl_diag.txt 2>&1
