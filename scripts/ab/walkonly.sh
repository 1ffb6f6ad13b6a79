for v in ${VARIANTS:-F H F H}; do
  cp scripts/ab/fusion_$v.cu paper_2511_21459_b200/csrc/fusion.cu
  (cd paper_2511_21459_b200/csrc && make -s -j8 > /dev/null 2>&1)
  python - <<'P' > gpurun_out/walkonly_$v.txt 2>&1
import sys, torch
sys.path.insert(0, '.')
import bench
import paper_2511_21459_b200 as P
wl = bench.WORKLOADS["room"]
frames = bench.make_frames(wl, 40)
dev = [(torch.as_tensor(f[0]).cuda(), torch.as_tensor(f[1]).cuda()) for f in frames]
t = bench.make_table(P, wl, stream=torch.cuda.current_stream().cuda_stream)
for w in range(2):
    bench.window_and_merge(P, t, wl, frames[10*w:10*w+10], dev[10*w:10*w+10])
t.profile(True); t.kernel_times(reset=True)
for w in range(2, 4):
    bench.window_and_merge(P, t, wl, frames[10*w:10*w+10], dev[10*w:10*w+10])
torch.cuda.synchronize()
kt = t.kernel_times(reset=True)
print({k: round(v[0] / v[1] * 1e3, 1) for k, v in kt.items() if k in ("k_dda_walk", "k_depth_frame")})
P
  cat gpurun_out/walkonly_$v.txt | tail -1
done
