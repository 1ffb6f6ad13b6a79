// Throughput microbenchmark of the walk's inner loop (k_dda_walk): the
// lock-step FP64 DDA step of dda.py:64-82 alone, with the per-CTA smem
// "already queued" filter, and with two rays interleaved per thread.
// Synthetic rays from one origin (like a depth frame), ~100 cells long.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 --fmad=false -o dda_step dda_step.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

struct Ray {
  double tm[3], td[3];
  uint32_t key, lkey, inc[3];
};

__device__ __forceinline__ uint32_t step(double& tx, double& ty, double& tz, uint32_t& key, uint32_t it,
                                         double dx, double dy, double dz, uint32_t lkey, uint32_t cap,
                                         uint32_t ix, uint32_t iy, uint32_t iz) {
  const bool py = ty < tx;
  const double m1 = py ? ty : tx;
  const bool pz = tz < m1;
  const double m = pz ? tz : m1;
  if (m > 1.0 || key == lkey || it >= cap) return 1;
  if (pz) tz += dz;
  else if (py) ty += dy;
  else tx += dx;
  key += pz ? iz : (py ? iy : ix);
  return 0;
}

__device__ void make_ray(uint64_t r, Ray& R) {
  // direction from a hash of r, length 60-120 cells, origin (0.3, 0.4, 0.5)
  uint64_t h = r * 0x9E3779B97F4A7C15ull;
  double d[3];
  for (int a = 0; a < 3; a++) {
    h ^= h >> 29;
    h *= 0xBF58476D1CE4E5B9ull;
    d[a] = ((double)(h >> 11) / 9007199254740992.0) * 2.0 - 1.0;
  }
  const double L = 60.0 + (double)(r % 61);
  const double o[3] = {0.3, 0.4, 0.5};
  const double n = sqrt(d[0] * d[0] + d[1] * d[1] + d[2] * d[2]) + 1e-9;
  uint32_t key = 512u << 20 | 512u << 10 | 512u, lkey = 0;
  int last[3];
  for (int a = 0; a < 3; a++) {
    const double e = o[a] + d[a] / n * L, dd = e - o[a];
    last[a] = (int)floor(e);
    const int st = dd > 0 ? 1 : (dd < 0 ? -1 : 0);
    R.tm[a] = dd != 0 ? ((double)(st > 0 ? 1 : 0) - o[a]) / dd : 1e300;
    R.td[a] = dd != 0 ? 1.0 / fabs(dd) : 1e300;
    const uint32_t u = 1u << (20 - 10 * a);
    R.inc[a] = st > 0 ? u : (st < 0 ? 0u - u : 0u);
  }
  lkey = (uint32_t)(last[0] + 512) << 20 | (uint32_t)(last[1] + 512) << 10 | (uint32_t)(last[2] + 512);
  R.key = key;
  R.lkey = lkey;
}

// kMode 0: DDA only; 1: DDA + smem filter; 2: two rays per thread + filter
template <int kMode>
__global__ void __launch_bounds__(256) k_bench(uint64_t n_rays, unsigned long long* steps_out,
                                               unsigned long long* queued) {
  __shared__ uint32_t set[4096];
  for (int i = threadIdx.x; i < 4096; i += 256) set[i] = ~0u;
  __syncthreads();
  unsigned long long steps = 0, q = 0;
  const int per = kMode == 2 ? 2 : 1;
  const uint64_t r0 = ((uint64_t)blockIdx.x * 256 + threadIdx.x) * per;
  if (r0 >= n_rays) return;
  auto visit = [&](uint32_t k) {
    const uint32_t h = (k * 0x9E3779B1u) >> 20;
    if (set[h] != k && atomicExch(&set[h], k) != k) q++;
  };
  if (kMode < 2) {
    Ray R;
    make_ray(r0 / 16, R);  // 16 neighbouring threads share a ray: filter hits like a tile
    double tx = R.tm[0], ty = R.tm[1], tz = R.tm[2];
    uint32_t key = R.key, it = 0;
    for (;;) {
      if (step(tx, ty, tz, key, it, R.td[0], R.td[1], R.td[2], R.lkey, 100000, R.inc[0], R.inc[1], R.inc[2]))
        break;
      it++;
      if (kMode == 1) visit(key);
    }
    steps = it;
  } else {
    Ray A, B;
    make_ray(r0 / 16, A);
    make_ray((r0 + 1) / 16 + 7777, B);
    double ax = A.tm[0], ay = A.tm[1], az = A.tm[2], bx = B.tm[0], by = B.tm[1], bz = B.tm[2];
    uint32_t ka = A.key, kb = B.key, ia = 0, ib = 0;
    bool la = true, lb = true;
    while (la || lb) {
      if (la) {
        if (step(ax, ay, az, ka, ia, A.td[0], A.td[1], A.td[2], A.lkey, 100000, A.inc[0], A.inc[1], A.inc[2]))
          la = false;
        else {
          ia++;
          visit(ka);
        }
      }
      if (lb) {
        if (step(bx, by, bz, kb, ib, B.td[0], B.td[1], B.td[2], B.lkey, 100000, B.inc[0], B.inc[1], B.inc[2]))
          lb = false;
        else {
          ib++;
          visit(kb);
        }
      }
    }
    steps = ia + ib;
  }
  atomicAdd(steps_out, steps);
  atomicAdd(queued, q);
}

template <int kMode>
void run(uint64_t n_rays, const char* name) {
  unsigned long long *d, h[2];
  cudaMalloc(&d, 16);
  const int per = kMode == 2 ? 2 : 1;
  const unsigned grid = (unsigned)((n_rays / per + 255) / 256);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 5; rep++) {
    cudaMemset(d, 0, 16);
    cudaEventRecord(e0);
    k_bench<kMode><<<grid, 256>>>(n_rays, d, d + 1);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("%-28s %8.3f ms  %.3e steps  %.1f Gsteps/s  queued %.2f%%\n", name, best, (double)h[0],
         h[0] / best / 1e6, 100.0 * h[1] / (double)h[0]);
  cudaFree(d);
}

int main() {
  const uint64_t n = 307200;  // one 640x480 frame
  run<0>(n, "dda only");
  run<1>(n, "dda + smem filter");
  run<2>(n, "2 rays/thread + filter");
  return 0;
}
