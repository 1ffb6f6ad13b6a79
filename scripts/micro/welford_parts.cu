// Which part of a Welford step costs: the TSDF chain alone, + variance,
// + the reciprocal of W + 1, one warp, cycles per step.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double div_by_int(double x, double n, double y) {
  const double q0 = x * y;
  const double r = __fma_rn(-q0, n, x);
  return __fma_rn(r, y, q0);
}

template <int kMode>
__global__ void k_part(double* out, long long* cyc, int n, double a, double b) {
  double D = a, S = 0, W = 1.0, y = 0.5;
  long long t0 = clock64();
  for (int i = 0; i < n; i++) {
    const double sdf = b * (double)(i & 7);
    const double w_old = W, d_old = D, n1 = w_old + 1.0;
    if (kMode >= 2) y = __drcp_rn(n1);
    const double num = w_old * d_old + sdf;
    const double d_new = div_by_int(num, n1, y);
    if (kMode >= 1) S = S + (sdf - d_old) * (sdf - d_new);
    D = d_new;
    W = n1;
  }
  long long t1 = clock64();
  out[threadIdx.x] = D + S + y;
  if (threadIdx.x == 0) cyc[kMode] = t1 - t0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 256);
  cudaMallocManaged(&cyc, 32);
  const int n = 100000;
  for (int rep = 0; rep < 2; rep++) {
    k_part<0><<<1, 32>>>(out, cyc, n, 1.0000001, 0.9999999);
    k_part<1><<<1, 32>>>(out, cyc, n, 1.0000001, 0.9999999);
    k_part<2><<<1, 32>>>(out, cyc, n, 1.0000001, 0.9999999);
    cudaDeviceSynchronize();
  }
  printf("{\"tsdf_chain\": %.1f, \"plus_variance\": %.1f, \"plus_reciprocal\": %.1f}\n", (double)cyc[0] / n,
         (double)cyc[1] / n, (double)cyc[2] / n);
  return 0;
}
