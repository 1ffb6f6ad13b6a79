// Dependent-latency microbenchmark: cycles per dependent FP64 op (DMUL, DFMA,
// DADD) and per Welford step as k_lidar_hot_apply runs it, one warp alone.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double div_by_int(double x, double n, double y) {
  const double q0 = x * y;
  const double r = __fma_rn(-q0, n, x);
  return __fma_rn(r, y, q0);
}

__global__ void k_lat(double* out, long long* cyc, int n, double a, double b) {
  double x = a, y = b;
  long long t0 = clock64();
  for (int i = 0; i < n; i++) x = __fma_rn(x, y, a);
  long long t1 = clock64();
  double z = a;
  for (int i = 0; i < n; i++) z = __dmul_rn(z, y);
  long long t2 = clock64();
  // Welford step chain (no colour, integer weights)
  double D = a, S = 0, W = 1.0, yn = __drcp_rn(W + 1.0);
  for (int i = 0; i < n; i++) {
    const double sdf = b * (double)(i & 7);
    const double w_old = W, d_old = D, n1 = w_old + 1.0, y1 = yn;
    const double num = w_old * d_old + sdf;
    const double d_new = div_by_int(num, n1, y1);
    S = S + (sdf - d_old) * (sdf - d_new);
    D = d_new;
    W = n1;
    yn = __drcp_rn(W + 1.0);
  }
  long long t3 = clock64();
  out[threadIdx.x] = x + z + D + S;
  if (threadIdx.x == 0) {
    cyc[0] = t1 - t0;
    cyc[1] = t2 - t1;
    cyc[2] = t3 - t2;
  }
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 32 * 8);
  cudaMallocManaged(&cyc, 3 * 8);
  const int n = 100000;
  k_lat<<<1, 32>>>(out, cyc, n, 1.0000001, 0.9999999);
  cudaDeviceSynchronize();
  k_lat<<<1, 32>>>(out, cyc, n, 1.0000001, 0.9999999);
  cudaDeviceSynchronize();
  printf("{\"dfma_cycles\": %.2f, \"dmul_cycles\": %.2f, \"welford_step_cycles\": %.2f}\n",
         (double)cyc[0] / n, (double)cyc[1] / n, (double)cyc[2] / n);
  return 0;
}
