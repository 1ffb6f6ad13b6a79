// Branch-free RN(1/n) for the Welford weights (k_lidar_hot_apply): MUFU seed,
// two Newton steps, then the correctly rounded value picked among the three
// neighbouring doubles by exact FMA residuals.  Checks it against __drcp_rn
// for every integer n in [1, 2^24] and times the Welford step with it.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double rcp_rn_nobranch(double n) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(n));
  double e = __fma_rn(-n, y, 1.0);
  y = __fma_rn(y, e, y);
  e = __fma_rn(-n, y, 1.0);
  y = __fma_rn(y, e, y);
  // y is within an ulp of 1/n: keep the neighbour with the smallest exact residual
  const double lo = __longlong_as_double(__double_as_longlong(y) - 1);
  const double hi = __longlong_as_double(__double_as_longlong(y) + 1);
  const double r0 = fabs(__fma_rn(-n, y, 1.0)), rl = fabs(__fma_rn(-n, lo, 1.0)),
               rh = fabs(__fma_rn(-n, hi, 1.0));
  double best = y, rb = r0;
  best = rl < rb ? lo : best;
  rb = rl < rb ? rl : rb;
  best = rh < rb ? hi : best;
  return best;
}

__device__ __forceinline__ double div_by_int(double x, double n, double y) {
  const double q0 = x * y;
  const double r = __fma_rn(-q0, n, x);
  return __fma_rn(r, y, q0);
}

__global__ void k_check(long long n_max, unsigned long long* bad) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x + 1; i <= n_max;
       i += (long long)gridDim.x * blockDim.x) {
    const double n = (double)i;
    if (rcp_rn_nobranch(n) != __drcp_rn(n)) atomicAdd(bad, 1ull);
  }
}

__global__ void k_step(double* out, long long* cyc, int n, double a, double b) {
  double D = a, S = 0, W = 1.0, yn = rcp_rn_nobranch(W + 1.0);
  long long t0 = clock64();
  for (int i = 0; i < n; i++) {
    const double sdf = b * (double)(i & 7);
    const double w_old = W, d_old = D, n1 = w_old + 1.0, y1 = yn;
    yn = rcp_rn_nobranch(n1 + 1.0);  // next step's reciprocal, off the TSDF chain
    const double num = w_old * d_old + sdf;
    const double d_new = div_by_int(num, n1, y1);
    S = S + (sdf - d_old) * (sdf - d_new);
    D = d_new;
    W = n1;
  }
  long long t1 = clock64();
  out[threadIdx.x] = D + S;
  if (threadIdx.x == 0) cyc[0] = t1 - t0;
}

// the same chain with the variance term applied one step late and the
// reciprocal computed two steps ahead: every instruction between the five
// dependent TSDF operations is independent of them
__global__ void k_step2(double* out, long long* cyc, int n, double a, double b) {
  double D = a, S = 0, W = 1.0;
  double y1 = rcp_rn_nobranch(W + 1.0), y2 = rcp_rn_nobranch(W + 2.0);
  double sp = 0, dop = 0, dnp = 0;
  long long t0 = clock64();
#pragma unroll 2
  for (int i = 0; i < n; i++) {
    const double sdf = b * (double)(i & 7);
    const double n1 = W + 1.0;
    const double t1 = W * D;
    S = S + (sp - dop) * (sp - dnp);
    const double y3 = rcp_rn_nobranch(n1 + 2.0);
    const double num = t1 + sdf;
    const double q0 = num * y1;
    const double r = __fma_rn(-q0, n1, num);
    const double d_new = __fma_rn(r, y1, q0);
    sp = sdf;
    dop = D;
    dnp = d_new;
    D = d_new;
    W = n1;
    y1 = y2;
    y2 = y3;
  }
  S = S + (sp - dop) * (sp - dnp);
  long long t1 = clock64();
  out[threadIdx.x] = D + S;
  if (threadIdx.x == 0) cyc[1] = t1 - t0;
}

// reciprocals for the next four steps computed together (four independent
// chains the scheduler interleaves), then four dependent TSDF steps
__global__ void k_step4(double* out, long long* cyc, int n, double a, double b) {
  double D = a, S = 0, W = 1.0;
  long long t0 = clock64();
  for (int i = 0; i < n; i += 4) {
    double y[4];
#pragma unroll
    for (int j = 0; j < 4; j++) y[j] = rcp_rn_nobranch(W + (double)(j + 1));
#pragma unroll
    for (int j = 0; j < 4; j++) {
      const double sdf = b * (double)((i + j) & 7);
      const double w_old = W, d_old = D, n1 = w_old + 1.0;
      const double num = w_old * d_old + sdf;
      const double d_new = div_by_int(num, n1, y[j]);
      S = S + (sdf - d_old) * (sdf - d_new);
      D = d_new;
      W = n1;
    }
  }
  long long t1 = clock64();
  out[threadIdx.x] = D + S;
  if (threadIdx.x == 0) cyc[2] = t1 - t0;
}

int main() {
  unsigned long long* bad;
  long long* cyc;
  double* out;
  cudaMallocManaged(&bad, 8);
  cudaMallocManaged(&cyc, 24);
  cudaMalloc(&out, 256);
  *bad = 0;
  const long long n_max = 1ll << 24;
  k_check<<<148 * 8, 256>>>(n_max, bad);
  cudaDeviceSynchronize();
  k_step<<<1, 32>>>(out, cyc, 100000, 1.0000001, 0.9999999);
  cudaDeviceSynchronize();
  k_step<<<1, 32>>>(out, cyc, 100000, 1.0000001, 0.9999999);
  k_step2<<<1, 32>>>(out, cyc, 100000, 1.0000001, 0.9999999);
  cudaDeviceSynchronize();
  k_step2<<<1, 32>>>(out, cyc, 100000, 1.0000001, 0.9999999);
  k_step4<<<1, 32>>>(out, cyc, 100000, 1.0000001, 0.9999999);
  cudaDeviceSynchronize();
  k_step4<<<1, 32>>>(out, cyc, 100000, 1.0000001, 0.9999999);
  cudaDeviceSynchronize();
  printf("{\"batch4_step_cycles\": %.2f}\n", (double)cyc[2] / 100000);
  printf("{\"n_checked\": %lld, \"mismatches\": %llu, \"welford_step_cycles\": %.2f, \"pipelined_step_cycles\": %.2f}\n",
         n_max, *bad, (double)cyc[0] / 100000, (double)cyc[1] / 100000);
  return 0;
}
