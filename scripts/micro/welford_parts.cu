// Which part of a Welford step costs: the TSDF chain alone, + variance,
// + the reciprocal of W + 1, one warp, cycles per step.
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ double div_by_int(double x, double n, double y) {
  const double q0 = x * y;
  const double r = __fma_rn(-q0, n, x);
  return __fma_rn(r, y, q0);
}

__device__ __forceinline__ double rcp_rn_nobranch(double n) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(n));
  double e = __fma_rn(-n, y, 1.0);
  y = __fma_rn(y, e, y);
  e = __fma_rn(-n, y, 1.0);
  y = __fma_rn(y, e, y);
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

template <int kMode>
__global__ void k_part(double* out, long long* cyc, int n, double a, double b) {
  double D = a, S = 0, W = 1.0, y = 0.5;
  long long t0 = clock64();
  for (int i = 0; i < n; i++) {
    const double sdf = b * (double)(i & 7);
    const double w_old = W, d_old = D, n1 = w_old + 1.0;
    if (kMode == 2) y = __drcp_rn(n1);
    if (kMode == 3) y = rcp_rn_nobranch(n1);
    if (kMode == 4) y = __drcp_rn(n1 + 1.0);  // next step's (as the kernel does)
    if (kMode == 5) y = rcp_rn_nobranch(n1 + 1.0);
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

// the reciprocal software-pipelined over four steps: each step advances the
// in-flight reciprocals of steps k+1..k+4 by one stage (two dependent FP64
// operations), so no step waits on a whole reciprocal chain
__global__ void k_pipe(double* out, long long* cyc, int n, double a, double b) {
  double D = a, S = 0, W = 1.0;
  // in flight: stage-1 values for n4 (step k+4), stage-2 for n3, stage-3 for n2; y1 ready for step k+1
  double y_cur = __drcp_rn(W + 1.0);
  double n2 = W + 3.0, n3 = W + 4.0, n4 = W + 5.0;
  double y2_pre = __drcp_rn(W + 2.0);  // step k+1's value, complete
  double a3, e3, a4, e4, b2, r2l, r2h, r20, l2, h2;
  // prime: stage values for n2 (needs S3), n3 (needs S2), n4 (needs S1)
  {
    double y0 = 0;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y0) : "d"(n2));
    double e = __fma_rn(-n2, y0, 1.0);
    y0 = __fma_rn(y0, e, y0);
    e = __fma_rn(-n2, y0, 1.0);
    b2 = __fma_rn(y0, e, y0);
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(a3) : "d"(n3));
    e3 = __fma_rn(-n3, a3, 1.0);
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(a4) : "d"(n4));
    e4 = 0;
  }
  long long t0 = clock64();
  for (int i = 0; i < n; i++) {
    const double sdf = b * (double)(i & 7);
    const double w_old = W, d_old = D, n1 = w_old + 1.0;
    const double t1 = w_old * d_old;
    // stage 4 of n2: pick the correctly rounded neighbour of b2
    l2 = __longlong_as_double(__double_as_longlong(b2) - 1);
    h2 = __longlong_as_double(__double_as_longlong(b2) + 1);
    r20 = fabs(__fma_rn(-n2, b2, 1.0));
    r2l = fabs(__fma_rn(-n2, l2, 1.0));
    r2h = fabs(__fma_rn(-n2, h2, 1.0));
    const double num = t1 + sdf;
    // stage 3 of n3: second Newton step
    double y3 = __fma_rn(a3, e3, a3);
    double e3b = __fma_rn(-n3, y3, 1.0);
    const double q0 = num * y_cur;
    // stage 2 of n4: first Newton step
    e4 = __fma_rn(-n4, a4, 1.0);
    const double r = __fma_rn(-q0, n1, num);
    double best = r2l < r20 ? l2 : b2;
    const double rb = r2l < r20 ? r2l : r20;
    best = r2h < rb ? h2 : best;
    const double d_new = __fma_rn(r, y_cur, q0);
    S = S + (sdf - d_old) * (sdf - d_new);
    D = d_new;
    W = n1;
    // rotate: y for the next step, pipeline shifts by one
    y_cur = y2_pre;
    y2_pre = best;
    n2 = n3; b2 = __fma_rn(y3, e3b, y3);
    n3 = n4; a3 = __fma_rn(a4, e4, a4); e3 = __fma_rn(-n3, a3, 1.0);
    n4 = n4 + 1.0;
    asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(a4) : "d"(n4));
  }
  long long t1 = clock64();
  out[threadIdx.x] = D + S + y_cur;
  if (threadIdx.x == 0) cyc[6] = t1 - t0;
}

// reciprocals from a precomputed RN(1/n) table, loaded eight steps ahead
// into a register ring
__global__ void k_table(const double* __restrict__ tab, double* out, long long* cyc, int n, double a,
                        double b) {
  double D = a, S = 0, W = 1.0;
  double y0 = tab[2], y1 = tab[3], y2 = tab[4], y3 = tab[5], y4 = tab[6], y5 = tab[7], y6 = tab[8],
         y7 = tab[9];
  long long t0 = clock64();
  for (int i = 0; i < n; i++) {
    const double sdf = b * (double)(i & 7);
    const double w_old = W, d_old = D, n1 = w_old + 1.0;
    const double yl = __ldg(&tab[(int)n1 + 8]);
    const double num = w_old * d_old + sdf;
    const double d_new = div_by_int(num, n1, y0);
    S = S + (sdf - d_old) * (sdf - d_new);
    D = d_new;
    W = n1;
    y0 = y1; y1 = y2; y2 = y3; y3 = y4; y4 = y5; y5 = y6; y6 = y7; y7 = yl;
  }
  long long t1 = clock64();
  out[threadIdx.x] = D + S;
  if (threadIdx.x == 0) cyc[7] = t1 - t0;
}

__global__ void k_fill(double* tab, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    tab[i] = i ? __drcp_rn((double)i) : 0.0;
}

int main() {
  double* out;
  long long* cyc;
  cudaMalloc(&out, 256);
  cudaMallocManaged(&cyc, 64);
  double* tab;
  cudaMalloc(&tab, (1 << 20) * 8);
  k_fill<<<148, 256>>>(tab, 1 << 20);
  const int n = 100000;
  for (int rep = 0; rep < 2; rep++) {
    k_part<0><<<1, 32>>>(out, cyc, n, 1.0000001, 0.9999999);
    k_part<1><<<1, 32>>>(out, cyc, n, 1.0000001, 0.9999999);
    k_part<2><<<1, 32>>>(out, cyc, n, 1.0000001, 0.9999999);
    k_part<3><<<1, 32>>>(out, cyc, n, 1.0000001, 0.9999999);
    k_part<4><<<1, 32>>>(out, cyc, n, 1.0000001, 0.9999999);
    k_part<5><<<1, 32>>>(out, cyc, n, 1.0000001, 0.9999999);
    k_pipe<<<1, 32>>>(out, cyc, n, 1.0000001, 0.9999999);
    k_table<<<1, 32>>>(tab, out, cyc, n, 1.0000001, 0.9999999);
    cudaDeviceSynchronize();
  }
  printf("{\"tsdf_chain\": %.1f, \"plus_variance\": %.1f, \"plus_drcp\": %.1f, \"plus_branchfree_rcp\": %.1f, "
         "\"plus_drcp_next\": %.1f, \"plus_branchfree_next\": %.1f, \"pipelined_rcp\": %.1f, \"table_ring\": %.1f}\n", (double)cyc[0] / n, (double)cyc[1] / n,
         (double)cyc[2] / n, (double)cyc[3] / n, (double)cyc[4] / n, (double)cyc[5] / n, (double)cyc[6] / n, (double)cyc[7] / n);
  return 0;
}
