// Nearest-neighbour distances for the reconstruction metrics
// (reference metrics.py:48-80: cKDTree(reference).query(samples, k=1) and the
// reverse; SURVEY.md §8f row 3 "GPU Chamfer / F-score").
//
// B200 design: instead of a k-d tree, the tree points are counting-sorted
// into a uniform grid (about four cells per point, SoA coordinates so a
// grid row is one contiguous run) and every query walks Chebyshev rings of
// cells outward from its own until no unseen cell can hold a closer point.
// Queries are processed in cell order, so the threads of a warp read the
// same runs.  Distances are sqrt((dx*dx + dy*dy) + dz*dz) in FP64 with no
// contraction -- the brute-force / cKDTree value bit for bit -- and the
// minimum over candidates does not depend on visiting order, so the
// distances are exact; the means and threshold fractions are then taken on
// the host with the reference's own numpy expressions.
#include <cub/cub.cuh>
#include <math_constants.h>

#include <algorithm>
#include <cmath>
#include <cstring>

#include "../../include/tsdf_b200.h"
#include "fusion.h"

namespace {
using tsdf::cuda_status;
using tsdf::set_error;

constexpr int kThreads = 256;
constexpr int64_t kMaxCells = 1ll << 26;

// order-preserving map of doubles to u64 (for atomicMin / atomicMax)
__host__ __device__ inline unsigned long long ord_key(double x) {
#ifdef __CUDA_ARCH__
  const unsigned long long b = (unsigned long long)__double_as_longlong(x);
#else
  unsigned long long b;
  memcpy(&b, &x, 8);
#endif
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}
inline double from_key(unsigned long long k) {
  const unsigned long long b = (k >> 63) ? (k & 0x7FFFFFFFFFFFFFFFull) : ~k;
  double x;
  memcpy(&x, &b, 8);
  return x;
}

__global__ void k_bbox(const double* __restrict__ p, int64_t n, unsigned long long* lohi,
                       unsigned int* bad) {
  unsigned long long lo[3] = {~0ull, ~0ull, ~0ull}, hi[3] = {0, 0, 0};
  unsigned int nonfinite = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
#pragma unroll
    for (int a = 0; a < 3; a++) {
      const double v = p[3 * i + a];
      nonfinite |= !isfinite(v);
      const unsigned long long k = ord_key(v);
      lo[a] = min(lo[a], k);
      hi[a] = max(hi[a], k);
    }
  }
#pragma unroll
  for (int a = 0; a < 3; a++)
    for (int o = 16; o; o >>= 1) {
      lo[a] = min(lo[a], __shfl_xor_sync(0xffffffffu, lo[a], o));
      hi[a] = max(hi[a], __shfl_xor_sync(0xffffffffu, hi[a], o));
    }
  nonfinite = __any_sync(0xffffffffu, nonfinite);
  if ((threadIdx.x & 31) == 0) {
#pragma unroll
    for (int a = 0; a < 3; a++) {
      atomicMin(&lohi[a], lo[a]);
      atomicMax(&lohi[3 + a], hi[a]);
    }
    if (nonfinite) atomicOr(bad, 1u);
  }
}

struct Grid {
  double o[3], h;
  int64_t g[3];
};

__device__ inline int64_t cell_axis(double v, double o, double h) {
  const double c = floor((v - o) / h);
  return (int64_t)fmin(fmax(c, -1e15), 1e15);
}

__device__ inline uint32_t cell_index(const Grid& G, const int64_t* c) {
  return (uint32_t)((c[2] * G.g[1] + c[1]) * G.g[0] + c[0]);
}

__device__ inline void clamp_cell(const Grid& G, int64_t* c) {
#pragma unroll
  for (int a = 0; a < 3; a++) c[a] = min(max(c[a], (int64_t)0), G.g[a] - 1);
}

// per tree point: its cell and its rank within the cell
__global__ void k_count(const double* __restrict__ p, int64_t n, Grid G, uint32_t* cnt,
                        uint32_t* cell, uint32_t* rank) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t c[3];
#pragma unroll
  for (int a = 0; a < 3; a++) c[a] = cell_axis(p[3 * i + a], G.o[a], G.h);
  clamp_cell(G, c);  // only rounding at the top face can step outside
  const uint32_t id = cell_index(G, c);
  cell[i] = id;
  rank[i] = atomicAdd(&cnt[id], 1u);
}

__global__ void k_scatter(const double* __restrict__ p, int64_t n, const uint32_t* __restrict__ start,
                          const uint32_t* __restrict__ cell, const uint32_t* __restrict__ rank,
                          double* sx, double* sy, double* sz) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const uint32_t pos = start[cell[i]] + rank[i];
  sx[pos] = p[3 * i];
  sy[pos] = p[3 * i + 1];
  sz[pos] = p[3 * i + 2];
}

__global__ void k_query_keys(const double* __restrict__ q, int64_t n, Grid G, uint32_t* key,
                             uint32_t* idx) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  int64_t c[3];
#pragma unroll
  for (int a = 0; a < 3; a++) c[a] = cell_axis(q[3 * i + a], G.o[a], G.h);
  clamp_cell(G, c);
  key[i] = cell_index(G, c);
  idx[i] = (uint32_t)i;
}

__device__ inline double d2(double x, double y, double z, double px, double py, double pz) {
  const double dx = __dsub_rn(x, px), dy = __dsub_rn(y, py), dz = __dsub_rn(z, pz);
  return __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
}

__device__ inline void scan_run(uint32_t b, uint32_t e, const double* __restrict__ sx,
                                const double* __restrict__ sy, const double* __restrict__ sz,
                                double x, double y, double z, double& best) {
  for (uint32_t j = b; j < e; j++) best = fmin(best, d2(x, y, z, sx[j], sy[j], sz[j]));
}

// Chebyshev ring search.  A tree point in a cell k >= 1 cells away (per
// axis) from the query's cell lies more than (k - 1) h + (the query's gap
// to its own cell face) away, so after rings 0..r every unseen point is at
// least r h + gap away; the slack absorbs the rounding of the cell
// assignment.
__global__ void __launch_bounds__(kThreads) k_nn(const double* __restrict__ q,
                                                 const uint32_t* __restrict__ order, int64_t n,
                                                 Grid G, const uint32_t* __restrict__ start,
                                                 const double* __restrict__ sx,
                                                 const double* __restrict__ sy,
                                                 const double* __restrict__ sz, double* out) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= n) return;
  const uint32_t qi = order[t];
  const double x = q[3 * qi], y = q[3 * qi + 1], z = q[3 * qi + 2];
  if (!isfinite(x) || !isfinite(y) || !isfinite(z)) {
    out[qi] = CUDART_NAN;
    return;
  }
  const double v[3] = {x, y, z};
  int64_t c[3];
  double gap = CUDART_INF;
  int64_t r0 = 0, rmax = 0;
#pragma unroll
  for (int a = 0; a < 3; a++) {
    c[a] = cell_axis(v[a], G.o[a], G.h);
    const double f0 = G.o[a] + (double)c[a] * G.h;
    gap = fmin(gap, fmin(v[a] - f0, f0 + G.h - v[a]));
    r0 = max(r0, max(-c[a], c[a] - (G.g[a] - 1)));
    rmax = max(rmax, max(c[a], G.g[a] - 1 - c[a]));
  }
  const double slack = 1e-6 * G.h + 1e-13 * (fabs(x) + fabs(y) + fabs(z));
  gap = fmax(0.0, gap) - slack;
  double best = CUDART_INF;
  for (int64_t r = r0;; r++) {
    const int64_t z0 = max(c[2] - r, (int64_t)0), z1 = min(c[2] + r, G.g[2] - 1);
    const int64_t y0 = max(c[1] - r, (int64_t)0), y1 = min(c[1] + r, G.g[1] - 1);
    const int64_t x0 = max(c[0] - r, (int64_t)0), x1 = min(c[0] + r, G.g[0] - 1);
    for (int64_t zz = z0; zz <= z1; zz++) {
      const bool zface = (zz - c[2] == r) || (c[2] - zz == r);
      for (int64_t yy = y0; yy <= y1; yy++) {
        const int64_t row = (zz * G.g[1] + yy) * G.g[0];
        if (zface || yy - c[1] == r || c[1] - yy == r) {
          if (x0 <= x1) scan_run(start[row + x0], start[row + x1 + 1], sx, sy, sz, x, y, z, best);
        } else {
          const int64_t xa = c[0] - r, xb = c[0] + r;
          if (xa >= 0 && xa < G.g[0]) scan_run(start[row + xa], start[row + xa + 1], sx, sy, sz, x, y, z, best);
          if (r > 0 && xb >= 0 && xb < G.g[0])
            scan_run(start[row + xb], start[row + xb + 1], sx, sy, sz, x, y, z, best);
        }
      }
    }
    const double bound = (double)r * G.h + gap;
    if (r >= rmax || (bound > 0 && best <= bound * bound)) break;
  }
  out[qi] = sqrt(best);
}

struct Scratch {
  cudaStream_t s;
  std::vector<void*> p;
  ~Scratch() {
    for (void* x : p) cudaFreeAsync(x, s);
  }
  template <class T>
  T* get(size_t n) {
    void* x = nullptr;
    if (cudaMallocAsync(&x, std::max<size_t>(n, 1) * sizeof(T), s) != cudaSuccess) return nullptr;
    p.push_back(x);
    return (T*)x;
  }
};

double cells_for(const double* e, double h, int64_t* g) {
  double tot = 1;
  for (int a = 0; a < 3; a++) {
    const double ga = std::floor(e[a] / h) + 1;
    g[a] = (int64_t)std::min(ga, 1e12);
    tot *= ga;
  }
  return tot;
}

}  // namespace

// cell edge: the smallest h (binary search on a log scale) whose grid has
// at most ~4 cells per tree point
static Grid choose_grid(const double* lo, const double* hi, int64_t n) {
  Grid G;
  double e[3], emax = 0;
  for (int a = 0; a < 3; a++) {
    G.o[a] = lo[a];
    e[a] = hi[a] - lo[a];
    emax = std::max(emax, e[a]);
  }
  const int64_t target = std::min<int64_t>(std::max<int64_t>(4 * n, 1), kMaxCells);
  if (!(emax > 0)) {
    G.h = 1.0;
  } else {
    double a = std::log(emax / 1e7), b = std::log(emax) + 1e-9;  // cells(a) >= target >= cells(b)
    int64_t g[3];
    for (int it = 0; it < 60; it++) {
      const double m = 0.5 * (a + b);
      if (cells_for(e, std::exp(m), g) > (double)target) a = m;
      else b = m;
    }
    G.h = std::exp(b);
  }
  cells_for(e, G.h, G.g);
  return G;
}

extern "C" int tsdf_nn_distance(const double* tree, int64_t n_tree, const double* query,
                                int64_t n_query, int32_t mem, double* dist, void* cuda_stream) {
  if (n_tree <= 0 || n_query < 0 || n_tree >= (1ll << 31) || n_query >= (1ll << 31) ||
      (mem != TSDF_MEM_HOST && mem != TSDF_MEM_DEVICE) || !tree || (n_query && (!query || !dist))) {
    set_error("nn_distance: need a non-empty tree, sizes below 2^31, and valid buffers");
    return TSDF_EVALUE;
  }
  if (n_query == 0) return TSDF_OK;
  cudaStream_t s = (cudaStream_t)cuda_stream;
  Scratch S{s, {}};
  const double *dt = tree, *dq = query;
  double* dout = dist;
  if (mem == TSDF_MEM_HOST) {
    double* a = S.get<double>(3 * n_tree);
    double* b = S.get<double>(3 * n_query);
    dout = S.get<double>(n_query);
    if (!a || !b || !dout) {
      set_error("nn_distance: device allocation failed");
      return TSDF_ECUDA;
    }
    cudaMemcpyAsync(a, tree, 24 * n_tree, cudaMemcpyHostToDevice, s);
    cudaMemcpyAsync(b, query, 24 * n_query, cudaMemcpyHostToDevice, s);
    dt = a;
    dq = b;
  }
  unsigned long long* lohi = S.get<unsigned long long>(8);
  if (!lohi) {
    set_error("nn_distance: device allocation failed");
    return TSDF_ECUDA;
  }
  unsigned long long init[8] = {~0ull, ~0ull, ~0ull, 0, 0, 0, 0, 0};
  cudaMemcpyAsync(lohi, init, sizeof(init), cudaMemcpyHostToDevice, s);
  k_bbox<<<std::min<int64_t>((n_tree + kThreads - 1) / kThreads, 148 * 8), kThreads, 0, s>>>(
      dt, n_tree, lohi, (unsigned int*)(lohi + 6));
  unsigned long long h_lohi[8];
  cudaMemcpyAsync(h_lohi, lohi, sizeof(h_lohi), cudaMemcpyDeviceToHost, s);
  if (cudaError_t e = cudaStreamSynchronize(s)) return cuda_status(e, "nn_distance bbox");
  if ((unsigned int)h_lohi[6]) {
    set_error("nn_distance: non-finite tree coordinate");
    return TSDF_EVALUE;
  }
  double lo[3], hi[3];
  for (int a = 0; a < 3; a++) {
    lo[a] = from_key(h_lohi[a]);
    hi[a] = from_key(h_lohi[3 + a]);
  }
  const Grid G = choose_grid(lo, hi, n_tree);
  const int64_t ncell = G.g[0] * G.g[1] * G.g[2];
  uint32_t* cnt = S.get<uint32_t>(ncell + 1);
  uint32_t* start = S.get<uint32_t>(ncell + 1);
  uint32_t* cell = S.get<uint32_t>(n_tree);
  uint32_t* rank = S.get<uint32_t>(n_tree);
  double* sx = S.get<double>(n_tree);
  double* sy = S.get<double>(n_tree);
  double* sz = S.get<double>(n_tree);
  uint32_t* qkey = S.get<uint32_t>(n_query);
  uint32_t* qidx = S.get<uint32_t>(n_query);
  uint32_t* qkey2 = S.get<uint32_t>(n_query);
  uint32_t* order = S.get<uint32_t>(n_query);
  size_t scan_bytes = 0, sort_bytes = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, cnt, start, (int)(ncell + 1), s);
  int end_bit = 1;
  while (end_bit < 32 && (1ll << end_bit) < ncell) end_bit++;
  cub::DeviceRadixSort::SortPairs(nullptr, sort_bytes, qkey, qkey2, qidx, order, (int)n_query, 0,
                                  end_bit, s);
  void* tmp = S.get<char>(std::max(scan_bytes, sort_bytes));
  if (!cnt || !start || !cell || !rank || !sx || !sy || !sz || !qkey || !qidx || !qkey2 || !order ||
      !tmp) {
    set_error("nn_distance: device allocation failed");
    return TSDF_ECUDA;
  }
  cudaMemsetAsync(cnt, 0, sizeof(uint32_t) * (ncell + 1), s);
  const int bt = (int)((n_tree + kThreads - 1) / kThreads), bq = (int)((n_query + kThreads - 1) / kThreads);
  k_count<<<bt, kThreads, 0, s>>>(dt, n_tree, G, cnt, cell, rank);
  cub::DeviceScan::ExclusiveSum(tmp, scan_bytes, cnt, start, (int)(ncell + 1), s);
  k_scatter<<<bt, kThreads, 0, s>>>(dt, n_tree, start, cell, rank, sx, sy, sz);
  k_query_keys<<<bq, kThreads, 0, s>>>(dq, n_query, G, qkey, qidx);
  cub::DeviceRadixSort::SortPairs(tmp, sort_bytes, qkey, qkey2, qidx, order, (int)n_query, 0,
                                  end_bit, s);
  k_nn<<<bq, kThreads, 0, s>>>(dq, order, n_query, G, start, sx, sy, sz, dout);
  if (mem == TSDF_MEM_HOST) cudaMemcpyAsync(dist, dout, 8 * n_query, cudaMemcpyDeviceToHost, s);
  if (cudaError_t e = cudaStreamSynchronize(s)) return cuda_status(e, "nn_distance");
  return TSDF_OK;
}
