// Mixed-resolution Marching Cubes over the device-resident grid
// (reference meshing.py:94-552), bit-identical to the reference output.
//
// Stages (all on the device):
//   M1  per live block: observed tsdf range (w > 0)                 k_block_range
//   M2  27-neighbourhood range cull, per-level kept list            k_keep
//   M3  canonical order: radix sort of packed keys per level; 256-block
//       chunks as in the reference (meshing.py:457-459)
//   M4  pass A, one CTA per kept block: corner gather (cross-level
//       blend), gradients, cases -> cut-edge / triangle counts        k_mc<false>
//   M5  exclusive scans of the counts laid out in the reference's emission
//       order (level, chunk, axis, block) / (level, chunk, slot, block)
//   M6  pass B: the same CTA recomputes and writes vertices + triangles  k_mc<true>
//   M7  exact vertex dedup: stable LSD radix sort on (x, y, z) f64 keys,
//       merged normals summed in emission order, winding fix, then the
//       epsilon-bucket collapse (same sort on int64 cells) and compaction.
#include <cub/cub.cuh>
#include <math_constants.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "fusion.h"
#include "mc_tables.h"

namespace tsdf {

#define MCK(x)                                  \
  do {                                          \
    int _s = cuda_status((x), #x);              \
    if (_s) return _s;                          \
  } while (0)

__constant__ int8_t c_corner[8][3];
__constant__ int8_t c_edge_loc[12][4];
__constant__ uint16_t c_edge_table[256];
__constant__ int8_t c_tri_table[256][16];

static bool g_tables_loaded = false;
static int load_tables() {
  if (g_tables_loaded) return kOk;
  MCK(cudaMemcpyToSymbol(c_corner, MC_CORNER, sizeof(MC_CORNER)));
  MCK(cudaMemcpyToSymbol(c_edge_loc, MC_EDGE_LOC, sizeof(MC_EDGE_LOC)));
  MCK(cudaMemcpyToSymbol(c_edge_table, MC_EDGE_TABLE, sizeof(MC_EDGE_TABLE)));
  MCK(cudaMemcpyToSymbol(c_tri_table, MC_TRI_TABLE, sizeof(MC_TRI_TABLE)));
  g_tables_loaded = true;
  return kOk;
}

// scratch buffers owned by one extraction call
// per-call device scratch from the stream-ordered pool: after the first
// extraction the pool keeps the memory, so later calls allocate for free
struct DevBuf {
  std::vector<void*> ptrs;
  cudaStream_t stream = nullptr;
  static void keep_pool() {
    static bool done = false;
    if (done) return;
    int dev = 0;
    cudaMemPool_t pool;
    if (cudaGetDevice(&dev) == cudaSuccess && cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
      uint64_t keep = ~0ull;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
    done = true;
  }
  ~DevBuf() {
    for (void* p : ptrs) cudaFreeAsync(p, stream);
  }
  template <class T>
  T* get(size_t n) {
    keep_pool();
    void* p = nullptr;
    if (cudaMallocAsync(&p, std::max<size_t>(n, 1) * sizeof(T), stream) != cudaSuccess) return nullptr;
    ptrs.push_back(p);
    return (T*)p;
  }
};

// ---------------------------------------------------------------------------
// M1 / M2
// ---------------------------------------------------------------------------

// observed tsdf range of every live block (meshing.py:428-438); one warp per slot
__global__ void k_block_range(DevTable t, uint8_t* obs, double* rlo, double* rhi) {
  const int lane = threadIdx.x & 31;
  uint64_t warp = (blockIdx.x * (uint64_t)blockDim.x + threadIdx.x) >> 5;
  uint64_t nw = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  for (uint64_t s = warp; s <= t.mask; s += nw) {
    uint64_t k = t.keys[s];
    uint32_t v = t.vals[s];
    bool live = key_live(k) && v != kPending;
    if (!live) {
      if (lane == 0) obs[s] = 0;
      continue;
    }
    const DevHeap& h = t.heap[val_level(v)];
    int64_t base = (int64_t)val_handle(v) * h.nvox;
    double lo = CUDART_INF_F, hi = -CUDART_INF_F;
    bool any = false;
    for (int i = lane; i < h.nvox; i += 32) {
      if (h.weight[base + i] > 0.0f) {
        double d = h.tsdf[base + i];
        lo = fmin(lo, d);
        hi = fmax(hi, d);
        any = true;
      }
    }
    for (int o = 16; o; o >>= 1) {
      lo = fmin(lo, __shfl_xor_sync(0xffffffffu, lo, o));
      hi = fmax(hi, __shfl_xor_sync(0xffffffffu, hi, o));
    }
    any = __any_sync(0xffffffffu, any);
    if (lane == 0) {
      obs[s] = any;
      rlo[s] = lo;
      rhi[s] = hi;
    }
  }
}

// 27-neighbourhood straddle test (meshing.py:440-456); appends kept blocks
// per level as (packed key, slot)
__global__ void k_keep(DevTable t, const uint8_t* obs, const double* rlo, const double* rhi,
                       double iso, uint64_t* keys_out, uint32_t* slots_out, uint64_t cap_per_level,
                       unsigned long long* counts) {
  for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s <= t.mask;
       s += (uint64_t)gridDim.x * blockDim.x) {
    if (!obs[s]) continue;
    uint64_t key = t.keys[s];
    int64_t c[3];
    unpack_key(key, c);
    double lo = CUDART_INF, hi = -CUDART_INF;
    for (int q = 0; q < 27; q++) {
      int64_t n0 = c[0] + q / 9 - 1, n1 = c[1] + (q / 3) % 3 - 1, n2 = c[2] + q % 3 - 1;
      if (!key_in_range(n0, n1, n2)) continue;
      int64_t ns = table_find(t, pack_key(n0, n1, n2));
      if (ns < 0 || !obs[ns]) continue;
      lo = fmin(lo, rlo[ns]);
      hi = fmax(hi, rhi[ns]);
    }
    if (lo <= iso && iso <= hi) {
      int level = val_level(t.vals[s]);
      unsigned long long i = atomicAdd(&counts[level], 1ull);
      keys_out[level * cap_per_level + i] = key;
      slots_out[level * cap_per_level + i] = (uint32_t)s;
    }
  }
}

// ---------------------------------------------------------------------------
// M4 / M6: per-block Marching Cubes (meshing.py:94-158, 252-409)
// ---------------------------------------------------------------------------

constexpr int kMcThreads = 256;
constexpr int kMaxN1 = 9;
constexpr int kMaxCorners = kMaxN1 * kMaxN1 * kMaxN1;  // 729

struct NbInfo {
  int32_t found, level;
  int64_t handle;
};

struct McSmem {
  NbInfo nb[27];
  double axes[3][kMaxN1];
  double val[kMaxCorners];
  double col[kMaxCorners][3];
  double grad[kMaxCorners][3];
  uint8_t valid[kMaxCorners];
  uint8_t cases[512];
  int16_t erank[3][kMaxN1 * kMaxN1 * (kMaxN1 - 1)];  // rank of each cut edge (pass B)
};

struct McArgs {
  DevTable t;
  const uint32_t* slots;     // kept blocks, canonical order, levels concatenated
  const int32_t* blk_level;  // level of each kept block
  const int64_t* chunk_of;   // global chunk id of each kept block
  const int64_t* chunk_start;
  const int32_t* chunk_size;
  uint64_t n_blocks;
  double iso;
  // pass A outputs
  int32_t* edge_cnt;  // [n_blocks][3]
  int32_t* tri_cnt;   // [n_blocks][5]
  uint8_t* emit_any;  // [n_blocks]
  // pass B inputs / outputs
  const uint8_t* chunk_emits;
  const int64_t* voff;  // exclusive scan over (chunk, axis, block) sequence
  const int64_t* toff;  // exclusive scan over (chunk, slot, block) sequence
  double* vpos;         // raw vertices, half units, 3 per row
  double* vnrm;
  double* vcol;
  int64_t* tri;  // raw vertex ids, 3 per row
};

__device__ inline double pw8(const double* a) {
  return ((a[0] + a[1]) + (a[2] + a[3])) + ((a[4] + a[5]) + (a[6] + a[7]));
}

__device__ inline int64_t floordiv16(int64_t a) { return a >= 0 ? a / 16 : -((15 - a) / 16); }

// corner blend of the up-to-8 octant voxels meeting lattice point h
// (block-local half units) -- _gather, meshing.py:94-158
__device__ void gather_corner(const DevTable& t, const NbInfo* nb, const int64_t* c,
                              const int64_t* h, double* value, uint8_t* valid, double* color) {
  double w[8], sdf[8], col[8][3];
  int64_t key[8];
#pragma unroll
  for (int o = 0; o < 8; o++) {
    const int so[3] = {(o >> 2 & 1) ? 1 : -1, (o >> 1 & 1) ? 1 : -1, (o & 1) ? 1 : -1};
    int64_t off[3], local[3], v3[3];
#pragma unroll
    for (int a = 0; a < 3; a++) {
      int64_t probe = h[a] + so[a];
      off[a] = floordiv16(probe);
      local[a] = probe - off[a] * 16;
    }
    const NbInfo& e = nb[((off[0] + 1) * 3 + (off[1] + 1)) * 3 + (off[2] + 1)];
    int lvl = e.found ? e.level : 0;
    int64_t csize = (int64_t)2 << lvl, side = 16 / csize;
#pragma unroll
    for (int a = 0; a < 3; a++) v3[a] = local[a] / csize;
    double wob = 0.0;
    sdf[o] = 0.0;
    col[o][0] = col[o][1] = col[o][2] = 0.0;
    if (e.found) {
      uint64_t g0 = (uint64_t)((c[0] + off[0]) * side + v3[0] + (1 << 19));
      uint64_t g1 = (uint64_t)((c[1] + off[1]) * side + v3[1] + (1 << 19));
      uint64_t g2 = (uint64_t)((c[2] + off[2]) * side + v3[2] + (1 << 19));
      key[o] = (int64_t)(((uint64_t)lvl << 60) | (g0 << 40) | (g1 << 20) | g2);
      const DevHeap& hp = t.heap[lvl];
      int64_t flat = e.handle * hp.nvox + (v3[0] * side + v3[1]) * side + v3[2];
      size_t plane = (size_t)hp.cap * hp.nvox;
      sdf[o] = hp.tsdf[flat];
      wob = (double)hp.weight[flat];
      col[o][0] = (double)hp.color[flat];
      col[o][1] = (double)hp.color[plane + flat];
      col[o][2] = (double)hp.color[2 * plane + flat];
    } else {
      key[o] = -1;
    }
    bool dup = false;
    for (int i = 0; i < o; i++) dup |= key[o] == key[i];
    dup &= (bool)e.found;
    double m[3];
#pragma unroll
    for (int a = 0; a < 3; a++) {
      double center = (double)(off[a] * 16) + ((double)v3[a] + 0.5) * (double)csize;
      double x = 1.0 - fabs((double)h[a] - center) / (double)csize;
      m[a] = x > 0.0 ? x : 0.0;
    }
    double coeff = (m[0] * m[1]) * m[2];
    w[o] = (((coeff * (2.0 / (double)csize)) * (double)(wob > 0)) * (double)(e.found != 0)) *
           (double)(!dup);
  }
  double wsum = pw8(w);
  bool ok = wsum > 0;
  double denom = ok ? wsum : 1.0;
  double ws[8];
#pragma unroll
  for (int o = 0; o < 8; o++) ws[o] = w[o] * sdf[o];
  *value = ok ? pw8(ws) / denom : 0.0;
  *valid = ok;
#pragma unroll
  for (int k = 0; k < 3; k++) {
    double acc = 0.0;
#pragma unroll
    for (int o = 0; o < 8; o++) acc += w[o] * col[o][k];
    color[k] = acc / denom;
  }
}

template <bool kWrite>
__global__ void __launch_bounds__(kMcThreads, 2) k_mc(McArgs A) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  McSmem& S = *reinterpret_cast<McSmem*>(smem_raw);
  typedef cub::BlockScan<int32_t, kMcThreads> Scan;
  __shared__ typename Scan::TempStorage scan_tmp;
  __shared__ int32_t s_total;
  const int tid = threadIdx.x;
  for (uint64_t gb = blockIdx.x; gb < A.n_blocks; gb += gridDim.x) {
    if (kWrite && !A.chunk_emits[A.chunk_of[gb]]) continue;
    const uint32_t slot = A.slots[gb];
    const int level = A.blk_level[gb];
    const int side = kFineSide >> level, n1 = side + 1, n3 = n1 * n1 * n1;
    int64_t c[3];
    unpack_key(A.t.keys[slot], c);
    if (tid < 27) {
      int64_t n0 = c[0] + tid / 9 - 1, nn1 = c[1] + (tid / 3) % 3 - 1, n2 = c[2] + tid % 3 - 1;
      int64_t s = key_in_range(n0, nn1, n2) ? table_find(A.t, pack_key(n0, nn1, n2)) : -1;
      uint32_t v = s >= 0 ? A.t.vals[s] : kPending;
      bool f = s >= 0 && v != kPending;
      S.nb[tid].found = f;
      S.nb[tid].level = f ? val_level(v) : 0;
      S.nb[tid].handle = f ? (int64_t)val_handle(v) : -1;
    }
    __syncthreads();
    // corner planes with transition truncation (meshing.py:252-262, 312-321)
    if (tid < 3 * n1) {
      int a = tid / n1, i = tid % n1;
      double step = (double)(16 / side);
      double x = (double)i * step;
      if (level > 0) {
        const int lo_face[3] = {4, 10, 12}, hi_face[3] = {22, 16, 14};
        const NbInfo& L = S.nb[lo_face[a]];
        const NbInfo& H = S.nb[hi_face[a]];
        if (i == 0 && L.found && L.level < level) x += step / 2;
        if (i == side && H.found && H.level < level) x -= step / 2;
      }
      S.axes[a][i] = x;
    }
    __syncthreads();
    for (int ci = tid; ci < n3; ci += kMcThreads) {
      int i = ci / (n1 * n1), j = (ci / n1) % n1, k = ci % n1;
      int64_t h[3] = {(int64_t)S.axes[0][i], (int64_t)S.axes[1][j], (int64_t)S.axes[2][k]};
      gather_corner(A.t, S.nb, c, h, &S.val[ci], &S.valid[ci], S.col[ci]);
    }
    __syncthreads();
    // central differences (meshing.py:265-297)
    for (int ci = tid; ci < n3; ci += kMcThreads) {
      int idx[3] = {ci / (n1 * n1), (ci / n1) % n1, ci % n1};
      const int stride[3] = {n1 * n1, n1, 1};
#pragma unroll
      for (int a = 0; a < 3; a++) {
        int p = idx[a];
        int lo = p == 0 ? 0 : p - 1, hi = p == n1 - 1 ? p : p + 1;
        double num = S.val[ci + (hi - p) * stride[a]] - S.val[ci + (lo - p) * stride[a]];
        S.grad[ci][a] = num / (S.axes[a][hi] - S.axes[a][lo]);
      }
    }
    // cases
    const int ncell = side * side * side;
    int any = 0;
    for (int cell = tid; cell < ncell; cell += kMcThreads) {
      int i = cell / (side * side), j = (cell / side) % side, k = cell % side;
      int cs = 0;
      bool ok = true;
#pragma unroll
      for (int q = 0; q < 8; q++) {
        int ci = ((i + c_corner[q][0]) * n1 + (j + c_corner[q][1])) * n1 + (k + c_corner[q][2]);
        cs |= (S.val[ci] < A.iso) << q;
        ok &= S.valid[ci] != 0;
      }
      if (!ok) cs = 0;
      S.cases[cell] = (uint8_t)cs;
      any |= c_edge_table[cs] != 0;
    }
    any = __syncthreads_or(any);
    if (!kWrite && tid == 0) A.emit_any[gb] = (uint8_t)any;
    const int64_t G = A.chunk_of[gb];
    const int64_t cstart = A.chunk_start[G];
    const int32_t csize = A.chunk_size[G];
    const int64_t bi = (int64_t)gb - cstart;
    // cut edges per axis, C order over the axis-shaped grid
    for (int a = 0; a < 3; a++) {
      const int d0 = a == 0 ? side : n1, d1 = a == 1 ? side : n1, d2 = a == 2 ? side : n1;
      const int ne = d0 * d1 * d2;
      const int per = (ne + kMcThreads - 1) / kMcThreads;
      int32_t mine = 0;
      for (int e = tid * per; e < min(ne, (tid + 1) * per); e++) {
        int i = e / (d1 * d2), j = (e / d2) % d1, k = e % d2;
        int c0 = (i * n1 + j) * n1 + k;
        int c1 = ((i + (a == 0)) * n1 + (j + (a == 1))) * n1 + (k + (a == 2));
        mine += ((S.val[c0] < A.iso) != (S.val[c1] < A.iso)) && S.valid[c0] && S.valid[c1];
      }
      int32_t ex, tot;
      Scan(scan_tmp).ExclusiveSum(mine, ex, tot);
      __syncthreads();
      if (!kWrite) {
        if (tid == 0) A.edge_cnt[gb * 3 + a] = tot;
      } else {
        int64_t base = A.voff[3 * cstart + (int64_t)a * csize + bi] + ex;
        const double wh[3] = {(double)c[0] * 16.0, (double)c[1] * 16.0, (double)c[2] * 16.0};
        for (int e = tid * per; e < min(ne, (tid + 1) * per); e++) {
          int i = e / (d1 * d2), j = (e / d2) % d1, k = e % d2;
          int i1 = i + (a == 0), j1 = j + (a == 1), k1 = k + (a == 2);
          int c0 = (i * n1 + j) * n1 + k, c1 = (i1 * n1 + j1) * n1 + k1;
          bool cut = ((S.val[c0] < A.iso) != (S.val[c1] < A.iso)) && S.valid[c0] && S.valid[c1];
          S.erank[a][e] = (int16_t)(base - A.voff[3 * cstart + (int64_t)a * csize + bi]);
          if (!cut) continue;
          double tt = (A.iso - S.val[c0]) / (S.val[c1] - S.val[c0]);
          double p0[3] = {S.axes[0][i], S.axes[1][j], S.axes[2][k]};
          double p1[3] = {S.axes[0][i1], S.axes[1][j1], S.axes[2][k1]};
#pragma unroll
          for (int d = 0; d < 3; d++) {
            A.vpos[3 * base + d] = (p0[d] + tt * (p1[d] - p0[d])) + wh[d];
            A.vnrm[3 * base + d] = S.grad[c0][d] + tt * (S.grad[c1][d] - S.grad[c0][d]);
            A.vcol[3 * base + d] = S.col[c0][d] + tt * (S.col[c1][d] - S.col[c0][d]);
          }
          base++;
        }
      }
    }
    __syncthreads();
    // triangles: slot-major, then cells in (i, j, k) order (meshing.py:385-409)
    const int cper = (ncell + kMcThreads - 1) / kMcThreads;
    for (int k3 = 0; k3 < 5; k3++) {
      int32_t mine = 0;
      for (int cell = tid * cper; cell < min(ncell, (tid + 1) * cper); cell++) {
        int cs = S.cases[cell];
        mine += c_edge_table[cs] != 0 && c_tri_table[cs][3 * k3] >= 0;
      }
      int32_t ex, tot;
      Scan(scan_tmp).ExclusiveSum(mine, ex, tot);
      __syncthreads();
      if (!kWrite) {
        if (tid == 0) A.tri_cnt[gb * 5 + k3] = tot;
        continue;
      }
      int64_t base = A.toff[5 * cstart + (int64_t)k3 * csize + bi] + ex;
      for (int cell = tid * cper; cell < min(ncell, (tid + 1) * cper); cell++) {
        int cs = S.cases[cell];
        if (!(c_edge_table[cs] != 0 && c_tri_table[cs][3 * k3] >= 0)) continue;
        int ci = cell / (side * side), cj = (cell / side) % side, ck = cell % side;
        for (int sidx = 0; sidx < 3; sidx++) {
          int e = c_tri_table[cs][3 * k3 + sidx];
          int a = c_edge_loc[e][0];
          int ii = ci + c_edge_loc[e][1], jj = cj + c_edge_loc[e][2], kk = ck + c_edge_loc[e][3];
          // rank of this cut edge among the block's axis-a cut edges
          const int d1 = a == 1 ? side : n1, d2 = a == 2 ? side : n1;
          int rank = S.erank[a][(ii * d1 + jj) * d2 + kk];
          A.tri[3 * base + sidx] = A.voff[3 * cstart + (int64_t)a * csize + bi] + rank;
        }
        base++;
      }
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// M7: dedup, normals, winding, collapse
// ---------------------------------------------------------------------------

__device__ inline uint64_t f64_order_key(double x) {
  x = x + 0.0;  // -0.0 -> +0.0 so equal values sort together
  uint64_t b = (uint64_t)__double_as_longlong(x);
  return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__global__ void k_iota(uint64_t* v, uint64_t n) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    v[i] = i;
}

// keys for one LSD pass: component d of the row each index points to
__global__ void k_pos_keys(const double* pos, const uint64_t* idx, uint64_t n, int d, uint64_t* keys) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    keys[i] = f64_order_key(pos[3 * idx[i] + d]);
}
__global__ void k_cell_keys(const int64_t* cells, const uint64_t* idx, uint64_t n, int d,
                            uint64_t* keys) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    keys[i] = (uint64_t)cells[3 * idx[i] + d] ^ 0x8000000000000000ull;
}

// group-start flags over a sorted index list; rows equal iff all 3 comps equal
template <typename T>
__global__ void k_group_flags(const T* rows, const uint64_t* idx, uint64_t n, int64_t* flag) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    bool start = i == 0;
    if (!start) {
      const T* a = rows + 3 * idx[i];
      const T* b = rows + 3 * idx[i - 1];
      start = !(a[0] == b[0] && a[1] == b[1] && a[2] == b[2]);
    }
    flag[i] = start;
  }
}

// inclusive-scan ids -> inverse map and group starts
__global__ void k_group_assign(const uint64_t* idx, const int64_t* gid_incl, uint64_t n,
                               int64_t* inverse, int64_t* group_start) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    int64_t g = gid_incl[i] - 1;
    inverse[idx[i]] = g;
    if (i == 0 || gid_incl[i] != gid_incl[i - 1]) group_start[g] = (int64_t)i;
  }
}

__device__ inline double norm_rows3(double x, double y, double z) {
  return sqrt((x * x + y * y) + z * z);
}

// exact dedup outputs (meshing.py:468-479): first occurrence position/colour,
// normals summed in emission order then normalised
__global__ void k_dedup_out(const double* vpos, const double* vnrm, const double* vcol,
                            const uint64_t* idx, const int64_t* gstart, int64_t ng, uint64_t n,
                            double scale, double* v, double* nrm, double* col) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < ng;
       g += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = gstart[g], e = g + 1 < ng ? gstart[g + 1] : (int64_t)n;
    uint64_t first = idx[b];
    double s[3] = {0.0, 0.0, 0.0};
    for (int64_t i = b; i < e; i++)
      for (int k = 0; k < 3; k++) s[k] += vnrm[3 * idx[i] + k];
    double nr = norm_rows3(s[0], s[1], s[2]);
    for (int k = 0; k < 3; k++) {
      v[3 * g + k] = vpos[3 * first + k] * scale;
      double c = vcol[3 * first + k];
      col[3 * g + k] = c < 0.0 ? 0.0 : (c > 1.0 ? 1.0 : c);
      nrm[3 * g + k] = nr > 0 ? s[k] / nr : (k == 2 ? 1.0 : 0.0);
    }
  }
}

// triangles through the dedup map, then winding fix (meshing.py:490-499)
__global__ void k_orient(const int64_t* tri_raw, const int64_t* inverse, uint64_t nt,
                         const double* v, const double* nrm, int64_t* tri) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nt;
       i += (uint64_t)gridDim.x * blockDim.x) {
    int64_t a = inverse[tri_raw[3 * i]], b = inverse[tri_raw[3 * i + 1]], c = inverse[tri_raw[3 * i + 2]];
    double e1[3], e2[3], ref[3];
    for (int k = 0; k < 3; k++) {
      e1[k] = v[3 * b + k] - v[3 * a + k];
      e2[k] = v[3 * c + k] - v[3 * a + k];
      ref[k] = (nrm[3 * a + k] + nrm[3 * b + k]) + nrm[3 * c + k];
    }
    double g0 = e1[1] * e2[2] - e1[2] * e2[1];
    double g1 = e1[2] * e2[0] - e1[0] * e2[2];
    double g2 = e1[0] * e2[1] - e1[1] * e2[0];
    bool flip = ((g0 * ref[0] + g2 * ref[2]) + g1 * ref[1]) < 0;
    tri[3 * i] = flip ? c : a;
    tri[3 * i + 1] = b;
    tri[3 * i + 2] = flip ? a : c;
  }
}

__global__ void k_cells(const double* v, uint64_t n, double eps, int64_t* cells) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < 3 * n;
       i += (uint64_t)gridDim.x * blockDim.x)
    cells[i] = (int64_t)floor(v[i] / eps);
}

// collapse_vertices (meshing.py:502-545): centroid / normalised-normal / mean colour
// per bucket, members summed in vertex order; eps == 0 keeps first occurrences
__global__ void k_collapse_out(const double* v, const double* nrm, const double* col,
                               const uint64_t* idx, const int64_t* gstart, int64_t ng, uint64_t n,
                               int exact, double* ov, double* on, double* oc) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < ng;
       g += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = gstart[g], e = g + 1 < ng ? gstart[g + 1] : (int64_t)n;
    if (exact) {
      uint64_t f = idx[b];
      for (int k = 0; k < 3; k++) {
        ov[3 * g + k] = v[3 * f + k];
        on[3 * g + k] = nrm[3 * f + k];
        oc[3 * g + k] = col[3 * f + k];
      }
      continue;
    }
    double sv[3] = {0, 0, 0}, sn[3] = {0, 0, 0}, sc[3] = {0, 0, 0};
    for (int64_t i = b; i < e; i++) {
      uint64_t r = idx[i];
      for (int k = 0; k < 3; k++) {
        sv[k] += v[3 * r + k];
        sn[k] += nrm[3 * r + k];
        sc[k] += col[3 * r + k];
      }
    }
    double cnt = (double)(e - b);
    double nr = norm_rows3(sn[0], sn[1], sn[2]);
    double d = nr > 0 ? nr : 1.0;
    for (int k = 0; k < 3; k++) {
      ov[3 * g + k] = sv[k] / cnt;
      on[3 * g + k] = sn[k] / d;
      oc[3 * g + k] = sc[k] / cnt;
    }
  }
}

// remap triangles, drop repeated-index and sub-1e-12 m^2 ones, mark used vertices
__global__ void k_tri_filter(const int64_t* tri, const int64_t* inverse, uint64_t nt,
                             const double* v, int64_t* tri_out, int64_t* keep, uint8_t* used) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nt;
       i += (uint64_t)gridDim.x * blockDim.x) {
    int64_t a = inverse[tri[3 * i]], b = inverse[tri[3 * i + 1]], c = inverse[tri[3 * i + 2]];
    bool ok = a != b && b != c && a != c;
    if (ok) {
      double e1[3], e2[3];
      for (int k = 0; k < 3; k++) {
        e1[k] = v[3 * b + k] - v[3 * a + k];
        e2[k] = v[3 * c + k] - v[3 * a + k];
      }
      double x = e1[1] * e2[2] - e1[2] * e2[1];
      double y = e1[2] * e2[0] - e1[0] * e2[2];
      double z = e1[0] * e2[1] - e1[1] * e2[0];
      ok = 0.5 * norm_rows3(x, y, z) >= 1e-12;
    }
    keep[i] = ok;
    tri_out[3 * i] = a;
    tri_out[3 * i + 1] = b;
    tri_out[3 * i + 2] = c;
    if (ok) used[a] = used[b] = used[c] = 1;
  }
}

__global__ void k_u8_to_i64(const uint8_t* a, uint64_t n, int all, int64_t* out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x)
    out[i] = all ? 1 : a[i];
}

__global__ void k_compact_verts(const double* v, const double* n, const double* c,
                                const int64_t* used, const int64_t* remap, uint64_t nv, double* ov,
                                double* on, double* oc) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nv;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (!used[i]) continue;
    int64_t r = remap[i];
    for (int k = 0; k < 3; k++) {
      ov[3 * r + k] = v[3 * i + k];
      on[3 * r + k] = n[3 * i + k];
      oc[3 * r + k] = c[3 * i + k];
    }
  }
}

__global__ void k_compact_tris(const int64_t* tri, const int64_t* keep, const int64_t* pos,
                               const int64_t* remap, uint64_t nt, int64_t* out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nt;
       i += (uint64_t)gridDim.x * blockDim.x) {
    if (!keep[i]) continue;
    int64_t p = pos[i];
    for (int k = 0; k < 3; k++) out[3 * p + k] = remap[tri[3 * i + k]];
  }
}

// ---------------------------------------------------------------------------
// chunk bookkeeping on the device (was a host loop over every kept block):
// the blocks of level l occupy [loff[l], loff[l] + n[l]) in canonical order,
// cut into chunks of 256 numbered from cbase[l]
struct ChunkMeta {
  int64_t loff[kMaxLevels + 1], cbase[kMaxLevels];
  int n_levels;
};
__global__ void k_chunk_meta(ChunkMeta M, uint64_t nb, int64_t* chunk_of, int32_t* blevel,
                             int64_t* chunk_start, int32_t* chunk_size) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nb;
       i += (uint64_t)gridDim.x * blockDim.x) {
    int l = 0;
    while (l + 1 < M.n_levels && (int64_t)i >= M.loff[l + 1]) l++;
    const int64_t li = (int64_t)i - M.loff[l], n = M.loff[l + 1] - M.loff[l];
    const int64_t G = M.cbase[l] + li / 256;
    chunk_of[i] = G;
    blevel[i] = l;
    if (li % 256 == 0) {
      chunk_start[G] = (int64_t)i;
      chunk_size[G] = (int32_t)(n - li < 256 ? n - li : 256);
    }
  }
}
// a chunk emits if any of its blocks does (pass A's emit_any)
__global__ void k_chunk_emits(const uint8_t* emit_any, const int64_t* chunk_of, uint64_t nb,
                              uint8_t* chunk_emits) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nb;
       i += (uint64_t)gridDim.x * blockDim.x)
    if (emit_any[i]) chunk_emits[chunk_of[i]] = 1;
}
// pass A's per-block counts laid out in emission order -- chunk by chunk,
// then slot k of K (axis / triangle case), then block within the chunk --
// and zeroed for chunks that emit nothing; an exclusive scan of this is
// pass B's offsets
__global__ void k_emit_order(const int32_t* cnt, int K, const int64_t* chunk_of,
                             const int64_t* chunk_start, const int32_t* chunk_size,
                             const uint8_t* chunk_emits, uint64_t nb, int64_t* out) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < nb * K;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t b = i / K;
    const int k = (int)(i % K);
    const int64_t G = chunk_of[b], cs = chunk_start[G];
    const int64_t pos = K * cs + (int64_t)k * chunk_size[G] + ((int64_t)b - cs);
    out[pos] = chunk_emits[G] ? cnt[i] : 0;
  }
}

// host orchestration
// ---------------------------------------------------------------------------

static unsigned gridn(uint64_t n) {
  return (unsigned)std::max<uint64_t>(1, std::min<uint64_t>((n + 255) / 256, 148 * 32));
}

struct Scratch {
  DevBuf bufs;
  void* tmp = nullptr;
  size_t tmp_bytes = 0;
  explicit Scratch(cudaStream_t st = nullptr) { bufs.stream = st; }
  ~Scratch() {
    if (tmp) cudaFreeAsync(tmp, bufs.stream);
  }
  int need(size_t b) {
    if (b <= tmp_bytes) return kOk;
    if (tmp) cudaFreeAsync(tmp, bufs.stream);
    tmp = nullptr;
    tmp_bytes = 0;
    DevBuf::keep_pool();
    if (cudaMallocAsync(&tmp, b, bufs.stream) != cudaSuccess) {
      set_error("device allocation failed for sort scratch");
      return kCapacityError;
    }
    tmp_bytes = b;
    return kOk;
  }
};

static int exclusive_scan(Scratch& S, const int64_t* in, int64_t* out, uint64_t n, cudaStream_t st) {
  size_t b = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, b, in, out, (int64_t)n, st);
  if (int s = S.need(b)) return s;
  MCK(cub::DeviceScan::ExclusiveSum(S.tmp, b, in, out, (int64_t)n, st));
  return kOk;
}
static int inclusive_scan(Scratch& S, const int64_t* in, int64_t* out, uint64_t n, cudaStream_t st) {
  size_t b = 0;
  cub::DeviceScan::InclusiveSum(nullptr, b, in, out, (int64_t)n, st);
  if (int s = S.need(b)) return s;
  MCK(cub::DeviceScan::InclusiveSum(S.tmp, b, in, out, (int64_t)n, st));
  return kOk;
}

// stable lexicographic order of 3-component rows: LSD radix passes z, y, x
template <typename T, bool kFloat>
static int sort_rows(Scratch& S, const T* rows, uint64_t n, uint64_t* idx, cudaStream_t st) {
  uint64_t* keys = S.bufs.get<uint64_t>(n);
  uint64_t* keys2 = S.bufs.get<uint64_t>(n);
  uint64_t* idx2 = S.bufs.get<uint64_t>(n);
  if (!keys || !keys2 || !idx2) return kCapacityError;
  k_iota<<<gridn(n), 256, 0, st>>>(idx, n);
  for (int d = 2; d >= 0; d--) {
    if (kFloat)
      k_pos_keys<<<gridn(n), 256, 0, st>>>((const double*)rows, idx, n, d, keys);
    else
      k_cell_keys<<<gridn(n), 256, 0, st>>>((const int64_t*)rows, idx, n, d, keys);
    size_t b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, b, keys, keys2, idx, idx2, (int64_t)n, 0, 64, st);
    if (int s = S.need(b)) return s;
    MCK(cub::DeviceRadixSort::SortPairs(S.tmp, b, keys, keys2, idx, idx2, (int64_t)n, 0, 64, st));
    MCK(cudaMemcpyAsync(idx, idx2, n * 8, cudaMemcpyDeviceToDevice, st));
  }
  return kOk;
}

// unique over rows: inverse[n], group starts (in sorted order); returns ng
template <typename T, bool kFloat>
static int unique_rows(Scratch& S, const T* rows, uint64_t n, uint64_t* idx, int64_t* inverse,
                       int64_t* gstart, int64_t* ng, cudaStream_t st) {
  if (int s = sort_rows<T, kFloat>(S, rows, n, idx, st)) return s;
  int64_t* flag = S.bufs.get<int64_t>(n);
  int64_t* gid = S.bufs.get<int64_t>(n);
  if (!flag || !gid) return kCapacityError;
  k_group_flags<T><<<gridn(n), 256, 0, st>>>(rows, idx, n, flag);
  if (int s = inclusive_scan(S, flag, gid, n, st)) return s;
  k_group_assign<<<gridn(n), 256, 0, st>>>(idx, gid, n, inverse, gstart);
  MCK(cudaMemcpyAsync(ng, gid + n - 1, 8, cudaMemcpyDeviceToHost, st));
  MCK(cudaStreamSynchronize(st));
  return kOk;
}

// collapse + compaction on device arrays (consumes v/n/c/tri); fills host out
// a mesh in device memory: vertices, normals, colours (nv x 3 f64 each)
// then triangles (nt x 3 i64), one allocation in that order
struct DevMesh {
  char* base = nullptr;
  int64_t nv = 0, nt = 0;
  double* v() const { return (double*)base; }
  double* n() const { return v() + 3 * nv; }
  double* c() const { return n() + 3 * nv; }
  int64_t* tri() const { return (int64_t*)(c() + 3 * nv); }
  static size_t bytes(int64_t nv, int64_t nt) { return (size_t)nv * 72 + (size_t)nt * 24 + 64; }
};

// D2H of a device mesh into caller-owned host arrays
// The mesh is one contiguous device range (v, n, c, tri).  Copies to
// pageable host memory run at a few GB/s, so large meshes go through two
// pinned 4 MB staging buffers: the D2H of chunk k overlaps the host copy of
// chunk k-1 out of the other buffer into the caller's arrays.
static int mesh_to_host(const DevMesh& m, cudaStream_t st, double* v, double* n, double* c, int64_t* tri) {
  const size_t segs[4] = {(size_t)m.nv * 24, (size_t)m.nv * 24, (size_t)m.nv * 24, (size_t)m.nt * 24};
  char* dst[4] = {(char*)v, (char*)n, (char*)c, (char*)tri};
  const size_t total = segs[0] + segs[1] + segs[2] + segs[3];
  constexpr size_t kChunk = 4u << 20;
  // per host thread (tables on different threads extract concurrently)
  static thread_local char* pin[2] = {nullptr, nullptr};
  static thread_local cudaEvent_t ev[2] = {nullptr, nullptr};
  if (total >= 2 * kChunk && !pin[0]) {
    if (cudaMallocHost(&pin[0], kChunk) != cudaSuccess || cudaMallocHost(&pin[1], kChunk) != cudaSuccess ||
        cudaEventCreateWithFlags(&ev[0], cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&ev[1], cudaEventDisableTiming) != cudaSuccess) {
      cudaGetLastError();
      pin[0] = pin[1] = nullptr;
    }
  }
  if (total < 2 * kChunk || !pin[0]) {
    if (m.nv) {
      MCK(cudaMemcpyAsync(v, m.v(), m.nv * 24, cudaMemcpyDeviceToHost, st));
      MCK(cudaMemcpyAsync(n, m.n(), m.nv * 24, cudaMemcpyDeviceToHost, st));
      MCK(cudaMemcpyAsync(c, m.c(), m.nv * 24, cudaMemcpyDeviceToHost, st));
    }
    if (m.nt) MCK(cudaMemcpyAsync(tri, m.tri(), m.nt * 24, cudaMemcpyDeviceToHost, st));
    MCK(cudaStreamSynchronize(st));
    return kOk;
  }
  const char* src = (const char*)m.v();
  // host copy of device bytes [off, off + len) out of a staging buffer
  auto scatter = [&](const char* buf, size_t off, size_t len) {
    size_t seg_off = 0;
    for (int i = 0; i < 4 && len; i++) {
      if (off < seg_off + segs[i]) {
        const size_t in = off - seg_off, take = std::min(len, segs[i] - in);
        memcpy(dst[i] + in, buf, take);
        buf += take;
        off += take;
        len -= take;
      }
      seg_off += segs[i];
    }
  };
  const size_t nchunks = (total + kChunk - 1) / kChunk;
  for (size_t k = 0; k <= nchunks; k++) {
    if (k < nchunks) {
      const size_t off = k * kChunk, len = std::min(kChunk, total - off);
      MCK(cudaMemcpyAsync(pin[k & 1], src + off, len, cudaMemcpyDeviceToHost, st));
      MCK(cudaEventRecord(ev[k & 1], st));
    }
    if (k > 0) {
      const size_t j = k - 1, off = j * kChunk, len = std::min(kChunk, total - off);
      MCK(cudaEventSynchronize(ev[j & 1]));
      scatter(pin[j & 1], off, len);
    }
  }
  return kOk;
}

// ... into malloc'd arrays (the MeshOut of tsdf_extract_mesh / collapse)
static int mesh_to_malloc(const DevMesh& m, cudaStream_t st, MeshOut* out) {
  memset(out, 0, sizeof(*out));
  if (m.nv == 0 && m.nt == 0) return kOk;
  out->nv = m.nv;
  out->nt = m.nt;
  out->v = (double*)malloc(std::max<int64_t>(m.nv, 1) * 24);
  out->n = (double*)malloc(std::max<int64_t>(m.nv, 1) * 24);
  out->c = (double*)malloc(std::max<int64_t>(m.nv, 1) * 24);
  out->tri = (int64_t*)malloc(std::max<int64_t>(m.nt, 1) * 24);
  return mesh_to_host(m, st, out->v, out->n, out->c, out->tri);
}

// collapse + compaction on device arrays (consumes v/n/c/tri); the result
// lands in `keep` (a table-owned buffer) or in the scratch
static int collapse_device(Scratch& S, const double* v, const double* nrm, const double* col,
                           uint64_t nv, const int64_t* tri, uint64_t nt, double eps,
                           cudaStream_t st, DevMesh* out, Buf* keep) {
  *out = DevMesh{};
  if (nv == 0) return kOk;
  uint64_t* idx = S.bufs.get<uint64_t>(nv);
  int64_t* inv = S.bufs.get<int64_t>(nv);
  int64_t* gst = S.bufs.get<int64_t>(nv);
  if (!idx || !inv || !gst) return kCapacityError;
  int64_t ng = 0;
  bool exact = eps == 0.0;
  if (exact) {
    if (int s = unique_rows<double, true>(S, v, nv, idx, inv, gst, &ng, st)) return s;
  } else {
    int64_t* cells = S.bufs.get<int64_t>(3 * nv);
    if (!cells) return kCapacityError;
    k_cells<<<gridn(3 * nv), 256, 0, st>>>(v, nv, eps, cells);
    if (int s = unique_rows<int64_t, false>(S, cells, nv, idx, inv, gst, &ng, st)) return s;
  }
  double* cv = S.bufs.get<double>(3 * ng);
  double* cn = S.bufs.get<double>(3 * ng);
  double* cc = S.bufs.get<double>(3 * ng);
  int64_t* tri2 = S.bufs.get<int64_t>(3 * nt);
  int64_t* keep_t = S.bufs.get<int64_t>(nt);
  int64_t* kpos = S.bufs.get<int64_t>(nt);
  uint8_t* used8 = S.bufs.get<uint8_t>(ng);
  int64_t* used = S.bufs.get<int64_t>(ng);
  int64_t* remap = S.bufs.get<int64_t>(ng);
  if (!cv || !cn || !cc || !tri2 || !keep_t || !kpos || !used8 || !used || !remap) return kCapacityError;
  k_collapse_out<<<gridn(ng), 256, 0, st>>>(v, nrm, col, idx, gst, ng, nv, exact, cv, cn, cc);
  MCK(cudaMemsetAsync(used8, 0, ng, st));
  if (nt) k_tri_filter<<<gridn(nt), 256, 0, st>>>(tri, inv, nt, cv, tri2, keep_t, used8);
  k_u8_to_i64<<<gridn(ng), 256, 0, st>>>(used8, ng, nt == 0, used);
  if (int s = exclusive_scan(S, used, remap, ng, st)) return s;
  int64_t last_r, last_u, last_p = 0, last_k = 0;
  MCK(cudaMemcpyAsync(&last_r, remap + ng - 1, 8, cudaMemcpyDeviceToHost, st));
  MCK(cudaMemcpyAsync(&last_u, used + ng - 1, 8, cudaMemcpyDeviceToHost, st));
  if (nt) {
    if (int s = exclusive_scan(S, keep_t, kpos, nt, st)) return s;
    MCK(cudaMemcpyAsync(&last_p, kpos + nt - 1, 8, cudaMemcpyDeviceToHost, st));
    MCK(cudaMemcpyAsync(&last_k, keep_t + nt - 1, 8, cudaMemcpyDeviceToHost, st));
  }
  MCK(cudaStreamSynchronize(st));
  int64_t nu = last_r + last_u, ntk = last_p + last_k;
  DevMesh m;
  m.nv = nu;
  m.nt = ntk;
  m.base = keep ? (char*)grow(*keep, DevMesh::bytes(nu, ntk)) : S.bufs.get<char>(DevMesh::bytes(nu, ntk));
  if (!m.base) return kCapacityError;
  k_compact_verts<<<gridn(ng), 256, 0, st>>>(cv, cn, cc, used, remap, ng, m.v(), m.n(), m.c());
  if (nt) k_compact_tris<<<gridn(nt), 256, 0, st>>>(tri2, keep_t, kpos, remap, nt, m.tri());
  MCK(cudaGetLastError());
  *out = m;
  return kOk;
}

// M1-M3: the kept blocks of the table in canonical order (packed keys ascend
// within a level, levels concatenated); loff[l] .. loff[l+1] is level l
static int kept_blocks(Table* T, Scratch& S, double iso, uint64_t** skeys_out, uint32_t** sslots_out,
                       int64_t* loff) {
  cudaStream_t st = T->stream;
  const DevTable& d = T->d;
  uint64_t slots = T->slots;
  uint8_t* obs = S.bufs.get<uint8_t>(slots);
  double* rlo = S.bufs.get<double>(slots);
  double* rhi = S.bufs.get<double>(slots);
  int64_t live[kMaxLevels] = {0, 0, 0, 0}, total = 0;
  for (int l = 0; l < d.n_levels; l++) {
    if (int s = live_count(T, l, &live[l])) return s;
    total = std::max<int64_t>(total, live[l]);
  }
  uint64_t cap = std::max<int64_t>(total, 1);
  uint64_t* kkeys = S.bufs.get<uint64_t>(cap * kMaxLevels);
  uint32_t* kslots = S.bufs.get<uint32_t>(cap * kMaxLevels);
  unsigned long long* kcnt = S.bufs.get<unsigned long long>(kMaxLevels);
  if (!obs || !rlo || !rhi || !kkeys || !kslots || !kcnt) {
    set_error("device allocation failed for mesh scratch");
    return kCapacityError;
  }
  MCK(cudaMemsetAsync(kcnt, 0, kMaxLevels * 8, st));
  {
    int _pid = prof_begin(T, "k_block_range");
    k_block_range<<<148 * 16, 256, 0, st>>>(d, obs, rlo, rhi);
    prof_end(T, _pid);
  }
  {
    int _pid = prof_begin(T, "k_keep");
    k_keep<<<gridn(slots), 256, 0, st>>>(d, obs, rlo, rhi, iso, kkeys, kslots, cap, kcnt);
    prof_end(T, _pid);
  }
  T->launches += 2;
  unsigned long long hcnt[kMaxLevels];
  MCK(cudaMemcpyAsync(hcnt, kcnt, sizeof(hcnt), cudaMemcpyDeviceToHost, st));
  MCK(cudaStreamSynchronize(st));
  uint64_t nb = 0;
  for (int l = 0; l < d.n_levels; l++) nb += hcnt[l];
  *skeys_out = nullptr;
  *sslots_out = nullptr;
  loff[0] = 0;
  for (int l = 0; l < d.n_levels; l++) loff[l + 1] = loff[l] + (int64_t)hcnt[l];
  if (nb == 0) return kOk;
  uint64_t* skeys = S.bufs.get<uint64_t>(nb);
  uint32_t* sslots = S.bufs.get<uint32_t>(nb);
  if (!skeys || !sslots) return kCapacityError;
  for (int l = 0; l < d.n_levels; l++) {
    const uint64_t n = hcnt[l];
    if (!n) continue;
    size_t b = 0;
    cub::DeviceRadixSort::SortPairs(nullptr, b, kkeys + l * cap, skeys + loff[l], kslots + l * cap,
                                    sslots + loff[l], (int64_t)n, 0, 63, st);
    if (int s = S.need(b)) return s;
    MCK(cub::DeviceRadixSort::SortPairs(S.tmp, b, kkeys + l * cap, skeys + loff[l], kslots + l * cap,
                                        sslots + loff[l], (int64_t)n, 0, 63, st));
  }
  *skeys_out = skeys;
  *sslots_out = sslots;
  return kOk;
}

// raw Marching Cubes output in the reference's emission order: lattice-unit
// positions, unnormalised normals, colours and triangles before the vertex
// dedup (device arrays in the scratch)
struct RawDev {
  double *v = nullptr, *n = nullptr, *c = nullptr;
  int64_t* tri = nullptr;
  int64_t nv = 0, nt = 0;
};

// M4-M6 over kept blocks given as slots in canonical order with level
// offsets loff[0..n_levels]; chunks of 256 restart at every level
static int emit_raw(Table* T, Scratch& S, const uint32_t* sslots, const int64_t* loff, double iso,
                    RawDev* raw) {
  *raw = RawDev{};
  cudaStream_t st = T->stream;
  const DevTable& d = T->d;
  const uint64_t nb = (uint64_t)loff[d.n_levels];
  if (nb == 0) return kOk;
  int32_t* blevel = S.bufs.get<int32_t>(nb);
  if (!blevel) return kCapacityError;
  ChunkMeta CM{};
  CM.n_levels = d.n_levels;
  uint64_t nchunks = 0;
  for (int l = 0; l < d.n_levels; l++) {
    CM.loff[l] = loff[l];
    CM.cbase[l] = (int64_t)nchunks;
    nchunks += (uint64_t)(loff[l + 1] - loff[l] + 255) / 256;
  }
  CM.loff[d.n_levels] = loff[d.n_levels];
  int64_t* chunk_of = S.bufs.get<int64_t>(nb);
  int64_t* chunk_start = S.bufs.get<int64_t>(nchunks);
  int32_t* chunk_size = S.bufs.get<int32_t>(nchunks);
  int32_t* edge_cnt = S.bufs.get<int32_t>(nb * 3);
  int32_t* tri_cnt = S.bufs.get<int32_t>(nb * 5);
  uint8_t* emit_any = S.bufs.get<uint8_t>(nb);
  if (!chunk_of || !chunk_start || !chunk_size || !edge_cnt || !tri_cnt || !emit_any)
    return kCapacityError;
  k_chunk_meta<<<gridn(nb), 256, 0, st>>>(CM, nb, chunk_of, blevel, chunk_start, chunk_size);
  McArgs A{};
  A.t = d;
  A.slots = sslots;
  A.blk_level = blevel;
  A.chunk_of = chunk_of;
  A.chunk_start = chunk_start;
  A.chunk_size = chunk_size;
  A.n_blocks = nb;
  A.iso = iso;
  A.edge_cnt = edge_cnt;
  A.tri_cnt = tri_cnt;
  A.emit_any = emit_any;
  size_t smem = sizeof(McSmem);
  MCK(cudaFuncSetAttribute(k_mc<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  MCK(cudaFuncSetAttribute(k_mc<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  unsigned g = (unsigned)std::min<uint64_t>(nb, 148 * 4);
  {
    int _pid = prof_begin(T, "k_mc_count");
    k_mc<false><<<g, kMcThreads, smem, st>>>(A);
    prof_end(T, _pid);
  }
  T->launches++;
  MCK(cudaGetLastError());
  // emission-order offsets for pass B, on the device
  uint8_t* chunk_emits = S.bufs.get<uint8_t>(nchunks);
  int64_t* ecnt = S.bufs.get<int64_t>(nb * 3);
  int64_t* tcnt = S.bufs.get<int64_t>(nb * 5);
  int64_t* voff = S.bufs.get<int64_t>(nb * 3);
  int64_t* toff = S.bufs.get<int64_t>(nb * 5);
  if (!chunk_emits || !ecnt || !tcnt || !voff || !toff) return kCapacityError;
  MCK(cudaMemsetAsync(chunk_emits, 0, nchunks, st));
  k_chunk_emits<<<gridn(nb), 256, 0, st>>>(emit_any, chunk_of, nb, chunk_emits);
  k_emit_order<<<gridn(nb * 3), 256, 0, st>>>(edge_cnt, 3, chunk_of, chunk_start, chunk_size, chunk_emits, nb, ecnt);
  k_emit_order<<<gridn(nb * 5), 256, 0, st>>>(tri_cnt, 5, chunk_of, chunk_start, chunk_size, chunk_emits, nb, tcnt);
  if (int s = exclusive_scan(S, ecnt, voff, nb * 3, st)) return s;
  if (int s = exclusive_scan(S, tcnt, toff, nb * 5, st)) return s;
  int64_t tails[4];
  MCK(cudaMemcpyAsync(&tails[0], voff + nb * 3 - 1, 8, cudaMemcpyDeviceToHost, st));
  MCK(cudaMemcpyAsync(&tails[1], ecnt + nb * 3 - 1, 8, cudaMemcpyDeviceToHost, st));
  MCK(cudaMemcpyAsync(&tails[2], toff + nb * 5 - 1, 8, cudaMemcpyDeviceToHost, st));
  MCK(cudaMemcpyAsync(&tails[3], tcnt + nb * 5 - 1, 8, cudaMemcpyDeviceToHost, st));
  MCK(cudaStreamSynchronize(st));
  const int64_t vtot = tails[0] + tails[1], ttot = tails[2] + tails[3];
  T->launches += 5;
  if (ttot == 0) return kOk;  // reference: no triangles -> empty mesh
  double* vpos = S.bufs.get<double>(3 * vtot);
  double* vnrm = S.bufs.get<double>(3 * vtot);
  double* vcol = S.bufs.get<double>(3 * vtot);
  int64_t* tri = S.bufs.get<int64_t>(3 * ttot);
  if (!vpos || !vnrm || !vcol || !tri) {
    set_error("device allocation failed for mesh output");
    return kCapacityError;
  }
  A.chunk_emits = chunk_emits;
  A.voff = voff;
  A.toff = toff;
  A.vpos = vpos;
  A.vnrm = vnrm;
  A.vcol = vcol;
  A.tri = tri;
  {
    int _pid = prof_begin(T, "k_mc_emit");
    k_mc<true><<<g, kMcThreads, smem, st>>>(A);
    prof_end(T, _pid);
  }
  T->launches++;
  MCK(cudaGetLastError());
  *raw = RawDev{vpos, vnrm, vcol, tri, vtot, ttot};
  return kOk;
}

// M7: exact dedup of bit-identical vertices (normals summed in emission
// order), winding fix, epsilon collapse and compaction
static int finish_raw(Scratch& S, const RawDev& r, double edge, double eps, cudaStream_t st,
                      DevMesh* out, Buf* keep) {
  *out = DevMesh{};
  if (r.nt == 0) return kOk;
  const uint64_t nv = (uint64_t)r.nv, nt = (uint64_t)r.nt;
  uint64_t* idx = S.bufs.get<uint64_t>(nv);
  int64_t* inv = S.bufs.get<int64_t>(nv);
  int64_t* gst = S.bufs.get<int64_t>(nv);
  if (!idx || !inv || !gst) return kCapacityError;
  int64_t ng = 0;
  if (int s = unique_rows<double, true>(S, r.v, nv, idx, inv, gst, &ng, st)) return s;
  double* mv = S.bufs.get<double>(3 * ng);
  double* mn = S.bufs.get<double>(3 * ng);
  double* mc = S.bufs.get<double>(3 * ng);
  int64_t* mt = S.bufs.get<int64_t>(3 * nt);
  if (!mv || !mn || !mc || !mt) return kCapacityError;
  k_dedup_out<<<gridn(ng), 256, 0, st>>>(r.v, r.n, r.c, idx, gst, ng, nv, edge / 16.0, mv, mn, mc);
  k_orient<<<gridn(nt), 256, 0, st>>>(r.tri, inv, nt, mv, mn, mt);
  MCK(cudaGetLastError());
  return collapse_device(S, mv, mn, mc, (uint64_t)ng, mt, nt, eps, st, out, keep);
}

static int extract_mesh_dev(Table* T, double iso, double eps, DevMesh* out) {
  *out = DevMesh{};
  if (eps < 0) {
    set_error("epsilon must be non-negative");
    return kValueError;
  }
  if (int s = load_tables()) return s;
  cudaStream_t st = T->stream;
  MCK(cudaStreamSynchronize(st));
  Scratch S(st);
  uint64_t* skeys;
  uint32_t* sslots;
  int64_t loff[kMaxLevels + 1];
  if (int s = kept_blocks(T, S, iso, &skeys, &sslots, loff)) return s;
  RawDev raw;
  if (int s = emit_raw(T, S, sslots, loff, iso, &raw)) return s;
  T->launches += 12;
  int s = finish_raw(S, raw, T->d.edge, eps, st, out, &T->mesh_out);
  prof_collect(T);
  return s;
}

// ---- sharded extraction with a halo (sharding.extract_mesh_halo) -----------

// the per-block summary the kept-set decision needs (meshing.py:428-456):
// packed key, level, "observed" flag and observed tsdf range of every live
// block of this table
__global__ void k_block_summary(DevTable t, const uint8_t* obs, const double* rlo, const double* rhi,
                                uint64_t* keys, int32_t* levels, uint8_t* o, double* lo, double* hi,
                                unsigned long long* n) {
  for (uint64_t s = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; s <= t.mask;
       s += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = t.keys[s];
    const uint32_t v = t.vals[s];
    if (!key_live(k) || v == kPending) continue;
    const unsigned long long i = atomicAdd(n, 1ull);
    keys[i] = k;
    levels[i] = val_level(v);
    o[i] = obs[s];
    lo[i] = rlo[s];
    hi[i] = rhi[s];
  }
}

int mesh_block_summary(Table* T, uint64_t* keys, int32_t* levels, uint8_t* obs_out, double* lo,
                       double* hi, int64_t cap, int64_t* n_out) {
  *n_out = 0;
  cudaStream_t st = T->stream;
  MCK(cudaStreamSynchronize(st));
  Scratch S(st);
  const uint64_t slots = T->slots;
  uint8_t* obs = S.bufs.get<uint8_t>(slots);
  double* rlo = S.bufs.get<double>(slots);
  double* rhi = S.bufs.get<double>(slots);
  int64_t total = 0;
  for (int l = 0; l < T->d.n_levels; l++) {
    int64_t nl = 0;
    if (int s = live_count(T, l, &nl)) return s;
    total += nl;
  }
  if (total > cap) {
    set_error("mesh_block_summary: output arrays too small");
    return kValueError;
  }
  const uint64_t m = (uint64_t)std::max<int64_t>(total, 1);
  uint64_t* dk = S.bufs.get<uint64_t>(m);
  int32_t* dl = S.bufs.get<int32_t>(m);
  uint8_t* dob = S.bufs.get<uint8_t>(m);
  double* dlo = S.bufs.get<double>(m);
  double* dhi = S.bufs.get<double>(m);
  unsigned long long* dn = S.bufs.get<unsigned long long>(1);
  if (!obs || !rlo || !rhi || !dk || !dl || !dob || !dlo || !dhi || !dn) return kCapacityError;
  MCK(cudaMemsetAsync(dn, 0, 8, st));
  k_block_range<<<148 * 16, 256, 0, st>>>(T->d, obs, rlo, rhi);
  k_block_summary<<<gridn(slots), 256, 0, st>>>(T->d, obs, rlo, rhi, dk, dl, dob, dlo, dhi, dn);
  T->launches += 2;
  unsigned long long hn = 0;
  MCK(cudaMemcpyAsync(&hn, dn, 8, cudaMemcpyDeviceToHost, st));
  MCK(cudaStreamSynchronize(st));
  if (hn) {
    MCK(cudaMemcpyAsync(keys, dk, hn * 8, cudaMemcpyDeviceToHost, st));
    MCK(cudaMemcpyAsync(levels, dl, hn * 4, cudaMemcpyDeviceToHost, st));
    MCK(cudaMemcpyAsync(obs_out, dob, hn, cudaMemcpyDeviceToHost, st));
    MCK(cudaMemcpyAsync(lo, dlo, hn * 8, cudaMemcpyDeviceToHost, st));
    MCK(cudaMemcpyAsync(hi, dhi, hn * 8, cudaMemcpyDeviceToHost, st));
    MCK(cudaStreamSynchronize(st));
  }
  *n_out = (int64_t)hn;
  return kOk;
}

__global__ void k_find_slots(DevTable t, const uint64_t* keys, uint64_t n, uint32_t* slots,
                             unsigned long long* missing) {
  for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n;
       i += (uint64_t)gridDim.x * blockDim.x) {
    const int64_t s = table_find(t, keys[i]);
    if (s < 0) atomicAdd(missing, 1ull);
    slots[i] = s < 0 ? 0u : (uint32_t)s;
  }
}

// raw emission (pre-dedup) for a caller-given kept list: `keys` packed, in
// canonical order per level, level_counts[l] of them at level l; every key
// and its 26 neighbours present in this table must be the map's own
int mesh_emit_keys(Table* T, const uint64_t* keys, const int64_t* level_counts, double iso,
                   MeshOut* out) {
  memset(out, 0, sizeof(*out));
  if (int s = load_tables()) return s;
  cudaStream_t st = T->stream;
  MCK(cudaStreamSynchronize(st));
  Scratch S(st);
  int64_t loff[kMaxLevels + 1];
  loff[0] = 0;
  for (int l = 0; l < T->d.n_levels; l++) loff[l + 1] = loff[l] + level_counts[l];
  const uint64_t nb = (uint64_t)loff[T->d.n_levels];
  if (nb == 0) return kOk;
  uint64_t* dk = S.bufs.get<uint64_t>(nb);
  uint32_t* ds = S.bufs.get<uint32_t>(nb);
  unsigned long long* miss = S.bufs.get<unsigned long long>(1);
  if (!dk || !ds || !miss) return kCapacityError;
  MCK(cudaMemcpyAsync(dk, keys, nb * 8, cudaMemcpyHostToDevice, st));
  MCK(cudaMemsetAsync(miss, 0, 8, st));
  k_find_slots<<<gridn(nb), 256, 0, st>>>(T->d, dk, nb, ds, miss);
  T->launches++;
  unsigned long long hm = 0;
  MCK(cudaMemcpyAsync(&hm, miss, 8, cudaMemcpyDeviceToHost, st));
  MCK(cudaStreamSynchronize(st));
  if (hm) {
    set_error("mesh_emit_keys: " + std::to_string(hm) + " kept blocks are not in the table");
    return kNotFound;
  }
  RawDev raw;
  if (int s = emit_raw(T, S, ds, loff, iso, &raw)) return s;
  if (raw.nt == 0) return kOk;
  DevMesh m;
  m.nv = raw.nv;
  m.nt = raw.nt;
  m.base = S.bufs.get<char>(DevMesh::bytes(raw.nv, raw.nt));
  if (!m.base) return kCapacityError;
  MCK(cudaMemcpyAsync(m.v(), raw.v, raw.nv * 24, cudaMemcpyDeviceToDevice, st));
  MCK(cudaMemcpyAsync(m.n(), raw.n, raw.nv * 24, cudaMemcpyDeviceToDevice, st));
  MCK(cudaMemcpyAsync(m.c(), raw.c, raw.nv * 24, cudaMemcpyDeviceToDevice, st));
  MCK(cudaMemcpyAsync(m.tri(), raw.tri, raw.nt * 24, cudaMemcpyDeviceToDevice, st));
  return mesh_to_malloc(m, st, out);
}

// M7 over raw arrays concatenated from several mesh_emit_keys calls (their
// triangle indices already offset): the same final mesh as extract_mesh
int mesh_finish(const double* v, const double* n, const double* c, int64_t nv, const int64_t* tri,
                int64_t nt, double edge, double eps, MeshOut* out) {
  memset(out, 0, sizeof(*out));
  if (eps < 0) {
    set_error("epsilon must be non-negative");
    return kValueError;
  }
  if (nt == 0 || nv == 0) return kOk;
  Scratch S;
  double* dv = S.bufs.get<double>(3 * nv);
  double* dn = S.bufs.get<double>(3 * nv);
  double* dc = S.bufs.get<double>(3 * nv);
  int64_t* dt = S.bufs.get<int64_t>(3 * nt);
  if (!dv || !dn || !dc || !dt) return kCapacityError;
  MCK(cudaMemcpy(dv, v, nv * 24, cudaMemcpyHostToDevice));
  MCK(cudaMemcpy(dn, n, nv * 24, cudaMemcpyHostToDevice));
  MCK(cudaMemcpy(dc, c, nv * 24, cudaMemcpyHostToDevice));
  MCK(cudaMemcpy(dt, tri, nt * 24, cudaMemcpyHostToDevice));
  RawDev raw{dv, dn, dc, dt, nv, nt};
  DevMesh m;
  if (int s = finish_raw(S, raw, edge, eps, 0, &m, nullptr)) return s;
  return mesh_to_malloc(m, 0, out);
}

int extract_mesh(Table* T, double iso, double eps, MeshOut* out) {
  memset(out, 0, sizeof(*out));
  DevMesh m;
  if (int s = extract_mesh_dev(T, iso, eps, &m)) return s;
  return mesh_to_malloc(m, T->stream, out);
}

// two-phase extraction: the mesh stays on the device until the caller has
// allocated its arrays, then one D2H per array straight into them
int extract_mesh_begin(Table* T, double iso, double eps, int64_t* nv, int64_t* nt) {
  DevMesh m;
  T->mesh_nv = -1;
  if (int s = extract_mesh_dev(T, iso, eps, &m)) return s;
  if (m.nv && m.base != (char*)T->mesh_out.p) {
    set_error("extract_mesh_begin: mesh not in the table buffer");
    return kCudaError;
  }
  T->mesh_nv = m.nv;
  T->mesh_nt = m.nt;
  *nv = m.nv;
  *nt = m.nt;
  return kOk;
}

int extract_mesh_read(Table* T, double* v, double* n, double* c, int64_t* tri) {
  if (T->mesh_nv < 0) {
    set_error("extract_mesh_read: no extracted mesh (call extract_mesh_begin first)");
    return kValueError;
  }
  DevMesh m;
  m.base = (char*)T->mesh_out.p;
  m.nv = T->mesh_nv;
  m.nt = T->mesh_nt;
  T->mesh_nv = -1;
  return mesh_to_host(m, T->stream, v, n, c, tri);
}

int collapse_vertices(const double* v, const double* n, const double* c, int64_t nv,
                      const int64_t* tri, int64_t nt, double eps, MeshOut* out) {
  memset(out, 0, sizeof(*out));
  if (eps < 0) {
    set_error("epsilon must be non-negative");
    return kValueError;
  }
  if (nv == 0) return kOk;
  Scratch S;
  double* dv = S.bufs.get<double>(3 * nv);
  double* dn = S.bufs.get<double>(3 * nv);
  double* dc = S.bufs.get<double>(3 * nv);
  int64_t* dt = S.bufs.get<int64_t>(3 * std::max<int64_t>(nt, 1));
  if (!dv || !dn || !dc || !dt) return kCapacityError;
  MCK(cudaMemcpy(dv, v, nv * 24, cudaMemcpyHostToDevice));
  MCK(cudaMemcpy(dn, n, nv * 24, cudaMemcpyHostToDevice));
  MCK(cudaMemcpy(dc, c, nv * 24, cudaMemcpyHostToDevice));
  if (nt) MCK(cudaMemcpy(dt, tri, nt * 24, cudaMemcpyHostToDevice));
  DevMesh m;
  if (int s = collapse_device(S, dv, dn, dc, (uint64_t)nv, dt, (uint64_t)nt, eps, 0, &m, nullptr)) return s;
  return mesh_to_malloc(m, 0, out);
}

void mesh_free(MeshOut* m) {
  free(m->v);
  free(m->n);
  free(m->c);
  free(m->tri);
  memset(m, 0, sizeof(*m));
}

}  // namespace tsdf
