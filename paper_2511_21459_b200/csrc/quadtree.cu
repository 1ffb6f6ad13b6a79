// Contrast quadtree and depth-seeded splats (reference quadtree.py:42-148,
// the paper's splat-seeding kernel).
//
// B200 design: the integral images are built with one thread per column and
// channel, then one per row and channel, each a sequential running sum --
// exactly numpy's cumsum(cumsum(img, axis=0), axis=1) -- so every box sum
// and every contrast is bit-identical.  The tree is built level-synchronously
// like the reference: one kernel evaluates a level's frontier (contrast,
// split decision, child count), two exclusive scans place the children and
// the leaves in frontier order, and an emit kernel writes them, so the leaf
// list comes out in the reference's breadth-first order.  Seeding is one
// thread per leaf.
#include <cub/cub.cuh>

#include <algorithm>
#include <cmath>
#include <cstring>

#include "../../include/tsdf_b200.h"
#include "fusion.h"

namespace {
using tsdf::cuda_status;
using tsdf::set_error;

constexpr int kThreads = 256;
__constant__ double kLuma[3] = {0.2989, 0.5870, 0.1140};  // quadtree.py:19

// S[y + 1][x + 1][c] = sum_{y' <= y} img[y'][x][c] (sequential in y)
__global__ void k_integral_cols(const double* __restrict__ img, int H, int W, double* S, double* S2) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 3 * W) return;
  const int x = i / 3, c = i % 3;
  double a = 0.0, b = 0.0;
  for (int y = 0; y < H; y++) {
    const double v = img[((int64_t)y * W + x) * 3 + c];
    a = __dadd_rn(a, v);
    b = __dadd_rn(b, __dmul_rn(v, v));
    const int64_t o = ((int64_t)(y + 1) * (W + 1) + x + 1) * 3 + c;
    S[o] = a;
    S2[o] = b;
  }
}

// then the running sum along x of each row (sequential in x)
__global__ void k_integral_rows(int H, int W, double* S, double* S2) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= 3 * H) return;
  const int y = i / 3 + 1, c = i % 3;
  double a = 0.0, b = 0.0;
  for (int x = 1; x <= W; x++) {
    const int64_t o = ((int64_t)y * (W + 1) + x) * 3 + c;
    a = __dadd_rn(a, S[o]);
    b = __dadd_rn(b, S2[o]);
    S[o] = a;
    S2[o] = b;
  }
}

struct Node {
  int x0, y0, w, h;
};

// _IntegralImage.contrast (quadtree.py:65-75): box sums left to right,
// var = s2 / n - (s / n)^2 clamped at 0 (np.maximum keeps -0.0), then the
// luma dot in OpenBLAS dgemv's order for this frontier size (a frontier of
// one node is dotted in another order than larger ones; SURVEY Appendix A
// method, measured on the reference host)
__device__ double node_contrast(const double* __restrict__ S, const double* __restrict__ S2, int W,
                                Node nd, bool single) {
  const double n = (double)((int64_t)nd.w * nd.h);
  const int64_t r0 = (int64_t)nd.y0 * (W + 1), r1 = (int64_t)(nd.y0 + nd.h) * (W + 1);
  const int64_t a = (r1 + nd.x0 + nd.w) * 3, b = (r0 + nd.x0 + nd.w) * 3, c = (r1 + nd.x0) * 3,
                d = (r0 + nd.x0) * 3;
  double var[3];
#pragma unroll
  for (int k = 0; k < 3; k++) {
    const double s = __dadd_rn(__dsub_rn(__dsub_rn(S[a + k], S[b + k]), S[c + k]), S[d + k]);
    const double s2 = __dadd_rn(__dsub_rn(__dsub_rn(S2[a + k], S2[b + k]), S2[c + k]), S2[d + k]);
    const double m = __ddiv_rn(s, n);
    const double v = __dsub_rn(__ddiv_rn(s2, n), __dmul_rn(m, m));
    var[k] = (v >= 0.0 || isnan(v)) ? v : 0.0;
  }
  return single ? __fma_rn(var[2], kLuma[2], __fma_rn(var[1], kLuma[1], __dmul_rn(var[0], kLuma[0])))
                : __fma_rn(var[2], kLuma[2], __fma_rn(var[0], kLuma[0], __dmul_rn(var[1], kLuma[1])));
}

// children at floor midpoints: top-left, bottom-left, top-right,
// bottom-right; zero-extent children are not created (quadtree.py:78-91)
__device__ inline int children(Node nd, Node* out) {
  const int w1 = nd.w / 2, h1 = nd.h / 2, w2 = nd.w - w1, h2 = nd.h - h1;
  const Node c[4] = {{nd.x0, nd.y0, w1, h1}, {nd.x0, nd.y0 + h1, w1, h2},
                     {nd.x0 + w1, nd.y0, w2, h1}, {nd.x0 + w1, nd.y0 + h1, w2, h2}};
  int k = 0;
#pragma unroll
  for (int j = 0; j < 4; j++)
    if (c[j].w > 0 && c[j].h > 0) out[k++] = c[j];
  return k;
}

__global__ void k_qt_level(const Node* __restrict__ front, int n, const double* __restrict__ S,
                           const double* __restrict__ S2, int W, double thr, int min_pixel,
                           double* con, int* nchild, int* leaf) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const Node nd = front[i];
  const double c = node_contrast(S, S2, W, nd, n == 1);
  con[i] = c;
  const bool split = c > thr && min(nd.w, nd.h) > min_pixel;
  Node tmp[4];
  nchild[i] = split ? children(nd, tmp) : 0;
  leaf[i] = split ? 0 : 1;
}

__global__ void k_qt_emit(const Node* __restrict__ front, int n, const double* __restrict__ con,
                          const int* __restrict__ nchild, const int* __restrict__ coff,
                          const int* __restrict__ loff, Node* next, Node* leaves, double* lcon,
                          int64_t leaf_base) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const Node nd = front[i];
  if (nchild[i]) {
    Node ch[4];
    const int k = children(nd, ch);
    for (int j = 0; j < k; j++) next[coff[i] + j] = ch[j];
  } else {
    // a splitting node always has a non-empty bottom-right child, so a
    // zero count means a leaf
    leaves[leaf_base + loff[i]] = nd;
    lcon[leaf_base + loff[i]] = con[i];
  }
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

__device__ inline double depth_at(const void* p, int dt, int64_t i, double scale) {
  switch (dt) {
    case TSDF_F64: return ((const double*)p)[i];
    case TSDF_F32: return (double)((const float*)p)[i];
    default: return (double)((const uint16_t*)p)[i] / scale;
  }
}
__device__ inline double color_at(const void* p, int dt, int64_t i) {
  switch (dt) {
    case TSDF_F64: return ((const double*)p)[i];
    case TSDF_F32: return (double)((const float*)p)[i];
    default: return (double)((const uint8_t*)p)[i] / 255.0;
  }
}

struct Cam {
  double fx, fy, cx, cy, R[9], t[3];
};

// seed_splats (quadtree.py:112-148): the leaf centre back-projected
// (geometry.py:122-125) and moved to world with the single-point matmul
// order (geometry.py:31, gemv), scale = w d / fx, colour = the leaf's mean
// (numpy's axis-0 mean: a sequential sum in row-major pixel order / n)
__global__ void k_seed(const Node* __restrict__ leaves, int64_t n, const void* depth, int ddt,
                       double scale, const void* rgb, int cdt, int W, Cam K, double* pos, double* sc,
                       double* col, uint8_t* ok) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const Node nd = leaves[i];
  const int u = nd.x0 + nd.w / 2, v = nd.y0 + nd.h / 2;
  const double d = depth_at(depth, ddt, (int64_t)v * W + u, scale);
  if (!(isfinite(d) && d > 0)) {
    ok[i] = 0;
    return;
  }
  ok[i] = 1;
  const double p[3] = {__dmul_rn(__ddiv_rn(__dsub_rn((double)u, K.cx), K.fx), d),
                       __dmul_rn(__ddiv_rn(__dsub_rn((double)v, K.cy), K.fy), d), d};
#pragma unroll
  for (int j = 0; j < 3; j++) {
    const double acc = __fma_rn(p[2], K.R[3 * j + 2], __fma_rn(p[0], K.R[3 * j], __dmul_rn(p[1], K.R[3 * j + 1])));
    pos[3 * i + j] = __dadd_rn(acc, K.t[j]);
  }
  sc[i] = __ddiv_rn(__dmul_rn((double)nd.w, d), K.fx);
  if (!rgb) {
    col[3 * i] = col[3 * i + 1] = col[3 * i + 2] = 0.5;
    return;
  }
  double s[3] = {0.0, 0.0, 0.0};
  for (int y = nd.y0; y < nd.y0 + nd.h; y++)
    for (int x = nd.x0; x < nd.x0 + nd.w; x++) {
      const int64_t o = ((int64_t)y * W + x) * 3;
#pragma unroll
      for (int k = 0; k < 3; k++) s[k] = __dadd_rn(s[k], color_at(rgb, cdt, o + k));
    }
  const double cnt = (double)((int64_t)nd.w * nd.h);
#pragma unroll
  for (int k = 0; k < 3; k++) col[3 * i + k] = __ddiv_rn(s[k], cnt);
}

}  // namespace

extern "C" int tsdf_quadtree_build(const double* image, int32_t height, int32_t width, int32_t mem,
                                   double threshold, int32_t min_pixel, int32_t* leaves_out,
                                   double* contrast_out, int64_t* n_leaves, void* cuda_stream) {
  if (height <= 0 || width <= 0 || !image || !leaves_out || !contrast_out || !n_leaves ||
      (mem != TSDF_MEM_HOST && mem != TSDF_MEM_DEVICE)) {
    set_error("quadtree_build: image is empty or a buffer is missing");
    return TSDF_EVALUE;
  }
  cudaStream_t s = (cudaStream_t)cuda_stream;
  Scratch M{s, {}};
  const int64_t npx = (int64_t)height * width;
  const double* img = image;
  if (mem == TSDF_MEM_HOST) {
    double* d = M.get<double>(3 * npx);
    if (!d) return cuda_status(cudaErrorMemoryAllocation, "quadtree_build");
    cudaMemcpyAsync(d, image, 24 * npx, cudaMemcpyHostToDevice, s);
    img = d;
  }
  const int64_t ns = (int64_t)(height + 1) * (width + 1) * 3;
  double* S = M.get<double>(ns);
  double* S2 = M.get<double>(ns);
  Node* fa = M.get<Node>(npx);
  Node* fb = M.get<Node>(npx);
  Node* leaves = M.get<Node>(npx);
  double* lcon = M.get<double>(npx);
  double* con = M.get<double>(npx);
  int* nchild = M.get<int>(npx);
  int* leaf = M.get<int>(npx);
  int* coff = M.get<int>(npx);
  int* loff = M.get<int>(npx);
  size_t tb = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tb, nchild, coff, (int)npx, s);
  void* tmp = M.get<char>(tb);
  int* h_tail = nullptr;
  if (!S || !S2 || !fa || !fb || !leaves || !lcon || !con || !nchild || !leaf || !coff || !loff || !tmp ||
      cudaMallocHost(&h_tail, 4 * sizeof(int)) != cudaSuccess)
    return cuda_status(cudaErrorMemoryAllocation, "quadtree_build");
  cudaMemsetAsync(S, 0, ns * sizeof(double), s);
  cudaMemsetAsync(S2, 0, ns * sizeof(double), s);
  k_integral_cols<<<(3 * width + kThreads - 1) / kThreads, kThreads, 0, s>>>(img, height, width, S, S2);
  k_integral_rows<<<(3 * height + kThreads - 1) / kThreads, kThreads, 0, s>>>(height, width, S, S2);
  const Node root{0, 0, width, height};
  cudaMemcpyAsync(fa, &root, sizeof(Node), cudaMemcpyHostToDevice, s);
  int n = 1;
  int64_t nl = 0;
  int rc = TSDF_OK;
  // every split halves the larger side, so a tree deeper than this only
  // happens when 1x1 nodes keep splitting (min_pixel 0 with a negative
  // threshold), where the reference never terminates
  int max_levels = 2;
  for (int e = std::max(height, width); e > 1; e = (e + 1) / 2) max_levels += 2;
  for (int level = 0; n > 0; level++) {
    if (level > max_levels) {
      set_error("quadtree_build: 1x1 nodes keep splitting (min_pixel 0 with a negative threshold)");
      rc = TSDF_EVALUE;
      break;
    }
    const int g = (n + kThreads - 1) / kThreads;
    k_qt_level<<<g, kThreads, 0, s>>>(fa, n, S, S2, width, threshold, min_pixel, con, nchild, leaf);
    cub::DeviceScan::ExclusiveSum(tmp, tb, nchild, coff, n, s);
    cub::DeviceScan::ExclusiveSum(tmp, tb, leaf, loff, n, s);
    k_qt_emit<<<g, kThreads, 0, s>>>(fa, n, con, nchild, coff, loff, fb, leaves, lcon, nl);
    cudaMemcpyAsync(h_tail, coff + n - 1, sizeof(int), cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(h_tail + 1, nchild + n - 1, sizeof(int), cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(h_tail + 2, loff + n - 1, sizeof(int), cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(h_tail + 3, leaf + n - 1, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (cudaError_t e = cudaStreamSynchronize(s)) {
      rc = cuda_status(e, "quadtree_build");
      break;
    }
    nl += h_tail[2] + h_tail[3];
    n = h_tail[0] + h_tail[1];
    std::swap(fa, fb);
  }
  if (rc == TSDF_OK) {
    cudaMemcpyAsync(leaves_out, leaves, nl * sizeof(Node), cudaMemcpyDeviceToHost, s);
    cudaMemcpyAsync(contrast_out, lcon, nl * sizeof(double), cudaMemcpyDeviceToHost, s);
    if (cudaError_t e = cudaStreamSynchronize(s)) rc = cuda_status(e, "quadtree_build");
    *n_leaves = nl;
  }
  cudaFreeHost(h_tail);
  return rc;
}

extern "C" int tsdf_seed_splats(const int32_t* leaves, int64_t n, const void* depth, int32_t depth_dtype,
                                double depth_scale, const void* rgb, int32_t rgb_dtype, int32_t height,
                                int32_t width, int32_t mem, const double* K, const double* R,
                                const double* trans, double* pos_out, double* scale_out,
                                double* color_out, uint8_t* valid_out, void* cuda_stream) {
  if (n < 0 || height <= 0 || width <= 0 || !depth || !K || !R || !trans ||
      (n && (!leaves || !pos_out || !scale_out || !color_out || !valid_out)) ||
      (depth_dtype != TSDF_F64 && depth_dtype != TSDF_F32 && depth_dtype != TSDF_U16) ||
      (rgb && rgb_dtype != TSDF_F64 && rgb_dtype != TSDF_F32 && rgb_dtype != TSDF_U8) ||
      !(depth_scale > 0) || (mem != TSDF_MEM_HOST && mem != TSDF_MEM_DEVICE)) {
    set_error("seed_splats: invalid arguments");
    return TSDF_EVALUE;
  }
  if (n == 0) return TSDF_OK;
  cudaStream_t s = (cudaStream_t)cuda_stream;
  Scratch M{s, {}};
  const int64_t npx = (int64_t)height * width;
  const size_t dsz = depth_dtype == TSDF_F64 ? 8 : depth_dtype == TSDF_F32 ? 4 : 2;
  const size_t csz = rgb_dtype == TSDF_F64 ? 8 : rgb_dtype == TSDF_F32 ? 4 : 1;
  const void *dd = depth, *dc = rgb;
  if (mem == TSDF_MEM_HOST) {
    void* a = M.get<char>(npx * dsz);
    if (!a) return cuda_status(cudaErrorMemoryAllocation, "seed_splats");
    cudaMemcpyAsync(a, depth, npx * dsz, cudaMemcpyHostToDevice, s);
    dd = a;
    if (rgb) {
      void* b = M.get<char>(npx * 3 * csz);
      if (!b) return cuda_status(cudaErrorMemoryAllocation, "seed_splats");
      cudaMemcpyAsync(b, rgb, npx * 3 * csz, cudaMemcpyHostToDevice, s);
      dc = b;
    }
  }
  Node* dl = M.get<Node>(n);
  double* pos = M.get<double>(3 * n);
  double* sc = M.get<double>(n);
  double* col = M.get<double>(3 * n);
  uint8_t* ok = M.get<uint8_t>(n);
  if (!dl || !pos || !sc || !col || !ok) return cuda_status(cudaErrorMemoryAllocation, "seed_splats");
  cudaMemcpyAsync(dl, leaves, n * sizeof(Node), cudaMemcpyHostToDevice, s);
  Cam cam;
  cam.fx = K[0];
  cam.fy = K[1];
  cam.cx = K[2];
  cam.cy = K[3];
  memcpy(cam.R, R, sizeof(cam.R));
  memcpy(cam.t, trans, sizeof(cam.t));
  k_seed<<<(int)((n + kThreads - 1) / kThreads), kThreads, 0, s>>>(dl, n, dd, depth_dtype, depth_scale, dc,
                                                                  rgb_dtype, width, cam, pos, sc, col, ok);
  cudaMemcpyAsync(pos_out, pos, 24 * n, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(scale_out, sc, 8 * n, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(color_out, col, 24 * n, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(valid_out, ok, n, cudaMemcpyDeviceToHost, s);
  if (cudaError_t e = cudaStreamSynchronize(s)) return cuda_status(e, "seed_splats");
  return TSDF_OK;
}
