// extern "C" boundary (include/tsdf_b200.h) over the device implementation.
#include <cmath>
#include <cstring>
#include <vector>

#include "../../include/tsdf_b200.h"
#include "fusion.h"

using namespace tsdf;

struct tsdf_table {
  Table* impl;
};

static inline Table* T_(tsdf_table* t) { return t ? t->impl : nullptr; }

#define NEED(t)                               \
  do {                                        \
    if (!(t) || !(t)->impl) {                 \
      set_error("null table handle");         \
      return TSDF_EVALUE;                     \
    }                                         \
  } while (0)

static Frame make_frame(const double* K, const double* R, const double* tr, double tau,
                        double wcap) {
  Frame f;
  memset(&f, 0, sizeof(f));
  if (K) {
    f.fx = K[0];
    f.fy = K[1];
    f.cx = K[2];
    f.cy = K[3];
  }
  memcpy(f.R, R, sizeof(f.R));
  memcpy(f.t, tr, sizeof(f.t));
  f.tau = tau;
  f.weight_cap = wcap;
  return f;
}

extern "C" {

int tsdf_table_create(int64_t n_hash, int32_t bucket, int32_t overflow, double block_edge,
                      int32_t n_levels, const int64_t* caps, void* stream, tsdf_table** out) {
  *out = nullptr;
  Table* impl = nullptr;
  int s = table_create(n_hash, bucket, overflow, block_edge, n_levels, caps, stream, &impl);
  if (s) return s;
  *out = new tsdf_table{impl};
  return TSDF_OK;
}

int tsdf_table_destroy(tsdf_table* t) {
  if (!t) return TSDF_OK;
  int s = table_destroy(t->impl);
  delete t;
  return s;
}

int tsdf_table_reset(tsdf_table* t) {
  NEED(t);
  T_(t)->version++;
  return table_reset(T_(t));
}

int tsdf_table_set_shard(tsdf_table* t, int32_t rank, int32_t world) {
  NEED(t);
  if (world < 1 || rank < 0 || rank >= world) {
    set_error("invalid shard (rank, world)");
    return TSDF_EVALUE;
  }
  T_(t)->d.shard_rank = rank;
  T_(t)->d.shard_world = world;
  return TSDF_OK;
}

int tsdf_table_set_depth_scale(tsdf_table* t, double depth_scale) {
  NEED(t);
  if (!(depth_scale > 0.0) || !std::isfinite(depth_scale)) {
    set_error("depth_scale must be positive and finite");
    return TSDF_EVALUE;
  }
  T_(t)->depth_scale = depth_scale;
  return TSDF_OK;
}

int tsdf_table_version(tsdf_table* t, uint64_t* version) {
  NEED(t);
  *version = T_(t)->version;
  return TSDF_OK;
}

int tsdf_table_stream(tsdf_table* t, void** stream) {
  NEED(t);
  *stream = (void*)T_(t)->stream;
  return TSDF_OK;
}

int tsdf_table_set_lidar_mode(tsdf_table* t, int32_t mode) {
  NEED(t);
  if (mode != TSDF_LIDAR_ORDERED && mode != TSDF_LIDAR_CHUNKED) {
    set_error("lidar mode must be TSDF_LIDAR_ORDERED (0) or TSDF_LIDAR_CHUNKED (1)");
    return TSDF_EVALUE;
  }
  T_(t)->lidar_mode = mode;
  return TSDF_OK;
}

int tsdf_table_merge_audit(tsdf_table* t, int64_t* near_threshold) {
  NEED(t);
  *near_threshold = (int64_t)T_(t)->merge_audit;
  return TSDF_OK;
}

int tsdf_integrate_depth(tsdf_table* t, const void* depth, int32_t depth_dtype, const void* rgb,
                         int32_t rgb_dtype, int32_t height, int32_t width, int32_t mem,
                         const double* K, const double* R, const double* trans, double tau,
                         double weight_cap, tsdf_integration_stats* stats) {
  NEED(t);
  T_(t)->version++;
  if (depth_dtype < 0 || depth_dtype > 3 || (rgb && (rgb_dtype < 0 || rgb_dtype > 2))) {
    set_error("unsupported dtype");
    return TSDF_EVALUE;
  }
  if (K[0] <= 0 || K[1] <= 0) {
    set_error("focal lengths must be positive");
    return TSDF_EDATASET;
  }
  IntegrationStats st;
  int s = integrate_depth(T_(t), depth, depth_dtype, rgb, rgb_dtype, height, width, mem,
                          make_frame(K, R, trans, tau, weight_cap), &st);
  memcpy(stats, &st, sizeof(st));
  return s;
}

int tsdf_integrate_depth_walk(tsdf_table* t, const void* depth, int32_t depth_dtype,
                              const void* rgb, int32_t rgb_dtype, int32_t height, int32_t width,
                              int32_t mem, const double* K, const double* R, const double* trans,
                              double tau, double weight_cap, int32_t ray_rank, int32_t ray_world,
                              uint64_t* buckets, int64_t bucket_cap, int64_t* counts,
                              tsdf_integration_stats* stats) {
  NEED(t);
  if (depth_dtype < 0 || depth_dtype > 3 || (rgb && (rgb_dtype < 0 || rgb_dtype > 2))) {
    set_error("unsupported dtype");
    return TSDF_EVALUE;
  }
  if (K[0] <= 0 || K[1] <= 0) {
    set_error("focal lengths must be positive");
    return TSDF_EDATASET;
  }
  if (bucket_cap <= 0) {
    set_error("bucket_cap must be positive");
    return TSDF_EVALUE;
  }
  IntegrationStats st;
  DepthArgs a{depth, depth_dtype, rgb, rgb_dtype, height, width, mem,
              make_frame(K, R, trans, tau, weight_cap)};
  int s = integrate_depth_walk(T_(t), a, ray_rank, ray_world, buckets, (uint64_t)bucket_cap, counts,
                               &st);
  memcpy(stats, &st, sizeof(st));
  return s;
}

int tsdf_integrate_depth_keys(tsdf_table* t, const uint64_t* keys, int64_t n,
                              tsdf_integration_stats* stats) {
  NEED(t);
  T_(t)->version++;
  if (n < 0 || (n > 0 && !keys)) {
    set_error("invalid key list");
    return TSDF_EVALUE;
  }
  IntegrationStats st;
  int s = integrate_depth_keys(T_(t), keys, n, &st);
  memcpy(stats, &st, sizeof(st));
  return s;
}

int tsdf_depth_keys(tsdf_table* t, const void* depth, int32_t depth_dtype, int32_t height,
                    int32_t width, int32_t mem, const double* K, const double* R, const double* trans,
                    double tau, uint64_t* keys, int64_t cap, int64_t* n_out) {
  NEED(t);
  if (depth_dtype < 0 || depth_dtype > 3) {
    set_error("unsupported dtype");
    return TSDF_EVALUE;
  }
  if (K[0] <= 0 || K[1] <= 0) {
    set_error("focal lengths must be positive");
    return TSDF_EDATASET;
  }
  DepthArgs a{depth, depth_dtype, nullptr, 0, height, width, mem, make_frame(K, R, trans, tau, 0.0)};
  return depth_keys(T_(t), a, keys, cap, n_out);
}

int tsdf_scan_keys(tsdf_table* t, const void* xyz, int32_t xyz_dtype, int64_t n, int32_t mem,
                   const double* R, const double* trans, double tau, uint64_t* keys, int64_t cap,
                   int64_t* n_out) {
  NEED(t);
  if (xyz_dtype < 0 || xyz_dtype > 1) {
    set_error("unsupported dtype");
    return TSDF_EVALUE;
  }
  *n_out = 0;
  if (n == 0) return TSDF_OK;
  return scan_keys(T_(t), xyz, xyz_dtype, n, mem, make_frame(nullptr, R, trans, tau, 0.0), keys, cap,
                   n_out);
}

int tsdf_evict_level(tsdf_table* t, int32_t level, const int64_t* coords, int64_t n, double* tsdf,
                     double* weight, double* s2, float* color) {
  NEED(t);
  T_(t)->version++;
  return evict_blocks(T_(t), level, coords, n, tsdf, weight, s2, color);
}

int tsdf_read_level_blocks(tsdf_table* t, int32_t level, const uint64_t* keys, int64_t n, double* tsdf,
                           double* weight, double* s2, float* color) {
  NEED(t);
  return read_blocks(T_(t), level, keys, n, tsdf, weight, s2, color);
}

int tsdf_import_level(tsdf_table* t, int32_t level, const int64_t* coords, int64_t n,
                      const double* tsdf, const double* weight, const double* s2,
                      const float* color) {
  NEED(t);
  T_(t)->version++;
  return import_blocks(T_(t), level, coords, n, tsdf, weight, s2, color);
}

int tsdf_integrate_points(tsdf_table* t, const void* xyz, int32_t xyz_dtype, const void* rgb,
                          int32_t rgb_dtype, int64_t n, int32_t mem, const double* R,
                          const double* trans, double tau, double weight_cap,
                          tsdf_integration_stats* stats) {
  NEED(t);
  T_(t)->version++;
  if (xyz_dtype < 0 || xyz_dtype > 1 || (rgb && (rgb_dtype < 0 || rgb_dtype > 2))) {
    set_error("unsupported dtype");
    return TSDF_EVALUE;
  }
  IntegrationStats st;
  int s = integrate_points(T_(t), xyz, xyz_dtype, rgb, rgb_dtype, n, mem,
                           make_frame(nullptr, R, trans, tau, weight_cap), &st);
  memcpy(stats, &st, sizeof(st));
  return s;
}

int tsdf_allocate_for_measurement(tsdf_table* t, const double* origin, const double* p,
                                  double tau, int64_t* handles, int64_t max_out, int64_t* n_out) {
  NEED(t);
  T_(t)->version++;
  return allocate_for_measurement(T_(t), origin, p, tau, handles, max_out, n_out);
}

int tsdf_apply_merges(tsdf_table* t, double sigma, double min_frac, double min_w,
                      int32_t all_levels, tsdf_merge_stats* stats) {
  NEED(t);
  T_(t)->version++;
  MergeStats st;
  int s = apply_merges(T_(t), sigma, min_frac, min_w, all_levels, &st);
  stats->candidates = st.candidates;
  stats->merged = st.merged;
  return s;
}

int tsdf_extract_mesh(tsdf_table* t, double iso, double eps, tsdf_mesh* out) {
  NEED(t);
  memset(out, 0, sizeof(*out));
  if (eps < 0) eps = 0.25 * (T_(t)->d.edge / kFineSide);
  MeshOut m{};
  int s = extract_mesh(T_(t), iso, eps, &m);
  out->vertices = m.v;
  out->normals = m.n;
  out->colors = m.c;
  out->num_vertices = m.nv;
  out->triangles = m.tri;
  out->num_triangles = m.nt;
  return s;
}

int tsdf_extract_mesh_begin(tsdf_table* t, double iso, double eps, int64_t* num_vertices,
                            int64_t* num_triangles) {
  NEED(t);
  if (eps < 0) eps = 0.25 * (T_(t)->d.edge / kFineSide);
  return extract_mesh_begin(T_(t), iso, eps, num_vertices, num_triangles);
}

int tsdf_extract_mesh_read(tsdf_table* t, double* vertices, double* normals, double* colors,
                           int64_t* triangles) {
  NEED(t);
  return extract_mesh_read(T_(t), vertices, normals, colors, triangles);
}

void tsdf_mesh_free(tsdf_mesh* m) {
  if (!m) return;
  MeshOut o{m->vertices, m->normals, m->colors, m->num_vertices, m->triangles, m->num_triangles};
  mesh_free(&o);
  memset(m, 0, sizeof(*m));
}

static void to_c_mesh(const MeshOut& m, tsdf_mesh* out) {
  out->vertices = m.v;
  out->normals = m.n;
  out->colors = m.c;
  out->num_vertices = m.nv;
  out->triangles = m.tri;
  out->num_triangles = m.nt;
}

int tsdf_mesh_block_summary(tsdf_table* t, uint64_t* keys, int32_t* levels, uint8_t* observed,
                            double* tsdf_lo, double* tsdf_hi, int64_t cap, int64_t* n_out) {
  NEED(t);
  return mesh_block_summary(T_(t), keys, levels, observed, tsdf_lo, tsdf_hi, cap, n_out);
}

int tsdf_mesh_emit_keys(tsdf_table* t, const uint64_t* keys, const int64_t* level_counts, double iso,
                        tsdf_mesh* raw) {
  NEED(t);
  memset(raw, 0, sizeof(*raw));
  MeshOut m{};
  int s = mesh_emit_keys(T_(t), keys, level_counts, iso, &m);
  to_c_mesh(m, raw);
  return s;
}

int tsdf_mesh_finish(const double* v, const double* n, const double* c, int64_t nv, const int64_t* tri,
                     int64_t nt, double block_edge, double eps, tsdf_mesh* out) {
  memset(out, 0, sizeof(*out));
  if (eps < 0) eps = 0.25 * (block_edge / kFineSide);
  MeshOut m{};
  int s = mesh_finish(v, n, c, nv, tri, nt, block_edge, eps, &m);
  to_c_mesh(m, out);
  return s;
}

int tsdf_find_batch(tsdf_table* t, const int64_t* coords, int64_t n, int64_t* handles,
                    int32_t* levels, uint8_t* found) {
  NEED(t);
  return find_batch(T_(t), coords, n, handles, levels, found);
}

int tsdf_insert(tsdf_table* t, const int64_t* coord, int32_t level, int64_t* handle) {
  NEED(t);
  T_(t)->version++;
  return insert_block(T_(t), coord, level, handle);
}

int tsdf_remove(tsdf_table* t, const int64_t* coord, int32_t* level, double* tsdf,
                double* weight, double* s2, float* color) {
  NEED(t);
  T_(t)->version++;
  return remove_block(T_(t), coord, level, tsdf, weight, s2, color);
}

int tsdf_read_block(tsdf_table* t, const int64_t* coord, int32_t* level, double* tsdf,
                    double* weight, double* s2, float* color) {
  NEED(t);
  return read_block(T_(t), coord, level, tsdf, weight, s2, color);
}

int tsdf_write_block(tsdf_table* t, const int64_t* coord, const double* tsdf,
                     const double* weight, const double* s2, const float* color) {
  NEED(t);
  T_(t)->version++;
  return write_block(T_(t), coord, tsdf, weight, s2, color);
}

int tsdf_table_probe_stats(tsdf_table* t, int64_t* out, double* mean_probe) {
  NEED(t);
  ProbeStats p;
  if (int s = probe_stats(T_(t), &p)) return s;
  out[0] = p.live;
  out[1] = p.tombstones;
  out[2] = p.max_probe;
  out[3] = p.rehashes;
  if (mean_probe) *mean_probe = p.mean_probe;
  return TSDF_OK;
}

int tsdf_probe_length(tsdf_table* t, const int64_t* coords, int64_t n, int32_t* out) {
  NEED(t);
  return probe_length(T_(t), coords, n, out);
}

int tsdf_table_compact(tsdf_table* t) {
  NEED(t);
  T_(t)->version++;
  return rehash_table(T_(t));
}

int tsdf_live_count(tsdf_table* t, int32_t level, int64_t* n) {
  NEED(t);
  return live_count(T_(t), level, n);
}

int tsdf_export_level(tsdf_table* t, int32_t level, int64_t max_blocks, int64_t* coords,
                      int64_t* handles, double* tsdf, double* weight, double* s2, float* color,
                      int64_t* n_out) {
  NEED(t);
  return export_level(T_(t), level, max_blocks, coords, handles, tsdf, weight, s2, color, n_out);
}

const char* tsdf_last_error(void) { return last_error(); }

int64_t tsdf_kernel_launches(tsdf_table* t) { return t && t->impl ? (int64_t)t->impl->launches : 0; }

int64_t tsdf_table_slots(tsdf_table* t) { return t && t->impl ? (int64_t)t->impl->slots : 0; }

int tsdf_device_info(int32_t* major, int32_t* minor, int32_t* sms) {
  int dev = 0, n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess || n == 0) {
    set_error("no CUDA device visible");
    return TSDF_ECUDA;
  }
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(major, cudaDevAttrComputeCapabilityMajor, dev);
  cudaDeviceGetAttribute(minor, cudaDevAttrComputeCapabilityMinor, dev);
  cudaDeviceGetAttribute(sms, cudaDevAttrMultiProcessorCount, dev);
  return TSDF_OK;
}

}  // extern "C"

extern "C" {

int tsdf_dda_blocks(const double* origins, const double* endpoints, int64_t n, double edge,
                    int32_t batch_cap, int64_t** ray_ids, int64_t** coords, int64_t* nrows) {
  return dda_trace(origins, endpoints, n, edge, batch_cap, ray_ids, coords, nrows);
}

int tsdf_merge_candidates(tsdf_table* t, double sigma, double min_frac, double min_w,
                          int64_t** coords, int64_t* n_out) {
  NEED(t);
  return merge_candidates(T_(t), sigma, min_frac, min_w, coords, n_out);
}

int tsdf_collapse_vertices(const double* v, const double* n, const double* c, int64_t nv,
                           const int64_t* tri, int64_t nt, double eps, tsdf_mesh* out) {
  memset(out, 0, sizeof(*out));
  MeshOut m{};
  int s = collapse_vertices(v, n, c, nv, tri, nt, eps, &m);
  out->vertices = m.v;
  out->normals = m.n;
  out->colors = m.c;
  out->num_vertices = m.nv;
  out->triangles = m.tri;
  out->num_triangles = m.nt;
  return s;
}

void tsdf_free(void* p) { free(p); }

}  // extern "C"

extern "C" {

int tsdf_profile_enable(tsdf_table* t, int32_t on) {
  NEED(t);
  T_(t)->prof = on != 0;
  if (!on) {
    prof_collect(T_(t));
  }
  return TSDF_OK;
}

int tsdf_profile_read(tsdf_table* t, int32_t reset, int32_t max_entries, char* names,
                      int32_t name_stride, double* ms, int64_t* counts, int32_t* n_out) {
  NEED(t);
  Table* T = T_(t);
  if (int s = prof_collect(T)) return s;
  int i = 0;
  for (const auto& kv : T->prof_acc) {
    if (i < max_entries) {
      strncpy(names + (size_t)i * name_stride, kv.first.c_str(), name_stride - 1);
      names[(size_t)i * name_stride + name_stride - 1] = 0;
      ms[i] = kv.second.ms;
      counts[i] = kv.second.count;
    }
    i++;
  }
  *n_out = i;
  if (reset) T->prof_acc.clear();
  return TSDF_OK;
}

}  // extern "C"

extern "C" {

int tsdf_integrate_depth_batch(tsdf_table* t, int32_t n_frames, const void* const* depth,
                               int32_t depth_dtype, const void* const* rgb, int32_t rgb_dtype,
                               int32_t height, int32_t width, int32_t mem, const double* K,
                               const double* R, const double* trans, double tau,
                               double weight_cap, tsdf_integration_stats* stats,
                               int32_t* n_done) {
  NEED(t);
  T_(t)->version++;
  if (n_frames <= 0) {
    *n_done = 0;
    return TSDF_OK;
  }
  if (depth_dtype < 0 || depth_dtype > 3 || (rgb && (rgb_dtype < 0 || rgb_dtype > 2))) {
    set_error("unsupported dtype");
    return TSDF_EVALUE;
  }
  std::vector<DepthArgs> args(n_frames);
  for (int i = 0; i < n_frames; i++) {
    if (K[4 * i] <= 0 || K[4 * i + 1] <= 0) {
      set_error("focal lengths must be positive");
      return TSDF_EDATASET;
    }
    args[i] = DepthArgs{depth[i], depth_dtype, rgb ? rgb[i] : nullptr, rgb_dtype, height, width,
                        mem, make_frame(K + 4 * i, R + 9 * i, trans + 3 * i, tau, weight_cap)};
  }
  std::vector<IntegrationStats> st(n_frames);
  int done = 0;
  int s = integrate_depth_batch(T_(t), n_frames, args.data(), st.data(), &done);
  for (int i = 0; i < n_frames; i++) memcpy(&stats[i], &st[i], sizeof(st[i]));
  *n_done = done;
  return s;
}

int tsdf_integrate_depth_window(tsdf_table* t, int32_t n_frames, const void* const* depth,
                               int32_t depth_dtype, const void* const* rgb, int32_t rgb_dtype,
                               int32_t height, int32_t width, int32_t mem, const double* K,
                               const double* R, const double* trans, double tau,
                               double weight_cap, tsdf_integration_stats* stats,
                               int32_t* n_done, double sigma, double min_frac, double min_w,
                               int32_t all_levels, double fill_limit,
                               tsdf_merge_stats* merge_stats) {
  NEED(t);
  T_(t)->version++;
  if (n_frames <= 0) {
    *n_done = 0;
    return TSDF_OK;
  }
  if (depth_dtype < 0 || depth_dtype > 3 || (rgb && (rgb_dtype < 0 || rgb_dtype > 2))) {
    set_error("unsupported dtype");
    return TSDF_EVALUE;
  }
  std::vector<DepthArgs> args(n_frames);
  for (int i = 0; i < n_frames; i++) {
    if (K[4 * i] <= 0 || K[4 * i + 1] <= 0) {
      set_error("focal lengths must be positive");
      return TSDF_EDATASET;
    }
    args[i] = DepthArgs{depth[i], depth_dtype, rgb ? rgb[i] : nullptr, rgb_dtype, height, width,
                        mem, make_frame(K + 4 * i, R + 9 * i, trans + 3 * i, tau, weight_cap)};
  }
  std::vector<IntegrationStats> st(n_frames);
  int done = 0;
  MergeArgs ma{sigma, min_frac, min_w, all_levels, fill_limit};
  MergeStats ms{0, 0};
  int s = integrate_depth_window(T_(t), n_frames, args.data(), st.data(), &done,
                                 merge_stats ? &ma : nullptr, &ms);
  if (merge_stats) {
    merge_stats->candidates = ms.candidates;
    merge_stats->merged = ms.merged;
  }
  for (int i = 0; i < n_frames; i++) memcpy(&stats[i], &st[i], sizeof(st[i]));
  *n_done = done;
  return s;
}

int tsdf_depth_window_frames(tsdf_table* t, int32_t n_frames, const void* const* depth,
                             int32_t depth_dtype, const void* const* rgb, int32_t rgb_dtype,
                             int32_t height, int32_t width, int32_t mem, const double* K,
                             const double* R, const double* trans, double tau, double weight_cap,
                             int32_t ray_rank, int32_t ray_world, uint64_t* caps) {
  NEED(t);
  if (n_frames <= 0) {
    set_error("a window needs at least one frame");
    return TSDF_EVALUE;
  }
  if (depth_dtype < 0 || depth_dtype > 3 || (rgb && (rgb_dtype < 0 || rgb_dtype > 2))) {
    set_error("unsupported dtype");
    return TSDF_EVALUE;
  }
  std::vector<DepthArgs> args(n_frames);
  for (int i = 0; i < n_frames; i++) {
    if (K[4 * i] <= 0 || K[4 * i + 1] <= 0) {
      set_error("focal lengths must be positive");
      return TSDF_EDATASET;
    }
    args[i] = DepthArgs{depth[i], depth_dtype, rgb ? rgb[i] : nullptr, rgb_dtype, height, width,
                        mem, make_frame(K + 4 * i, R + 9 * i, trans + 3 * i, tau, weight_cap)};
  }
  return depth_window_frames(T_(t), n_frames, args.data(), ray_rank, ray_world, caps);
}

int tsdf_depth_window_walk(tsdf_table* t, const uint64_t* caps, uint64_t* exchange, int64_t bucket_cap) {
  NEED(t);
  return depth_window_walk(T_(t), caps, exchange, bucket_cap);
}

int tsdf_depth_window_update(tsdf_table* t, const uint64_t* received, int32_t world, int64_t bucket_cap,
                             double sigma, double min_frac, double min_w, int32_t all_levels,
                             tsdf_integration_stats* stats, tsdf_merge_stats* merge_stats) {
  NEED(t);
  T_(t)->version++;
  const int B = T_(t)->win.B;
  std::vector<IntegrationStats> st(std::max(B, 1));
  MergeArgs ma{sigma, min_frac, min_w, all_levels, 0.0};
  MergeStats ms{0, 0};
  int s = depth_window_update(T_(t), received, world, bucket_cap, &ma, st.data(), &ms);
  for (int i = 0; i < B; i++) memcpy(&stats[i], &st[i], sizeof(st[i]));
  if (merge_stats) {
    merge_stats->candidates = ms.candidates;
    merge_stats->merged = ms.merged;
  }
  return s;
}

}  // extern "C"

extern "C" int tsdf_work_totals(tsdf_table* t, int64_t* out, int32_t reset) {
  NEED(t);
  for (int i = 0; i < 16; i++) out[i] = T_(t)->acc[i];
  if (reset)
    for (int i = 0; i < 16; i++) T_(t)->acc[i] = 0;
  return TSDF_OK;
}
