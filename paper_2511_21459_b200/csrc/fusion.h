// Host-side table object and the orchestration entry points behind the C-ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <array>
#include <map>
#include <string>
#include <vector>

#include "tsdf_common.cuh"

namespace tsdf {

struct Buf {
  void* p = nullptr;
  size_t bytes = 0;
};

struct ProfRec {
  const char* name;
  cudaEvent_t start, stop;
};
struct ProfAcc {
  double ms = 0;
  int64_t count = 0;
};

struct Frame {
  double fx, fy, cx, cy;
  double R[9];
  double t[3];
  double tau, weight_cap;
};

// a ray-sharded window between its three calls (fusion.cu "ray-sharded merge windows")
struct WindowState {
  int stage = 0;  // 1 after the frame passes, 2 after the walk
  int B = 0, H = 0, W = 0, ray_rank = 0, ray_world = 1, depth_dtype = 0, rgb_dtype = 0;
  int64_t cap = 0;
  Counters* c = nullptr;
  uint32_t* abort_word = nullptr;
  std::vector<std::array<double, 24>> f;  // FrameDev images (fusion.cu)
  std::vector<Frame> fr;
  std::vector<const void*> dptr, cptr;  // device inputs of each frame
  Buf depth, rgb, dray, pyr;            // staged inputs and per-frame scratch
};

struct Table {
  DevTable d{};
  uint32_t* free_top = nullptr;  // device [kMaxLevels]
  int64_t caps[kMaxLevels] = {0, 0, 0, 0};
  int32_t bucket = 0, overflow = 0;
  uint64_t slots = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  Counters* dcnt = nullptr;  // device
  Counters* hcnt = nullptr;  // pinned host mirror
  // pinned copy of DevTable::n_tomb, refreshed at the end of every call that
  // synchronises; maintain_table() rebuilds the index once it passes slots/4
  unsigned long long* htomb = nullptr;
  uint64_t rehashes = 0;
  size_t l2_window = 0;  // bytes of keys[] under the persisting L2 window (0: none)
  // LiDAR hot-segment mode: 0 = ordered (bit-exact ray order), 1 = chunked
  // (partial Welford states merged by Chan's formula; tsdf_table_set_lidar_mode)
  int lidar_mode = 0;
  // merge-pass audit: level decisions within 1e-6 relative of sigma so far
  uint64_t merge_audit = 0;
  // bumped by every call that can change the map (tsdf_table_version): host
  // snapshots of heap contents stay valid while it is unchanged
  uint64_t version = 0;
  uint32_t call_id = 0;
  double depth_scale = 1.0;  // raw u16 depth units per metre (tsdf_table_set_depth_scale)
  Buf mesh_out;                   // the last extract_mesh_begin result (device)
  int64_t mesh_nv = -1, mesh_nt = 0;
  // scratch (grown on demand, never shrunk)
  Buf in0, in1, dray, dcol, ends, flags, new_list, touched, work, pairs, pairs_alt, cub_tmp,
      ray_len, ray_nhat, ray_src, ray_rgb, block_sums, lists, cand, mesh_scratch;
  Buf cand_l[kMaxLevels];
  Buf batch, pyr, lidar_aux;
  Buf dblk, dmicro, dexact;  // depth update work lists (blocks, micro-bricks, voxels)
  Buf mdev;                  // MergeDev of the last enqueued merge pass
  // canonical allocation order: ranks by key (kept all-zero between uses),
  // for new blocks and for merge candidates, and the sorted candidates
  Buf rank_buf, rank_m, cand_sorted;
  // single-block calls (find / insert / remove / payload): one device staging
  // area and its pinned host twin, so a call is one or two round trips
  Buf blk_dev;
  void* blk_host = nullptr;
  size_t blk_host_bytes = 0;
  Buf lidar_hot;             // LiDAR hot-segment chunk offsets + hit masks
  // depth batches overlap frame k+1's allocation (walk stream) with frame
  // k's voxel update (main stream): per-parity copies of the frame scratch
  // that both sides read
  Buf in0b, in1b, drayb, flagsb, pyrb, touchedb, endsb;
  cudaStream_t walk_stream = nullptr;
  cudaStream_t copy_stream = nullptr;  // H2D of host frames, ahead of the walk stream
  cudaEvent_t ev_copy[2] = {nullptr, nullptr};
  cudaEvent_t ev_start = nullptr, ev_alloc[2] = {nullptr, nullptr}, ev_upd[2] = {nullptr, nullptr};
  cudaStream_t prof_stream = nullptr;  // stream the profiling events go to (null: stream)
  // ray-sharded allocation (multi-GPU): per-frame "emitted" key set and the
  // frame state kept between the walk call and the keys call
  Buf fset;
  struct ShardedFrame {
    bool ready = false;
    int H = 0, W = 0, rgb_dtype = 0;
    const void* rgb = nullptr;  // device colour of the frame (staged or caller-owned)
    Counters* c = nullptr;
    uint32_t* abort_word = nullptr;
    double f[24];               // FrameDev image
  } shf;
  Frame shf_frame{};
  WindowState win;
  Counters* hbatch = nullptr;  // pinned, hbatch_n entries
  int hbatch_n = 0;
  // work accounting for diagnostics: frames, touched, culled-in (depth
  // update work items), near pairs, DDA cap sum, 8-voxel items, then the
  // per-kernel Counters::diag fields
  int64_t acc[16] = {};
  // merge-pass memo: stats are re-evaluated only for dirty blocks while the
  // parameters are unchanged
  bool merge_memo = false;
  double memo_sigma = 0, memo_frac = 0, memo_w = 0;
  int memo_all = 0;
  // kernel launch telemetry: launches of our kernels since creation
  uint64_t launches = 0;
  // optional per-kernel event timing (bench / profiling)
  bool prof = false;
  std::vector<cudaEvent_t> prof_pool;
  size_t prof_used = 0;
  std::vector<ProfRec> prof_recs;
  std::map<std::string, ProfAcc> prof_acc;
};

int prof_begin(Table* T, const char* name);
void prof_end(Table* T, int id);
int prof_collect(Table* T);

struct IntegrationStats {
  int64_t measurements, skipped_invalid, blocks_allocated, blocks_touched, voxels_updated,
      observations;
  int32_t no_valid_warning;
  int32_t pad;
};

struct MergeStats {
  int64_t candidates, merged;
};


void set_error(const std::string& msg);
const char* last_error();
int cuda_status(cudaError_t e, const char* where);
void* grow(Buf& b, size_t bytes);

int table_create(int64_t n_hash, int32_t bucket, int32_t overflow, double block_edge,
                 int32_t n_levels, const int64_t* caps, void* stream, Table** out);
int table_destroy(Table* t);
int table_reset(Table* t);
// rebuild the block index without tombstones (slot ids change; callable only
// between calls); maintain_table() does it when tombstones pass slots / 4
int rehash_table(Table* T);
int maintain_table(Table* T);
struct ProbeStats {
  int64_t live, tombstones, max_probe, rehashes;
  double mean_probe;
};
int probe_stats(Table* T, ProbeStats* out);
int probe_length(Table* T, const int64_t* coords, int64_t n, int32_t* out);

struct DepthArgs {
  const void* depth;
  int depth_dtype;
  const void* rgb;
  int rgb_dtype;
  int H, W, mem;
  Frame f;
};
int integrate_depth_batch(Table* T, int B, const DepthArgs* frames, IntegrationStats* st,
                          int* n_done);
struct MergeArgs {
  double sigma, min_frac, min_w;
  int all_levels;
  double fill_limit;  // > 0: stop after the frame that brings a level to this occupancy
};
int integrate_depth_window(Table* T, int B, const DepthArgs* frames, IntegrationStats* st,
                           int* n_done, const MergeArgs* merge, MergeStats* mst);
int integrate_depth_walk(Table* T, const DepthArgs& a, int ray_rank, int ray_world,
                         uint64_t* buckets, uint64_t bucket_cap, int64_t* counts,
                         IntegrationStats* st);
int integrate_depth_keys(Table* T, const uint64_t* keys, int64_t n, IntegrationStats* st);
int depth_window_frames(Table* T, int B, const DepthArgs* frames, int ray_rank, int ray_world,
                        uint64_t* caps);
int depth_window_walk(Table* T, const uint64_t* caps, uint64_t* exch, int64_t cap);
int depth_window_update(Table* T, const uint64_t* recv, int world, int64_t cap, const MergeArgs* merge,
                        IntegrationStats* st, MergeStats* mst);
int depth_keys(Table* T, const DepthArgs& a, uint64_t* keys, int64_t cap, int64_t* n_out);
int scan_keys(Table* T, const void* xyz, int xyz_dtype, int64_t n, int mem, const Frame& fr,
              uint64_t* keys, int64_t cap, int64_t* n_out);
int integrate_depth(Table* T, const void* depth, int depth_dtype, const void* rgb,
                    int rgb_dtype, int H, int W, int mem, const Frame& f,
                    IntegrationStats* st);
int integrate_points(Table* T, const void* xyz, int xyz_dtype, const void* rgb, int rgb_dtype,
                     int64_t n, int mem, const Frame& f, IntegrationStats* st);
int allocate_for_measurement(Table* T, const double* o, const double* p, double tau,
                             int64_t* handles, int64_t max_out, int64_t* n_out);
int apply_merges(Table* T, double sigma, double min_frac, double min_w, int all_levels,
                 MergeStats* st);

// block-level access (payloads, parity export)
int find_batch(Table* T, const int64_t* coords, int64_t n, int64_t* handles, int32_t* levels,
               uint8_t* found);
int insert_block(Table* T, const int64_t* coord, int32_t level, int64_t* handle);
int remove_block(Table* T, const int64_t* coord, int32_t* level, double* tsdf, double* weight,
                 double* s2, float* color);
int read_block(Table* T, const int64_t* coord, int32_t* level, double* tsdf, double* weight,
               double* s2, float* color);
int write_block(Table* T, const int64_t* coord, const double* tsdf, const double* weight,
                const double* s2, const float* color);
int live_count(Table* T, int32_t level, int64_t* n);
int evict_blocks(Table* T, int32_t level, const int64_t* coords, int64_t n, double* tsdf,
                 double* weight, double* s2, float* color);
int import_blocks(Table* T, int32_t level, const int64_t* coords, int64_t n, const double* tsdf,
                  const double* weight, const double* s2, const float* color);
int export_level(Table* T, int32_t level, int64_t max_blocks, int64_t* coords, int64_t* handles,
                 double* tsdf, double* weight, double* s2, float* color, int64_t* n_out);

struct MeshOut {
  double *v, *n, *c;
  int64_t nv;
  int64_t* tri;
  int64_t nt;
};

int dda_trace(const double* origins, const double* endpoints, int64_t n, double edge, int capped,
              int64_t** ray_ids, int64_t** coords, int64_t* nrows);
int merge_candidates(Table* T, double sigma, double min_frac, double min_w, int64_t** coords,
                     int64_t* n_out);
int collapse_vertices(const double* v, const double* n, const double* c, int64_t nv,
                      const int64_t* tri, int64_t nt, double eps, MeshOut* out);

// mesh extraction (mesh.cu)
int extract_mesh(Table* T, double iso, double eps, MeshOut* out);
int extract_mesh_begin(Table* T, double iso, double eps, int64_t* nv, int64_t* nt);
int extract_mesh_read(Table* T, double* v, double* n, double* c, int64_t* tri);
void mesh_free(MeshOut* m);
int read_blocks(Table* T, int32_t level, const uint64_t* keys, int64_t n, double* tsdf, double* weight,
                double* s2, float* color);
int mesh_block_summary(Table* T, uint64_t* keys, int32_t* levels, uint8_t* obs, double* lo,
                       double* hi, int64_t cap, int64_t* n_out);
int mesh_emit_keys(Table* T, const uint64_t* keys, const int64_t* level_counts, double iso,
                   MeshOut* out);
int mesh_finish(const double* v, const double* n, const double* c, int64_t nv, const int64_t* tri,
                int64_t nt, double edge, double eps, MeshOut* out);

}  // namespace tsdf
