/*
 * tsdf_b200.h -- C ABI of the B200 (sm_100a) TSDF-fusion hot path.
 *
 * Drop-in boundary for the reference package's hot path
 * (/root/reference/pkg/src/tsdfusion).  Plain pointers and sizes only; no
 * torch or CUDA C++ types.  Every entry point returns an int status whose
 * values are the reference's FusionError exit codes (errors.py:4-37):
 *   0 ok, 2 ConfigError, 3 DatasetError, 4 CapacityError, 5 NotFoundError,
 *   6 FormatError, 8 ValueError (Python builtin), 9 CUDA/driver failure.
 * tsdf_last_error() returns a message for the calling thread's last failure.
 *
 * Threading: one host thread per table; every call enqueues on the table's
 * CUDA stream and returns after its results are on the host.
 * Ownership: the table owns all device memory; callers own input buffers
 * for the duration of a call.  `mem` says where input buffers live
 * (TSDF_MEM_HOST: pageable/pinned host memory, copied inside the call;
 * TSDF_MEM_DEVICE: device pointers, read in place on the table's stream:
 * their contents must be complete when the call is made -- a buffer written
 * by work on another stream, e.g. an NCCL collective on torch's current
 * stream, needs that stream synchronised (or an event waited on) first).
 */
#ifndef TSDF_B200_H
#define TSDF_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TSDF_OK 0
#define TSDF_ECONFIG 2
#define TSDF_EDATASET 3
#define TSDF_ECAPACITY 4
#define TSDF_ENOTFOUND 5
#define TSDF_EFORMAT 6
#define TSDF_EVALUE 8
#define TSDF_ECUDA 9

/* element types of input buffers */
#define TSDF_F64 0
#define TSDF_F32 1
#define TSDF_U8 2  /* colour channels: value/255.0, as datasets.py:118,163 */
#define TSDF_U16 3 /* depth: raw units / depth_scale (tsdf_table_set_depth_scale) */

#define TSDF_MEM_HOST 0
#define TSDF_MEM_DEVICE 1

typedef struct tsdf_table tsdf_table;

/* IntegrationStats (reference integrate.py:42-50) */
typedef struct {
  int64_t measurements;
  int64_t skipped_invalid;
  int64_t blocks_allocated;
  int64_t blocks_touched;
  int64_t voxels_updated;
  int64_t observations;
  int32_t no_valid_warning; /* "frame has no valid depth pixels" */
  int32_t pad;
} tsdf_integration_stats;

/* MergeStats (reference adapt.py:20-23) */
typedef struct {
  int64_t candidates;
  int64_t merged;
} tsdf_merge_stats;

/* Mesh (reference meshing.py:39-59); arrays owned by the library until
 * tsdf_mesh_free(). */
typedef struct {
  double *vertices;   /* nv x 3, metres */
  double *normals;    /* nv x 3, unit */
  double *colors;     /* nv x 3, [0, 1] */
  int64_t num_vertices;
  int64_t *triangles; /* nt x 3 */
  int64_t num_triangles;
} tsdf_mesh;

/* HashTable(n_hash, bucket_capacity, overflow_capacity, block_edge,
 * heap_capacities) -- reference hashgrid.py:142-165.  `cuda_stream` may be
 * NULL (the table creates its own non-blocking stream). */
int tsdf_table_create(int64_t n_hash, int32_t bucket_capacity, int32_t overflow_capacity,
                      double block_edge, int32_t n_levels, const int64_t *heap_capacities,
                      void *cuda_stream, tsdf_table **out);
int tsdf_table_destroy(tsdf_table *t);
/* drop every block (fresh table, same sizes) */
int tsdf_table_reset(tsdf_table *t);
/* block-key-hash sharding: this table owns only keys with
 * owner(key) == rank (world > 1); DESIGN.md "Multi-GPU". */
int tsdf_table_set_shard(tsdf_table *t, int32_t rank, int32_t world);
/* Units of raw uint16 depth (depth_dtype 3) for the following depth calls:
 * z = raw / depth_scale in f64, the conversion the reference's reader does
 * on the host (datasets.py:108-113, config.py:42 default 5000); default 1.0.
 * Lets a dataset's 16-bit PNG depth cross PCIe at 2 B/px. */
int tsdf_table_set_depth_scale(tsdf_table *t, double depth_scale);

/* Ray-sharded merge window for block-key-hash shards: B depth
 * frames and their merge pass in three stream-ordered calls with one
 * collective between consecutive calls and a single host synchronisation
 * (in _update).  Inputs as tsdf_integrate_depth_window.
 *  _frames: the pixel passes of all frames (d_ray and the min/max pyramid in
 *           full; the FP64 segment-end span that sets dda.py:63's lock-step
 *           cap only over this rank's tiles); writes the B partial caps to
 *           `caps` (device u64[B]).  Caller: all-reduce MAX of caps.
 *  _walk:   with the reduced caps, this rank's tiles of rays of every frame
 *           walk and write each block key they meet once per frame into the
 *           device exchange buffer: for owner o, stride = B * (bucket_cap + 1)
 *           words, [o*stride + i] = count of frame i, [o*stride + B + i*cap
 *           + j] = key j.  Caller: all-to-all of the buffer (equal splits of
 *           stride words).
 *  _update: `received` (same layout, source-major): per frame in order,
 *           insert the keys this rank owns, commit the new blocks, update the
 *           voxels; then one merge pass (sigma > 0); per-frame stats[B] of
 *           this shard.  A bucket count above bucket_cap is a CapacityError. */
int tsdf_depth_window_frames(tsdf_table *t, int32_t n_frames, const void *const *depth,
                             int32_t depth_dtype, const void *const *rgb, int32_t rgb_dtype,
                             int32_t height, int32_t width, int32_t mem, const double *K,
                             const double *R, const double *trans, double tau, double weight_cap,
                             int32_t ray_rank, int32_t ray_world, uint64_t *caps);
int tsdf_depth_window_walk(tsdf_table *t, const uint64_t *caps, uint64_t *exchange, int64_t bucket_cap);
int tsdf_depth_window_update(tsdf_table *t, const uint64_t *received, int32_t world, int64_t bucket_cap,
                             double sigma, double min_frac, double min_w, int32_t all_levels,
                             tsdf_integration_stats *stats, tsdf_merge_stats *merge_stats);

/* the CUDA stream every call of this table is ordered on (for callers that
 * interleave their own work, e.g. collectives, with the table's) */
int tsdf_table_stream(tsdf_table *t, void **stream);
/* a counter bumped by every call that can change the map (host caches of
 * heap contents, e.g. BlockHeap.tsdf, are valid while it is unchanged) */
int tsdf_table_version(tsdf_table *t, uint64_t *version);

/* LiDAR hot-block update order (integrate_pointcloud, integrate.py:175-252).
 * TSDF_LIDAR_ORDERED (default): every voxel applies its observations in ray
 * order, the reference's _apply_batch arrival order (integrate.py:92-119):
 * bit-identical state.  TSDF_LIDAR_CHUNKED: blocks crossed by more than 256
 * near rays fold each voxel's observations in groups of 512 rays into partial
 * Welford states, merged with the voxel's prior state in ray order by Chan's
 * pairwise formula -- the same mean / sum of squared deviations up to
 * rounding (the north star's 1e-4 relative TSDF / variance tolerance), exact
 * weights and block keys, and levels audited by tsdf_table_merge_audit.
 * Only without a weight cap; capped calls always run ordered. */
#define TSDF_LIDAR_ORDERED 0
#define TSDF_LIDAR_CHUNKED 1
int tsdf_table_set_lidar_mode(tsdf_table *t, int32_t mode);
/* Merge passes so far: level decisions whose block mean variance lay within
 * 1e-6 relative of sigma (adapt.py:41-72) -- the only decisions rounding
 * differences of the chunked mode could flip.  0 = levels provably exact. */
int tsdf_table_merge_audit(tsdf_table *t, int64_t *near_threshold);

/* integrate_depth(table, DepthFrame, tau, weight_cap) -- integrate.py:255-342.
 * depth: H*W z-depth in metres (0 / NaN invalid); rgb: H*W*3 or NULL.
 * K = (fx, fy, cx, cy); R row-major 3x3 and t (3) are world-from-sensor
 * (geometry.py:12-34). */
int tsdf_integrate_depth(tsdf_table *t, const void *depth, int32_t depth_dtype, const void *rgb,
                         int32_t rgb_dtype, int32_t height, int32_t width, int32_t mem,
                         const double *K, const double *R, const double *trans, double tau,
                         double weight_cap, tsdf_integration_stats *stats);

/* Ray-sharded depth integration for block-key-hash shards (
 * the multi-GPU split of integrate.py:255-342).  Step 1 (walk): this rank
 * walks the tiles of rays t with t % ray_world == ray_rank and writes every
 * block key it meets once (packed, 21 bits per axis) to its owner's bucket:
 * buckets is DEVICE memory [shard_world][bucket_cap], counts (host,
 * shard_world entries) receives the per-owner key counts; stats gets the
 * rank-invariant fields (measurements, skipped_invalid).  The caller
 * exchanges buckets with an all-to-all.  Step 2 (keys): the keys this rank
 * owns, gathered from every rank (DEVICE memory, duplicates allowed), are
 * inserted -- touched once each --, new blocks committed, and the voxel
 * update of the same frame runs; stats gets the block-partitioned fields.
 * The frame's buffers (and a device-resident colour image) must stay valid
 * until step 2 returns.  ray_world == 1 with an unsharded table equals
 * tsdf_integrate_depth. */
int tsdf_integrate_depth_walk(tsdf_table *t, const void *depth, int32_t depth_dtype,
                              const void *rgb, int32_t rgb_dtype, int32_t height, int32_t width,
                              int32_t mem, const double *K, const double *R, const double *trans,
                              double tau, double weight_cap, int32_t ray_rank, int32_t ray_world,
                              uint64_t *buckets, int64_t bucket_cap, int64_t *counts,
                              tsdf_integration_stats *stats);
int tsdf_integrate_depth_keys(tsdf_table *t, const uint64_t *keys, int64_t n,
                              tsdf_integration_stats *stats);

/* n_frames depth frames of one merge window (same size/dtypes), enqueued
 * back to back with one host synchronisation.  Per-frame K (4), R (9) and
 * trans (3) are packed consecutively.  Semantically identical to calling
 * tsdf_integrate_depth per frame: on an error at frame i the frames after
 * it leave the table untouched, *n_done = i and the error is returned. */
int tsdf_integrate_depth_batch(tsdf_table *t, int32_t n_frames, const void *const *depth,
                               int32_t depth_dtype, const void *const *rgb, int32_t rgb_dtype,
                               int32_t height, int32_t width, int32_t mem, const double *K,
                               const double *R, const double *trans, double tau,
                               double weight_cap, tsdf_integration_stats *stats,
                               int32_t *n_done);

/* One merge window (pipeline.py:88-137): tsdf_integrate_depth_batch's
 * frames followed -- when merge_stats is not NULL and every frame
 * succeeded -- by one tsdf_apply_merges pass (sigma, min_frac, min_w,
 * all_levels), all enqueued back to back with a single host
 * synchronisation (sigma <= 0: no merge pass).  fill_limit > 0 (with
 * merge_stats): the window stops
 * after the first frame i < n_frames - 1 that brings a level's occupancy
 * to fill_limit (the engine's stream-out mark); *n_done = i + 1, the
 * merge is not run and TSDF_OK is returned. */
int tsdf_integrate_depth_window(tsdf_table *t, int32_t n_frames, const void *const *depth,
                                int32_t depth_dtype, const void *const *rgb, int32_t rgb_dtype,
                                int32_t height, int32_t width, int32_t mem, const double *K,
                                const double *R, const double *trans, double tau,
                                double weight_cap, tsdf_integration_stats *stats,
                                int32_t *n_done, double sigma, double min_frac, double min_w,
                                int32_t all_levels, double fill_limit,
                                tsdf_merge_stats *merge_stats);

/* integrate_pointcloud(table, PointCloudFrame, tau, weight_cap) --
 * integrate.py:175-252.  xyz: n*3 sensor-frame points; rgb n*3 or NULL. */
int tsdf_integrate_points(tsdf_table *t, const void *xyz, int32_t xyz_dtype, const void *rgb,
                          int32_t rgb_dtype, int64_t n, int32_t mem, const double *R,
                          const double *trans, double tau, double weight_cap,
                          tsdf_integration_stats *stats);

/* allocate_for_measurement(table, origin, p, tau) -- integrate.py:143-161.
 * Writes up to max_out handles in traversal order; *n_out = total count. */
int tsdf_allocate_for_measurement(tsdf_table *t, const double *origin, const double *p,
                                  double tau, int64_t *handles, int64_t max_out, int64_t *n_out);

/* apply_merges(table, sigma_threshold, min_eligible_fraction,
 * min_mean_weight) -- adapt.py:119-136.  all_levels = 0 reproduces the
 * reference (level 0 -> 1 only); 1 enables the labelled multi-level
 * extension (every level L -> L+1, candidates snapshotted per pass). */
int tsdf_apply_merges(tsdf_table *t, double sigma_threshold, double min_eligible_fraction,
                      double min_mean_weight, int32_t all_levels, tsdf_merge_stats *stats);

/* extract_mesh(table, iso, collapse_epsilon) -- meshing.py:412-487.
 * collapse_epsilon < 0 selects the default 0.25 * voxel_size(0). */
int tsdf_extract_mesh(tsdf_table *t, double iso, double collapse_epsilon, tsdf_mesh *out);
void tsdf_mesh_free(tsdf_mesh *m);
/* Two-phase extract_mesh: _begin runs the extraction and keeps the mesh on
 * the device (returns its sizes); _read copies it straight into caller-owned
 * host arrays (vertices / normals / colours nv x 3 f64, triangles nt x 3
 * i64) -- no intermediate host copy.  Same mesh as tsdf_extract_mesh. */
int tsdf_extract_mesh_begin(tsdf_table *t, double iso, double eps, int64_t *num_vertices,
                            int64_t *num_triangles);
int tsdf_extract_mesh_read(tsdf_table *t, double *vertices, double *normals, double *colors,
                           int64_t *triangles);

/* Nearest-neighbour distance from every query point to the tree point set
 * (FP64, sqrt((dx*dx + dy*dy) + dz*dz), exact): the cKDTree(tree).query(q,
 * k=1)[0] of eval_reconstruction (metrics.py:63-64).  Points are n x 3 f64;
 * mem says where tree, query and dist live (TSDF_MEM_HOST / _DEVICE).  A
 * non-finite query gets NaN; a non-finite tree point is TSDF_EVALUE.
 * Table-independent; runs on cuda_stream (NULL: legacy default stream). */
int tsdf_nn_distance(const double *tree, int64_t n_tree, const double *query, int64_t n_query,
                     int32_t mem, double *dist, void *cuda_stream);

/* build_quadtree(image, contrast_threshold, min_pixel) -- quadtree.py:94-109.
 * image: H*W*3 f64 (host or device per mem).  Writes the leaves in the
 * reference's breadth-first order as (x0, y0, w, h) int32 quadruples and
 * their contrasts; both outputs are host arrays with room for H*W leaves. */
int tsdf_quadtree_build(const double *image, int32_t height, int32_t width, int32_t mem,
                        double threshold, int32_t min_pixel, int32_t *leaves_out,
                        double *contrast_out, int64_t *n_leaves, void *cuda_stream);
/* seed_splats(leaves, DepthFrame) -- quadtree.py:112-148.  One splat per
 * leaf with valid depth at its centre: world position (3 f64), scale
 * w * d / fx, mean colour (0.5 grey without rgb); valid_out[i] says whether
 * leaf i produced a splat.  depth: f64 / f32 metres or u16 raw / depth_scale;
 * rgb: f64 / f32 in [0, 1] or u8 (/ 255) or NULL.  Outputs are host arrays. */
int tsdf_seed_splats(const int32_t *leaves, int64_t n, const void *depth, int32_t depth_dtype,
                     double depth_scale, const void *rgb, int32_t rgb_dtype, int32_t height,
                     int32_t width, int32_t mem, const double *K, const double *R,
                     const double *trans, double *pos_out, double *scale_out, double *color_out,
                     uint8_t *valid_out, void *cuda_stream);

/* HashTable.find_batch (hashgrid.py:300-331) */
int tsdf_find_batch(tsdf_table *t, const int64_t *coords, int64_t n, int64_t *handles,
                    int32_t *levels, uint8_t *found);
/* HashTable.insert (hashgrid.py:212-251): idempotent, zero-initialised */
int tsdf_insert(tsdf_table *t, const int64_t *coord, int32_t level, int64_t *handle);
/* HashTable.remove (hashgrid.py:253-283): returns the payload (any pointer
 * may be NULL); buffers hold nvox(level) voxels, colour interleaved rgb */
int tsdf_remove(tsdf_table *t, const int64_t *coord, int32_t *level, double *tsdf,
                double *weight, double *s2, float *color);
/* BlockHeap.payload / write_payload (hashgrid.py:115-133) by coordinate */
int tsdf_read_block(tsdf_table *t, const int64_t *coord, int32_t *level, double *tsdf,
                    double *weight, double *s2, float *color);
int tsdf_write_block(tsdf_table *t, const int64_t *coord, const double *tsdf,
                     const double *weight, const double *s2, const float *color);
/* The distinct block keys (packed, 21 bits per axis, sorted) that the
 * allocation of a depth frame / a point scan would touch -- the reference's
 * unique DDA coordinates (integrate.py:203, :289) -- without changing the
 * table.  The capacity tier uses them to stream archived blocks back in
 * before integrating (integrate.py:122-140). */
int tsdf_depth_keys(tsdf_table *t, const void *depth, int32_t depth_dtype, int32_t height,
                    int32_t width, int32_t mem, const double *K, const double *R, const double *trans,
                    double tau, uint64_t *keys, int64_t cap, int64_t *n_out);
int tsdf_scan_keys(tsdf_table *t, const void *xyz, int32_t xyz_dtype, int64_t n, int32_t mem,
                   const double *R, const double *trans, double tau, uint64_t *keys, int64_t cap,
                   int64_t *n_out);

/* Capacity tier (streaming.py stream_out / stream_in, formats.py
 * save_map / load_map): bulk transfer of n blocks of one level in the
 * reference's BlockPayload layout -- tsdf, weight, s2 f64 [n][nvox], colour
 * f32 [n][nvox][3], host memory.  evict removes the blocks (payload out,
 * heap slots freed, TSDF_ENOTFOUND if one is not live at that level, table
 * untouched); import inserts them at `level` with their payload
 * (TSDF_EVALUE if one is already live, TSDF_ECAPACITY on heap / chain
 * exhaustion; either way the table is left as before the call). */
int tsdf_evict_level(tsdf_table *t, int32_t level, const int64_t *coords, int64_t n, double *tsdf,
                     double *weight, double *s2, float *color);
/* the payloads of live blocks of one level given as packed keys, the table
 * unchanged (evict's gather without the removal; TSDF_ENOTFOUND if one is
 * not live at that level) */
int tsdf_read_level_blocks(tsdf_table *t, int32_t level, const uint64_t *keys, int64_t n, double *tsdf,
                           double *weight, double *s2, float *color);
int tsdf_import_level(tsdf_table *t, int32_t level, const int64_t *coords, int64_t n,
                      const double *tsdf, const double *weight, const double *s2,
                      const float *color);

/* BlockHeap.occupied for one level; level -1: HashTable.live_count (every
 * level, one read-back) */
int tsdf_live_count(tsdf_table *t, int32_t level, int64_t *n);
/* all live blocks of a level in canonical (x, y, z) order with their
 * payloads (parity export / save_map).  Call with coords == NULL to get the
 * count in *n_out. */
int tsdf_export_level(tsdf_table *t, int32_t level, int64_t max_blocks, int64_t *coords,
                      int64_t *handles, double *tsdf, double *weight, double *s2, float *color,
                      int64_t *n_out);

/* dda_blocks / dda_blocks_batch (dda.py:8-86) on the device: rows grouped
 * by segment in traversal order; batch_cap = 1 applies the batched
 * variant's global lock-step cap.  *ray_ids / *coords are malloc'd
 * (release with tsdf_free). */
int tsdf_dda_blocks(const double *origins, const double *endpoints, int64_t n,
                    double block_edge, int32_t batch_cap, int64_t **ray_ids, int64_t **coords,
                    int64_t *nrows);
/* select_merge_candidates (adapt.py:61-72): canonical-order coords of the
 * level-0 blocks apply_merges would re-home; *coords malloc'd. */
int tsdf_merge_candidates(tsdf_table *t, double sigma_threshold, double min_eligible_fraction,
                          double min_mean_weight, int64_t **coords, int64_t *n_out);
/* Sharded extraction with a halo (sharding.extract_mesh_halo; the multi-GPU
 * split of extract_mesh, meshing.py:412-487).
 * _block_summary: every live block of this table -- packed key (21 bits per
 * axis), level, observed flag and observed tsdf range (meshing.py:428-438),
 * the inputs of the 27-neighbourhood kept test (:440-456).
 * _emit_keys: Marching Cubes output before the vertex dedup (positions in
 * half-voxel lattice units, unnormalised normals, colours, triangles), in
 * the reference's emission order, for a caller-given kept list: packed keys
 * in canonical order, level_counts[l] at level l, each level's list
 * starting on a 256-block chunk boundary of the map's kept list; every kept
 * block and its 26 live neighbours must be in the table.  Free with
 * tsdf_mesh_free.
 * _finish: the exact dedup, winding fix and epsilon collapse over
 * concatenated _emit_keys outputs (triangle indices offset) -- the mesh
 * tsdf_extract_mesh returns for the whole map (eps < 0: the default). */
int tsdf_mesh_block_summary(tsdf_table *t, uint64_t *keys, int32_t *levels, uint8_t *observed,
                            double *tsdf_lo, double *tsdf_hi, int64_t cap, int64_t *n_out);
int tsdf_mesh_emit_keys(tsdf_table *t, const uint64_t *keys, const int64_t *level_counts, double iso,
                        tsdf_mesh *raw);
int tsdf_mesh_finish(const double *vertices, const double *normals, const double *colors, int64_t nv,
                     const int64_t *triangles, int64_t nt, double block_edge, double epsilon,
                     tsdf_mesh *out);
/* collapse_vertices (meshing.py:502-552) on the device */
int tsdf_collapse_vertices(const double *vertices, const double *normals, const double *colors,
                           int64_t nv, const int64_t *triangles, int64_t nt, double epsilon,
                           tsdf_mesh *out);
void tsdf_free(void *p);

/* diagnostics */
/* per-kernel device time: CUDA events bracket every launch on the table's
 * stream while enabled; tsdf_profile_read returns {name, total ms, launches}
 * per kernel (names: name_stride bytes each). */
int tsdf_profile_enable(tsdf_table *t, int32_t on);
/* work totals since the last reset (out has 16 entries): [0] frames/scans,
 * [1] touched blocks, [2] depth blocks kept by the whole-block band cull,
 * [3] LiDAR near pairs, [4] sum of DDA lock-step caps, [5] reserved,
 * [6] depth blocks passing the near filter, [7] 2x2x2 micro-bricks kept by
 * the band cull, [8] voxels screened (FP32), [9] voxels on the exact FP64
 * path, [10] level-0 4x4x4 sub-bricks kept by the band cull, [11] DDA
 * steps walked, [12..15] reserved */
int tsdf_work_totals(tsdf_table *t, int64_t *out, int32_t reset);
int tsdf_profile_read(tsdf_table *t, int32_t reset, int32_t max_entries, char *names,
                      int32_t name_stride, double *ms, int64_t *counts, int32_t *n_out);
const char *tsdf_last_error(void);
int64_t tsdf_kernel_launches(tsdf_table *t);
int64_t tsdf_table_slots(tsdf_table *t);
/* Block-index health.  Erased entries (remove, evict, capacity rollback)
 * leave tombstones in the open-addressing index; inserts reuse them, and
 * the index is rebuilt without them (tsdf_table_compact, run automatically
 * before an inserting call once they pass a quarter of the slots).  The
 * reference frees its chain entries on remove (hashgrid.py:253-275).
 * out: [0] live entries, [1] tombstones, [2] longest probe sequence of a
 * live key (1 = at its home slot), [3] rebuilds so far; *mean_probe = the
 * average probe length of the live keys. */
int tsdf_table_probe_stats(tsdf_table *t, int64_t *out, double *mean_probe);

/* Replaces HashTable.probe_length (hashgrid.py:194-212), batched: out[j] =
 * index slots examined for coords[j] (host int64 [n][3]) until it resolves,
 * 1 = at its home slot; for an absent key, until the empty slot that proves
 * it absent.  Diagnostics only; the table is unchanged. */
int tsdf_probe_length(tsdf_table *t, const int64_t *coords, int64_t n, int32_t *out);
int tsdf_table_compact(tsdf_table *t);
int tsdf_device_info(int32_t *sm_major, int32_t *sm_minor, int32_t *num_sms);

#ifdef __cplusplus
}
#endif
#endif /* TSDF_B200_H */
