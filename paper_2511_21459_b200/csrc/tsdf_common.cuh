// Device-side data structures shared by all TSDF-fusion kernels (sm_100a).
//
// HBM layout:
//   * block index: flat open-addressing hash table, 2^k slots,
//       keys[slot]  u64  packed block coordinate (21 bits/axis, bit 63 clear)
//       vals[slot]  u32  handle | level << 29   (PENDING while being created)
//       stamp[slot] u32  id of the last integration call that touched it
//     ~16 B/slot, sized 2x the total heap capacity -> L2-resident for the
//     configs we run (1M slots = 16 MB of the 126 MB L2).
//   * per-level slab heaps, SoA, zero whenever free:
//       tsdf f64[cap*nvox], s2 f64[cap*nvox], weight f32[cap*nvox],
//       color f32[3][cap*nvox]  (r, g, b planes)
//     voxel order inside a block is x-slowest / z-fastest
//     (reference hashgrid.py:357-367), so a warp reads 32 consecutive
//     voxels of one block with one coalesced 256 B (f64) transaction.
//   * per-level LIFO free stacks of handles.
// Reference semantics this mirrors: hashgrid.py:65-354.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace tsdf {

constexpr int kFineSide = 8;
constexpr int kMaxLevels = 4;
constexpr int kHalfUnits = 16;
constexpr uint64_t kEmptyKey = ~0ull;
constexpr uint64_t kTombKey = ~0ull - 1;
constexpr uint32_t kPending = 0xFFFFFFFFu;
constexpr int kLevelShift = 29;
constexpr uint32_t kHandleMask = (1u << kLevelShift) - 1;
constexpr int64_t kCoordBias = 1 << 20;  // 21-bit signed range per axis

// status codes: the reference's FusionError exit codes (errors.py:4-37)
enum Status : int {
  kOk = 0,
  kConfigError = 2,
  kDatasetError = 3,
  kCapacityError = 4,
  kNotFound = 5,
  kFormatError = 6,
  kValueError = 8,
  kCudaError = 9,
};

// device-side error flags (bitmask, OR-ed by kernels)
enum ErrFlag : uint32_t {
  kErrHeapFull = 1u,        // level heap exhausted
  kErrSlotChain = 2u,       // reference bucket+overflow chain limit hit
  kErrCoordRange = 4u,      // block coordinate outside the 21-bit key range
  kErrPairOverflow = 8u,    // (ray, block) pair buffer too small
  kErrTableFull = 16u,      // hash slots exhausted
  kErrMeshOverflow = 32u,   // mesh output buffers too small
  kErrShardRoute = 64u,     // a key reached a shard that does not own it
};

struct DevHeap {
  double* tsdf;
  double* s2;
  float* weight;
  float* color;  // 3 planes of cap*nvox
  uint32_t* free_stack;
  int64_t cap;
  int32_t side, nvox;
};

struct DevTable {
  uint64_t* keys;
  uint32_t* vals;
  uint32_t* stamp;
  int32_t* ref_count;  // per reference slot (n_hash): bucket+chain occupancy
  uint64_t mask;       // slots - 1
  int64_t n_hash;
  int32_t chain_limit;  // bucket_capacity + overflow_capacity
  int32_t n_levels;
  double edge;
  int32_t shard_rank, shard_world;
  // blocks whose voxels changed since the last merge pass
  uint32_t* dirty;       // per slot flag
  uint32_t* dirty_list;  // slots, in first-dirtied order
  unsigned long long* n_dirty;
  // tombstones in keys[] (erased entries): reused by inserts, and the host
  // rebuilds the table once they pass a quarter of the slots (rehash_table)
  unsigned long long* n_tomb;
  DevHeap heap[kMaxLevels];
};

// per-frame min/max pyramid of the measured ray distance (band cull)
constexpr int kMaxPyr = 16;
struct Pyramid {
  float2* lh;  // (lo, hi) per cell
  int32_t n_levels;
  int32_t w[kMaxPyr], h[kMaxPyr];
  int64_t off[kMaxPyr];
};

// per-call device counters (one struct, read back once per call)
struct Counters {
  unsigned long long n_valid;
  unsigned long long n_new;
  unsigned long long n_touched;
  unsigned long long n_work;
  unsigned long long n_pairs;
  unsigned long long voxels_updated;
  unsigned long long observations;
  unsigned long long dda_cap;      // global lock-step cap (dda.py:63)
  unsigned long long zmin_inv;     // max of ~bits(z): a zeroed struct is the identity
  unsigned long long zmax_bits;    // positive doubles order like their bits
  unsigned long long candidates;
  unsigned long long merged;
  unsigned long long mesh_verts;
  unsigned long long mesh_tris;
  unsigned long long aux0, aux1;
  unsigned long long n_sub, n_micro, n_exact;  // depth update work lists
  unsigned long long tiles_done;                // k_depth_frame: finished tiles
  unsigned long long diag[6];      // work diagnostics (see fusion.cu kDiag*)
  uint32_t err;
  uint32_t pad;
  uint32_t free_top[kMaxLevels];
};

// device counters of one merge pass (enqueue_merges)
struct MergeDev {
  unsigned long long n_cand[kMaxLevels];
  unsigned long long n_list;
  unsigned long long n_dirty;  // dirty-list length at the pass (snapshot)
  uint32_t skip;
  uint32_t pad;  // k_merge_apply: 1 = a merged weight was rounded to binary32
  unsigned long long audit;  // level decisions within 1e-6 relative of sigma
};

__host__ __device__ inline uint64_t pack_key(int64_t x, int64_t y, int64_t z) {
  return ((uint64_t)(x + kCoordBias) << 42) | ((uint64_t)(y + kCoordBias) << 21) |
         (uint64_t)(z + kCoordBias);
}
__host__ __device__ inline bool key_in_range(int64_t x, int64_t y, int64_t z) {
  return x >= -kCoordBias && x < kCoordBias && y >= -kCoordBias && y < kCoordBias &&
         z >= -kCoordBias && z < kCoordBias;
}
__host__ __device__ inline void unpack_key(uint64_t k, int64_t* c) {
  c[0] = (int64_t)((k >> 42) & 0x1FFFFF) - kCoordBias;
  c[1] = (int64_t)((k >> 21) & 0x1FFFFF) - kCoordBias;
  c[2] = (int64_t)(k & 0x1FFFFF) - kCoordBias;
}
__host__ __device__ inline bool key_live(uint64_t k) { return (k >> 63) == 0; }

__host__ __device__ inline uint64_t mix64(uint64_t h) {
  h ^= h >> 33;
  h *= 0xff51afd7ed558ccdull;
  h ^= h >> 33;
  h *= 0xc4ceb9fe1a85ec53ull;
  h ^= h >> 33;
  return h;
}

// shard owner of a block key: decorrelated from the slot hash
__host__ __device__ inline int owner_of(uint64_t key, int world) {
  uint64_t z = key + 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  z ^= z >> 31;
  return (int)((z >> 32) % (uint64_t)world);
}

// reference slot: Teschner primes, 64-bit wrap, Euclidean mod (hashgrid.py:30-54)
__host__ __device__ inline int64_t ref_slot(int64_t x, int64_t y, int64_t z, int64_t n_hash) {
  uint64_t h = ((uint64_t)x * 73856093ull) ^ ((uint64_t)y * 19349669ull) ^
               ((uint64_t)z * 83492791ull);
  int64_t r = (int64_t)h % n_hash;
  return r < 0 ? r + n_hash : r;
}

__device__ inline uint32_t make_val(uint32_t handle, int level) {
  return handle | ((uint32_t)level << kLevelShift);
}
__device__ inline int val_level(uint32_t v) { return (int)(v >> kLevelShift); }
__device__ inline uint32_t val_handle(uint32_t v) { return v & kHandleMask; }

// lookup; returns slot or -1
__device__ inline int64_t table_find(const DevTable& t, uint64_t key) {
  uint64_t i = mix64(key) & t.mask;
  for (uint64_t probe = 0; probe <= t.mask; probe++) {
    uint64_t k = __ldcg(&t.keys[i]);
    if (k == key) return (int64_t)i;
    if (k == kEmptyKey) return -1;
    i = (i + 1) & t.mask;
  }
  return -1;
}

// Lock-free find-or-insert of a key (64-bit atomicCAS, linear probing).
// Returns slot (or -1 if the table is full); *inserted set when this
// thread created the entry.  The key goes to the first tombstone on its
// probe path, but only after the scan has reached an EMPTY slot without
// meeting the key (so a key is never live twice); with no tombstone on the
// path it takes that EMPTY slot.  A lost CAS race rescans from home.
// Erasure never runs concurrently with inserts (separate kernels).
__device__ inline int64_t table_find_or_insert(const DevTable& t, uint64_t key, bool* inserted) {
  *inserted = false;
  const uint64_t home = mix64(key) & t.mask;
  for (;;) {
    uint64_t i = home, probe = 0;
    int64_t tomb = -1;
    for (; probe <= t.mask; probe++) {
      const uint64_t k = __ldcg(&t.keys[i]);
      if (k == key) return (int64_t)i;
      if (k == kEmptyKey) break;
      if (k == kTombKey && tomb < 0) tomb = (int64_t)i;
      i = (i + 1) & t.mask;
    }
    if (probe > t.mask && tomb < 0) return -1;  // no EMPTY and no tombstone left
    const uint64_t at = tomb >= 0 ? (uint64_t)tomb : i;
    const unsigned long long expect = tomb >= 0 ? kTombKey : kEmptyKey;
    const unsigned long long old =
        atomicCAS((unsigned long long*)&t.keys[at], expect, (unsigned long long)key);
    if (old == expect) {
      if (tomb >= 0) atomicAdd(t.n_tomb, ~0ull);  // one tombstone fewer
      *inserted = true;
      return (int64_t)at;
    }
    if (old == key) return (int64_t)at;
  }
}

// erase a live entry (remove, evict, merge-free never erases: re-home keeps
// the key): the slot becomes a tombstone that later inserts reuse
__device__ inline void table_erase(const DevTable& t, uint64_t slot) {
  t.vals[slot] = kPending;
  t.stamp[slot] = 0;
  t.keys[slot] = kTombKey;
  atomicAdd(t.n_tomb, 1ull);
}

// warp-aggregated append to a device list: one atomic per warp
__device__ inline unsigned long long warp_append(unsigned long long* counter, bool pred) {
  unsigned mask = __ballot_sync(__activemask(), pred);
  // callers guarantee the full active set reaches here together
  unsigned lane = threadIdx.x & 31;
  int leader = __ffs(mask) - 1;
  unsigned long long base = 0;
  if (mask) {
    if ((int)lane == leader) base = atomicAdd(counter, (unsigned long long)__popc(mask));
    base = __shfl_sync(__activemask(), base, leader);
  }
  return base + __popc(mask & ((1u << lane) - 1));
}

}  // namespace tsdf
