// engine.cuh — internal definitions shared by the libdbtsdf CUDA sources.
//
// Device voxel record (8 bytes, one per voxel, stored as two 32-bit arrays —
// Cells below): the reference's serialized record (grid.py:30-34) — .x (m) =
// the 32-bit distance mask, .y (y) = sign (byte 0) | hits (byte 1) << 8 |
// pending shadow visits (bytes 2-3, 0 in every record that leaves the
// device). The two words are the single aligned words the two update kinds
// touch:
//   * mask update (integrator.py:145-149): a MIN on the voxel's length cache
//     word (below); the mask word itself is folded lazily;
//   * shadow update (integrator.py:151-159): one atomicAdd of 1 << 16 on .y
//     counts the visit. n visits of the step h += (h < h_max), sign = 0 when
//     h >= T, compose to h' = h >= h_max ? h : min(h + n, h_max) and sign = 0
//     when h' >= T (fold_meta), so counts are folded lazily: before any read
//     of the grid, before a launch with other (h_max, T), and by the visit
//     that takes a count to 2^15 (no 16-bit overflow).
// Any mask and sign byte the reference can hold is represented (no run-mask
// assumption).
//
// Length cache: one 16-bit word per voxel, the run length the voxel's mask
// is lowered to: the effective mask of voxel v is m[v] & run_mask(len[v]).
// The sweep never touches the mask words: a return lowers voxel v exactly
// when its kernel run length d < len[v] (for the run masks integration
// produces, len = bit length of the effective mask), and the lowering is one
// hardware MIN on the cache — REDG.MIN.F16x8 over 8 voxels, the lengths kept
// as raw 16-bit integers 0..64, which are (subnormal) f16 values ordered like
// the integers under .noftz. MIN is commutative and idempotent, so the cache
// is exact: AND-ing run masks composes as m & run(d1) & run(d2) =
// m & run(min(d1, d2)). The masks are folded lazily (m &= run_mask(len),
// fold_pending) before any read of the records, like the pending shadow
// visits below; uploads and resets set len = bit length of the mask.
// Stamp certificates: one bit per voxel, set when the full K^3 stamp centred
// at that voxel (on a sharded grid: the part of it on this part's planes) is
// in the grid or claimed by a return of the running launch;
// the AND being idempotent, a later return centred there needs no sweep (its
// shadow update still runs). Returns claim the bit with one atomicOr in
// preprocessing. Cleared on reset/upload and when a launch uses a different
// distance kernel.
//
// Layout in HBM: C-order (x, y, z) like the reference arrays, x restricted to
// the owned slab [x0, x1), z stride padded to a multiple of 8 voxels so every
// z-row of the cache starts 8-byte aligned.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <string>
#include <vector>

#include "../../include/dbtsdf.h"

namespace dbt {

constexpr uint32_t kFullMask = 0xFFFFFFFFu;
constexpr uint32_t kFreshMeta = 1u;   // sign free (1), 0 hits
constexpr uint32_t kSignByte = 0xFFu;
constexpr uint32_t kHitsByte = 0xFF00u;
constexpr int kCenterBits = 21;                 // packed centre: 3 x 21 bits
constexpr int64_t kMaxDim = (1 << kCenterBits) - 1;
constexpr uint64_t kEmptyKey = ~0ull;
constexpr int kMaxK = 31;          // kernel edge supported by the sweep templates
constexpr int kMaxScansPerLaunch = 4096;
constexpr int kBrickShift = 4;     // replica dirty bricks: 16^3 voxels

__host__ __device__ inline uint32_t make_meta(uint32_t sign, uint32_t hits) { return (sign & 0xFFu) | ((hits & 0xFFu) << 8); }
__host__ __device__ inline uint8_t meta_sign(uint32_t m) { return (uint8_t)(m & 0xFFu); }
__host__ __device__ inline uint8_t meta_hits(uint32_t m) { return (uint8_t)((m >> 8) & 0xFFu); }
__device__ inline int mask_bitlen(uint32_t m) { return 32 - __clz(m); }
__host__ __device__ inline uint32_t run_mask_of(int len) { return len ? (0xFFFFFFFFu >> (32 - len)) : 0u; }

constexpr int kPendShift = 16;        // pending shadow visits in .y bits 16-31
constexpr uint32_t kPendFold = 0x8000u;
// n pending visits of h += (h < h_max), sign = 0 when h >= T (integrator.py:
// 154-159) applied at once; the pending bits are cleared
__host__ __device__ inline uint32_t fold_meta(uint32_t y, uint32_t h_max, uint32_t t_occ) {
  const uint32_t n = y >> kPendShift;
  if (!n) return y;
  const uint32_t h = (y >> 8) & 0xFFu;
  uint32_t sign = y & 0xFFu;
  const uint32_t hn = h >= h_max ? h : (h + n < h_max ? h + n : h_max);
  if (hn >= t_occ) sign = 0;
  return sign | (hn << 8);
}

__host__ __device__ inline uint64_t pack_center(int64_t x, int64_t y, int64_t z) {
  return ((uint64_t)x << (2 * kCenterBits)) | ((uint64_t)y << kCenterBits) | (uint64_t)z;
}
__host__ __device__ inline void unpack_center(uint64_t c, int64_t& x, int64_t& y, int64_t& z) {
  const uint64_t m = (1ull << kCenterBits) - 1;
  x = (int64_t)(c >> (2 * kCenterBits));
  y = (int64_t)((c >> kCenterBits) & m);
  z = (int64_t)(c & m);
}

// Owned x-planes of a grid (multi-GPU sharding): every
// global plane x in [x0, x1) when w == 0 (a contiguous slab), else the planes
// of [x0, x1) whose block (x - x0) / w is congruent to r mod p (interleaved
// slabs of w planes dealt round-robin over p ranks). Owned planes are stored
// in increasing x order; local(x) is the storage plane or -1 when not owned.
struct XMap {
  int64_t x0 = 0, x1 = 0;
  int64_t w = 0;
  int32_t p = 1, r = 0;
  // 32-bit arithmetic: planes are < 2^21 (kMaxDim), and int64 division is a
  // long software sequence on the GPU
  __host__ __device__ __forceinline__ int64_t local(int64_t gx) const {
    if (gx < x0 || gx >= x1) return -1;
    if (w == 0) return gx - x0;
    const uint32_t u = (uint32_t)(gx - x0), ww = (uint32_t)w, blk = u / ww;
    const uint32_t q = blk / (uint32_t)p;
    if (blk - q * (uint32_t)p != (uint32_t)r) return -1;
    return (int64_t)(q * ww + (u - blk * ww));
  }
  // some owned plane lies in [lo, hi] (a return's K^3 cube [cx-R, cx+R]
  // touches this part)
  __host__ __device__ __forceinline__ bool touches(int64_t lo, int64_t hi) const {
    lo = lo < x0 ? x0 : lo;
    hi = hi >= x1 ? x1 - 1 : hi;
    if (lo > hi) return false;
    if (w == 0) return true;
    const uint32_t ww = (uint32_t)w, b0 = (uint32_t)(lo - x0) / ww, b1 = (uint32_t)(hi - x0) / ww;
    if (b1 - b0 + 1 >= (uint32_t)p) return true;
    for (uint32_t b = b0; b <= b1; ++b)
      if (b % (uint32_t)p == (uint32_t)r) return true;
    return false;
  }
  __host__ int64_t planes() const {
    if (w == 0) return x1 - x0;
    int64_t n = 0;
    for (int64_t b = r; b * w < x1 - x0; b += p) n += std::min(w, x1 - x0 - b * w);
    return n;
  }
};

// The voxel records, split into two arrays of 32-bit words with the same
// indexing: m = the distance masks (the sweep's RED.AND target), y = sign |
// hits << 8 | pending shadow visits << 16 (the shadow kernel's atomicAdd
// target). A record is (m[i], y[i]); the split keeps each update kind's
// traffic on its own array (4 bytes per touched voxel instead of the 8-byte
// record sector share).
struct Cells {
  uint32_t* m = nullptr;
  uint32_t* y = nullptr;
  __host__ __device__ __forceinline__ uint2 get(int64_t i) const { return make_uint2(m[i], y[i]); }
  __host__ __device__ __forceinline__ void put(int64_t i, uint2 v) const {
    m[i] = v.x;
    y[i] = v.y;
  }
  __host__ __device__ __forceinline__ Cells off(int64_t o) const { return Cells{m + o, y + o}; }
};

// Per-scan device counters (one entry per scan of a launch).
struct ScanCounters {
  unsigned long long n_ok;       // non-discarded returns
  unsigned long long n_applied;  // stamped returns (after first-return)
  unsigned long long n_fallback; // returns binned outside the SVML restatement
  unsigned long long pad;
};
// Launch-wide device counters.
struct LaunchCounters {
  unsigned long long n_unique;   // unique centre keys (sweep work items)
  unsigned long long changed;    // mask cells changed (voxels_written)
  unsigned long long skipped;    // centres whose stamp was already applied (cache byte 0)
  unsigned long long work;       // sweep work-item cursor (dynamic fetch)
  unsigned long long rows;       // kernel rows the sweep read
  unsigned long long exact_written;  // serial voxels_written (DBT_FLAG_EXACT_WRITTEN)
  unsigned long long pad[2];
};

// One in-flight asynchronous single-scan call (dbt_integrate_frame_async):
// the device copy of its points, its counters' pinned destination, its
// completion event.
struct AsyncSlot {
  int64_t ticket = -1;
  cudaEvent_t copied = nullptr, done = nullptr;
  void* d_buf = nullptr;
  int64_t cap = 0;
  void* h_stage = nullptr;      // pinned staging of a pageable scan (hostcopy.cu)
  int64_t cap_hstage = 0;
  LaunchCounters* h = nullptr;  // LaunchCounters + one ScanCounters, pinned
  int64_t points_in = 0;
  dbt_params p{};
  double t0 = 0;
};
constexpr int kAsyncSlots = 4;

struct ProfEvent {
  cudaEvent_t a, b;
  int kernel;  // index into prof_names
};

}  // namespace dbt

struct dbt_bank {
  int device = 0;
  int K = 0, R = 0, b_az = 0, b_el = 0, n_bins = 0;
  int max_shadow = 0;
  int64_t total_shadow = 0;
  uint8_t* d_len = nullptr;          // K^3 run lengths of distance_kernel
  uint2* d_dtab = nullptr;           // sweep table: [8 shifts][distinct rows][CH] 8 packed d bytes
  uint16_t* d_rowd = nullptr;        // K*K: distinct-row id * CH
  int n_distinct = 0;
  int chunks_per_row = 0;            // CH = ceil((K+7)/8) 8-voxel chunks per kernel row
  int max_d = 0;                     // largest kernel run length
  int iso = 0;                       // run length = h(|o|^2), h non-decreasing, CH <= 4:
                                     // sweep_cull_kernel (neighbour-dominance culling)
  int8_t* d_shadow_xyz = nullptr;    // total_shadow x 4 (dx,dy,dz,0)
  int32_t* d_shadow_start = nullptr; // n_bins + 1
  uint64_t serial = 0;               // identity for per-grid caches
  uint64_t dk_hash = 0;              // FNV-1a of K and the kernel run lengths
};

struct dbt_grid {
  int device = 0;
  int64_t nx = 0, ny = 0, nz = 0, nzp = 0;  // global dims, padded z stride
  int64_t x0 = 0, x1 = 0;                   // owned x range (xm.x0, xm.x1)
  dbt::XMap xm;                             // owned planes (contiguous or interleaved)
  int64_t lx = 0;                           // owned plane count (storage x extent)
  double vs = 0, org[3] = {0, 0, 0};
  dbt::Cells cells;                         // authoritative voxel records (masks | meta words)
  uint16_t* dist = nullptr;                 // length cache: effective mask = cells.m[v] & run_mask(dist[v])
  bool lazy_m = false;                      // masks not yet folded with the length cache (fold_pending)
  uint32_t* stamped = nullptr;              // stamp certificates, one bit per voxel of the GLOBAL grid
                                            // (index (x*ny + y)*nzp + z, x global): a part of a sharded
                                            // grid certifies every centre whose cube touches its planes
  int64_t n_cert = 0;                       // nx*ny*nzp certificate bits
  uint32_t* d_exact_bits = nullptr;         // centre + touched + centre-row bitmaps (exact.cu), lazily
  uint32_t* d_exact_m0 = nullptr;           // pre-launch masks of touched cells (exact.cu)
  uint8_t* d_base_hits = nullptr;           // replica mode: hits at the last merge (replica.cu)
  uint32_t* d_base_mask = nullptr;          // replica mode: masks at the last merge
  bool base_valid = false;                  // d_base_hits describes the current records' base
  // replica mode: one flag per 16^3 brick holding the centre of a return
  // applied since the last mark/merge (set by prep_kernel), so a merge moves
  // only the bricks within a kernel radius of some rank's returns
  uint8_t* d_dirty = nullptr;
  int64_t dbx = 0, dby = 0, dbz = 0;        // brick grid (ceil(n / 16) per axis)
  int dirty_reach = 0;                      // largest kernel radius R integrated since the last merge
  int32_t* d_sel = nullptr;                 // selected bricks of the pending merge (dbt_replica_select)
  int64_t n_sel = 0, cap_sel = 0;
  int64_t n_cells = 0;                      // lx*ny*nzp
  cudaStream_t stream = nullptr;
  bool own_stream = true;

  // --- per-launch scratch (grown on demand) ---
  int64_t cap_pts = 0;          // capacity in points (after downsampling)
  int64_t cap_raw_bytes = 0;    // raw input staging
  void* d_raw = nullptr;
  uint64_t* d_center = nullptr; // packed centre per point (kEmptyKey = not ok)
  double* d_ray = nullptr;       // map-frame ray per point (binned by the shadow kernel)
  uint16_t* d_bin = nullptr;
  uint32_t* d_slot = nullptr;
  uint64_t* d_uniq = nullptr;   // unique packed centres
  int64_t cap_hash = 0;
  uint32_t hash_epoch = 0;      // epoch tag of live hash keys (no per-launch clear)
  unsigned long long* d_hkey = nullptr;
  uint32_t* d_hmin = nullptr;
  double* d_sensor = nullptr;   // map-frame mode per-point sensor (n x 3)
  int64_t cap_sensor = 0;
  int8_t* d_outcome = nullptr;
  int64_t cap_outcome = 0;
  double* d_ts = nullptr;       // device deskew: per-point times
  int64_t cap_ts = 0;
  // per-scan metadata
  int64_t* d_scan_off = nullptr;    // kMaxScansPerLaunch + 1 (downsampled)
  dbt::ScanCounters* d_scnt = nullptr;
  dbt::LaunchCounters* d_lcnt = nullptr;
  dbt::ScanCounters* h_scnt = nullptr;   // pinned mirrors
  dbt::LaunchCounters* h_lcnt = nullptr;
  int64_t* h_meta = nullptr;             // pinned staging for offsets
  int last_scans = 0;
  std::vector<int64_t> last_points_in;
  std::vector<int64_t> last_points_in_host;
  // pinned, mapped host staging of pageable scans (hostcopy.cu)
  void* h_stage = nullptr;
  int64_t cap_hstage = 0;
  // staging for upload/download/readout
  void* d_stage = nullptr;
  int64_t cap_stage = 0;

  // --- per-bank derived table (depends on ny, nzp) ---
  uint64_t tab_bank = 0;
  int32_t* d_rowoff = nullptr;   // K*K row offsets (dx*ny+dy)*nzp (fit int32, checked)
  int tab_K = 0;

  // --- measurement ---
  bool profiling = false;
  std::vector<dbt::ProfEvent> pending;
  std::vector<cudaEvent_t> event_pool;
  std::vector<std::string> prof_names;
  std::vector<double> prof_ms;
  std::vector<int64_t> prof_launches;
  cudaEvent_t ev_a = nullptr, ev_b = nullptr;  // device_ms of the last call (timed calls)
  cudaEvent_t ev_done = nullptr;               // completion of a synchronous call (no timing)
  bool time_calls = false;                     // $DBT_DEVICE_MS: device_ms on every synchronous call
  cudaEvent_t ev_meta = nullptr;               // pinned metadata consumed by the stream
  cudaStream_t aux = nullptr;                  // shadow kernel, concurrent with the sweep
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int last_first_return = 0;
  // distance kernel the stamp certificates refer to (0: none yet)
  uint64_t cert_dk = 0;
  // shadow visits pending in the records (folded before reads, see above)
  bool pend = false;
  int pend_h_max = 0, pend_t_occ = 0;
  // stream of the last integration launch: reads on the grid stream wait for
  // it on the host (an event recorded per launch costs ~7 us of pipelined
  // throughput on config 2)
  cudaStream_t last_st = nullptr;
  // CUDA graph of the synchronous single-scan launch sequence (integrate.cu,
  // integrate_host_graph): captured once per launch shape, replayed with
  // updated prep / shadow kernel arguments
  cudaGraph_t ggraph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  cudaGraphNode_t gprep = nullptr, gshadow = nullptr;
  uint64_t gkey[12] = {};
  int gkernels = 0;
  bool gdisabled = false;                      // capture unsupported here, or $DBT_NO_GRAPH
  int sweep_ch = 0;                            // cached sweep launch shape
  int64_t sweep_blocks = 0;
  double last_device_ms = 0;
  // asynchronous single-scan calls (integrate.cu): copies on cstream
  dbt::AsyncSlot aslot[dbt::kAsyncSlots];
  // one executable graph per async slot (instantiated from ggraph): updating
  // the arguments of an executable graph that is still running waits for it,
  // so pipelined calls must not share one
  cudaGraphExec_t aexec[dbt::kAsyncSlots] = {};
  int64_t a_next = 0;
  cudaStream_t cstream = nullptr;
};

namespace dbt {

// pending shadow visits (grid.cu): make the records final before a read
int fold_pending(dbt_grid* g, cudaStream_t st);
// serial voxels_written of a one-scan launch (exact.cu): pre before the
// sweep, post after it
int launch_exact_pre(dbt_grid* g, const dbt_bank* b, cudaStream_t st);
int launch_exact_post(dbt_grid* g, const dbt_bank* b, cudaStream_t st);

// error plumbing (abi.cu)
int set_error(int code, const std::string& msg);
int cuda_error(cudaError_t e, const char* what);
void count_launch();
void add_launches(int64_t n);  // kernels run by a graph launch (or undo counts made under capture)

#define DBT_CUDA(call)                                   \
  do {                                                   \
    cudaError_t _e = (call);                             \
    if (_e != cudaSuccess) return dbt::cuda_error(_e, #call); \
  } while (0)

#define DBT_CHECK_LAUNCH(name)                                 \
  do {                                                         \
    cudaError_t _e = cudaGetLastError();                       \
    if (_e != cudaSuccess) return dbt::cuda_error(_e, name);   \
    dbt::count_launch();                                       \
  } while (0)

// profiling helpers (abi.cu)
void prof_begin(dbt_grid* g, const char* name, cudaStream_t s, int* token);
void prof_end(dbt_grid* g, cudaStream_t s, int token);
int prof_flush(dbt_grid* g);

// pageable scans -> pinned mapped staging with a host thread pool
// (hostcopy.cu): out[i] = device pointer of scan i; false = not staged
bool stage_pageable(dbt_grid* g, const void* const* srcs, const int64_t* bytes, int n, const void** out);
void pooled_host_copy(void* dst, const void* src, size_t bytes);

// scratch management (grid.cu)
int ensure_stage(dbt_grid* g, int64_t bytes);
int grid_set_device(const dbt_grid* g);

}  // namespace dbt
