// engine.cuh — internal definitions shared by the libdbtsdf CUDA sources.
//
// Device voxel word (32 bits, one per voxel, the "single aligned word" every
// per-voxel update is applied to):
//
//   bits  0..18  T: the low 19 bits of the reference's 32-bit distance mask.
//                Masks are low-bit runs (grid.py:118-136), so T is a run of
//                min(L, 19) ones where L = popcount(mask) is the distance.
//   bits 19..22  E: L - 19 when L >= 19 (0..13), else 0.
//   bit  23      1 = SIGN_FREE, 0 = SIGN_OCCUPIED (grid.py SIGN_*)
//   bits 24..31  saturating hit counter (u8)
//
// Every distance the K<=21 kernel can write is <= ceil(sqrt(3)*10) = 18, so
// "this return lowers the stored distance to d" is the single bit test
// (w >> d) & 1, and the update is one native atomicAnd (RED.AND) with
// 0xFF800000 | ((1 << d) - 1): T becomes the run of min(L, d) ones and E is
// cleared, exactly the reference's mask AND (integrator.py:145-149) on the
// encoded word. AND is commutative and idempotent, so no CAS loop and no
// retries. Hits/sign (|S| cells per return) use a 32-bit CAS.
//
// The reference stores mask u32 + sign u8 + hits u8 as three C-order arrays
// (grid.py:47-49) and serialises 8-byte records (grid.py:30-34); the device
// word is lossless for every grid the reference can produce (runs; sign 0/1)
// at half the record size.
//
// Distance cache: one byte per voxel, dist[v] >= run length of cells[v] at
// all times (equal after upload/reset).
//
// Stamp certificates: one bit per voxel, set by the warp that swept the
// stamp centred at that voxel (one writer per bit per launch: centres are
// deduplicated). A set bit means the full K^3 stamp of that centre is already
// in the grid; the AND being idempotent, a later return centred there needs
// no sweep (its shadow update still runs). Cleared on reset/upload and when a
// launch uses a different distance kernel. The sweep reads it (8 voxels per
// 64-bit load) to find the voxels a return lowers, then applies RED.AND to
// the word and stores the new distance into the cache. Cache stores race
// only with other lowering stores, so a cache byte can end up stale-high
// (a later redundant AND) but never below the word: no update is ever lost.
//
// Layout in HBM: C-order (x, y, z) like the reference arrays, x restricted to
// the owned slab [x0, x1), z stride padded to a multiple of 8 voxels so every
// z-row of the cache starts 8-byte aligned (and of the words 32-byte aligned).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

#include "../../include/dbtsdf.h"

namespace dbt {

typedef uint32_t cell_t;
constexpr uint32_t kTMask = 0x7FFFFu;        // run bits 0..18
constexpr int kTBits = 19;
constexpr int kEShift = 19;
constexpr uint32_t kEMask = 0xFu << kEShift;
constexpr uint32_t kFreeBit = 1u << 23;
constexpr int kHitsShift = 24;
constexpr uint32_t kKeepSignHits = 0xFF800000u;  // AND mask bits that a mask update keeps
constexpr uint32_t kFreshCell = kTMask | (13u << kEShift) | kFreeBit;  // L=32, free, 0 hits
constexpr int kMaxFastD = 18;                 // kernel distances the RED.AND path handles
constexpr int kCenterBits = 21;                 // packed centre: 3 x 21 bits
constexpr int64_t kMaxDim = (1 << kCenterBits) - 1;
constexpr uint64_t kEmptyKey = ~0ull;
constexpr int kMaxK = 31;          // kernel edge supported by the sweep templates
constexpr int kMaxScansPerLaunch = 4096;

__host__ __device__ inline int cell_len(uint32_t c) {
  const uint32_t t = c & kTMask;
#ifdef __CUDA_ARCH__
  return t == kTMask ? kTBits + (int)((c >> kEShift) & 0xF) : __popc(t);
#else
  return t == kTMask ? kTBits + (int)((c >> kEShift) & 0xF) : __builtin_popcount(t);
#endif
}
// distance run length L (0..32), sign (0/1), hits (0..255) -> word
__host__ __device__ inline uint32_t make_cell(int len, int free_, uint32_t hits) {
  const uint32_t t = len >= kTBits ? kTMask : ((1u << len) - 1u);
  const uint32_t e = len >= kTBits ? (uint32_t)(len - kTBits) : 0u;
  return t | (e << kEShift) | (free_ ? kFreeBit : 0u) | (hits << kHitsShift);
}
__host__ __device__ inline uint32_t cell_with_len(uint32_t c, int len) {
  return make_cell(len, (c & kFreeBit) ? 1 : 0, c >> kHitsShift);
}
__host__ __device__ inline uint32_t run_mask_of(int len) { return len ? (0xFFFFFFFFu >> (32 - len)) : 0u; }

__host__ __device__ inline uint64_t pack_center(int64_t x, int64_t y, int64_t z) {
  return ((uint64_t)x << (2 * kCenterBits)) | ((uint64_t)y << kCenterBits) | (uint64_t)z;
}
__host__ __device__ inline void unpack_center(uint64_t c, int64_t& x, int64_t& y, int64_t& z) {
  const uint64_t m = (1ull << kCenterBits) - 1;
  x = (int64_t)(c >> (2 * kCenterBits));
  y = (int64_t)((c >> kCenterBits) & m);
  z = (int64_t)(c & m);
}

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
  int error;                     // upload validation etc.
  int pad;
};

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
  int max_d = 0;                     // largest kernel run length (fast path needs <= 18)
  int8_t* d_shadow_xyz = nullptr;    // total_shadow x 4 (dx,dy,dz,0)
  int32_t* d_shadow_start = nullptr; // n_bins + 1
  uint64_t serial = 0;               // identity for per-grid caches
  uint64_t dk_hash = 0;              // FNV-1a of K and the kernel run lengths
};

struct dbt_grid {
  int device = 0;
  int64_t nx = 0, ny = 0, nz = 0, nzp = 0;  // global dims, padded z stride
  int64_t x0 = 0, x1 = 0;                   // owned slab
  double vs = 0, org[3] = {0, 0, 0};
  uint32_t* cells = nullptr;                // authoritative voxel words
  uint8_t* dist = nullptr;                  // distance cache, dist[v] >= len(cells[v])
  uint32_t* stamped = nullptr;              // stamp certificates, one bit per voxel
  int64_t n_cells = 0;                      // (x1-x0)*ny*nzp
  cudaStream_t stream = nullptr;
  bool own_stream = true;

  // --- per-launch scratch (grown on demand) ---
  int64_t cap_pts = 0;          // capacity in points (after downsampling)
  int64_t cap_raw_bytes = 0;    // raw input staging
  void* d_raw = nullptr;
  uint64_t* d_center = nullptr; // packed centre per point (kEmptyKey = not ok)
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
  cudaEvent_t ev_a = nullptr, ev_b = nullptr;  // device_ms of the last call
  cudaEvent_t ev_meta = nullptr;               // pinned metadata consumed by the stream
  cudaStream_t aux = nullptr;                  // shadow kernel, concurrent with the sweep
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int last_first_return = 0;
  // distance kernel the stamp certificates refer to (0: none yet)
  uint64_t cert_dk = 0;
  int sweep_ch = 0;                            // cached sweep launch shape
  int64_t sweep_blocks = 0;
  double last_device_ms = 0;
};

namespace dbt {

// error plumbing (abi.cu)
int set_error(int code, const std::string& msg);
int cuda_error(cudaError_t e, const char* what);
void count_launch();

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

// scratch management (grid.cu)
int ensure_stage(dbt_grid* g, int64_t bytes);
int grid_set_device(const dbt_grid* g);

}  // namespace dbt
