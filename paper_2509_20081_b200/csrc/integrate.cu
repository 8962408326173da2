// integrate.cu — the scan-integration hot path (reference integrator.py:139-287).
//
// One launch sequence per scan (or per batch of scans):
//   prep_kernel    one thread per return: sensor->map transform (numpy's
//                  matmul FMA chain, integrator.py:232), ray, norm, degenerate
//                  and boundary discards (integrator.py:192-199), centre voxel
//                  (grid.py:107-111), direction bin (kernels.py:49-57),
//                  centre dedup / first-return in a device hash table
//                  (integrator.py:256-262), per-scan counters.
//   shadow_kernel  one thread per (applied return, shadow offset): saturating
//                  hit increment + occupied sign (integrator.py:151-159) as a
//                  32-bit CAS on the record's sign/hits word; runs on a second
//                  stream, concurrent with the sweep.
//   sweep_kernel   one warp per centre to sweep: the K^3 AND (integrator.py:
//                  145-149) over the 1-byte distance cache, RED.AND of the
//                  kernel run mask into the record's mask word on change.
//
// Order independence: every voxel update is an atomic application of a
// monotone function (min on the run length; h -> h + (h < h_max) with the
// sign set when h >= T) and the functions for different returns commute, so
// the final grid equals the reference's serial sorted-order stamping
// (integrator.py:266-284) for any schedule. Duplicate centres stamp the same
// mask (AND is idempotent), so the sweep runs once per distinct centre.
#include <algorithm>
#include <climits>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <vector>

#include <chrono>

#include <mutex>
#include <thread>

#include "engine.cuh"
#include <math_constants.h>

#include "svml_emu.cuh"
#include "deskew.cuh"
#include "libm_table.h"

using namespace dbt;

extern const uint16_t dbt_svml_seeds[131072];  // build/svml_seeds.cu

namespace {

constexpr double kTwoPi = 6.283185307179586;     // 2.0 * math.pi   (kernels.py:28)
constexpr double kPi = 3.141592653589793;        // np.pi
constexpr double kHalfPi = 1.5707963267948966;   // np.pi / 2       (kernels.py:56)

struct PrepArgs {
  const void* pts;
  const double* sensor;  // map-frame mode: per-point sensor positions
  int dtype;
  int S;
  int ds;
  int map_mode;
  int64_t n;
  const int64_t* scan_off;
  const int64_t* src_off;
  const double* poses;  // S x 12 : R row-major (9), t (3)
  const uint64_t* scan_ptr;  // S device pointers, one per scan (nullptr: pts + src_off)
  int64_t nx, ny, nz;
  double vs, ox, oy, oz;
  int R, b_az, b_el;
  int skip_norm;
  int first_return;
  int key_scan_bits;  // first-return over several scans: key includes the scan
  int no_dedup;       // DBT_FLAG_NO_DEDUP: sweep every applied return
  uint64_t* center;
  uint16_t* bin;
  uint32_t* slot;
  unsigned long long* hkey;
  uint32_t* hmin;
  uint64_t hmask;
  uint64_t* uniq;
  LaunchCounters* lc;
  ScanCounters* sc;
  int8_t* outcome;
  const uint16_t* seeds;
  int inline_meta;     // single scan: pose below, offsets trivial (no device metadata)
  double pose0[12];
  uint64_t epoch;      // hash-key epoch tag (bits 52..63); stale slots count as empty
  // fused shadow update (no first-return, small shadow sets)
  int fuse_shadow;
  Cells cells;
  const int8_t* sxyz;
  const int32_t* sstart;
  int64_t x0, x1, nzp;
  XMap xm;  // owned planes (x0, x1 above are its range)
  int h_max, t_occ;
  // claim mode (no first-return): dedup + cross-launch skip through the stamp
  // certificate bits instead of the hash table
  int claim;
  uint32_t* stamped;
  int bins;     // direction bins here (else rays out, binned in shadow_bin_kernel)
  double* ray;  // n x 3 map-frame rays (bins == 0)
  // replica mode: dirty flag of the 16^3 brick holding each applied centre
  uint8_t* dirty;
  int64_t dby, dbz;
  // device deskew (compensation yaw/se3, single-scan launches): the point is
  // moved to the end-of-sweep frame first (deskew.cuh); dk_ts = per-point
  // times by raw index, or null for linspace over the n downsampled points
  int deskew;
  dbt_deskew dk;
  const double* dk_ts;
  const double* sincos;  // the C library's sin/cos table (libm_emu.cuh)
};

constexpr uint64_t kKeyMask = (1ull << 52) - 1;  // cflat (< 2^40) | scan << 40
// packed-centre flag (bit 63, above the 3 x 21 coordinate bits): the return
// is applied but its cube misses this part's planes (sharded grids)
constexpr uint64_t kRemote = 1ull << 63;
constexpr int kEpochShift = 52;
constexpr uint32_t kMaxEpoch = 4095;

// one shadow visit: count it in the record's pending field (engine.cuh);
// the visit that takes the count to 2^15 folds the record right away, so the
// 16-bit field never overflows
__device__ __forceinline__ void shadow_add(uint32_t* p, uint32_t h_max, uint32_t t_occ) {
  const uint32_t old = atomicAdd(p, 1u << kPendShift);
  if ((old >> kPendShift) + 1 != kPendFold) return;
  uint32_t cur = __ldcg(p);
  while (true) {
    const uint32_t nw = fold_meta(cur, h_max, t_occ);
    if (nw == cur) break;
    const uint32_t prev = atomicCAS(p, cur, nw);
    if (prev == cur) break;
    cur = prev;
  }
}

__device__ __forceinline__ uint64_t mix64(uint64_t k) {
  k ^= k >> 33;
  k *= 0xff51afd7ed558ccdull;
  k ^= k >> 33;
  k *= 0xc4ceb9fe1a85ec53ull;
  k ^= k >> 33;
  return k;
}

__device__ __forceinline__ int find_scan(const int64_t* off, int S, int64_t i) {
  int lo = 0, hi = S;  // off[lo] <= i < off[hi]
  while (hi - lo > 1) {
    int mid = (lo + hi) >> 1;
    if (off[mid] <= i) lo = mid;
    else hi = mid;
  }
  return lo;
}

// bin_index_array (kernels.py:49-57) for one direction whose axis-1 norm is
// nrm. arctan2/arcsin are the bit-exact restatement of numpy's SVML routines
// (svml_emu.cuh), every other step the same IEEE operation numpy performs, so
// the bin equals the reference's for every input. A ray with a nonzero
// component outside [2^-1020, 2^993) would take SVML's scalar helper, which is
// not restated: CUDA's atan2 is used and *fallback is set (counted).
__device__ __forceinline__ void bin_dev(double rx, double ry, double rz, double nrm, int b_az,
                                        int b_el, const uint16_t* seeds, int& ba, int& be,
                                        int& fallback) {
  int rare = 0;
  double az = svml::atan2(ry, rx, seeds, &rare);
  fallback = rare;
  if (rare) az = atan2(ry, rx);
  if (az < 0.0) az = __dadd_rn(az, kTwoPi);
  double ra = __dmul_rn(__ddiv_rn(az, kTwoPi), (double)b_az);
  double q = __ddiv_rn(rz, nrm);
  q = q < -1.0 ? -1.0 : (q > 1.0 ? 1.0 : q);
  double el = svml::asin(q, seeds);
  double re = __dmul_rn(__ddiv_rn(__dadd_rn(el, kHalfPi), kPi), (double)b_el);
  long long ia = (long long)ra;  // astype(np.int64) truncates toward zero
  long long ie = (long long)re;
  ba = (int)(ia < 0 ? 0 : (ia > b_az - 1 ? b_az - 1 : ia));
  be = (int)(ie < 0 ? 0 : (ie > b_el - 1 ? b_el - 1 : ie));
}

__device__ __forceinline__ bool floor_index(double v, double o, double vs, long long& out) {
  // np.floor((p - origin) / voxel_size).astype(np.int64) (grid.py:109-111);
  // values outside int64 (incl. NaN/inf) become an out-of-bounds index.
  double f = floor(__ddiv_rn(__dsub_rn(v, o), vs));
  if (!(f >= -9.2e18 && f <= 9.2e18)) {
    out = LLONG_MIN;
    return false;
  }
  out = (long long)f;
  return true;
}

constexpr int kPrepThreads = 256;

// Return i in the map frame (integrator.py:223-232): the source point
// (downsampled index, per-scan offsets), and m = p @ R.T + t with the sensor
// position t (map mode: given per point). Shared by prep and the shadow
// kernel's bin phase, so both see the same doubles.
template <bool DESKEW>
__device__ __forceinline__ void map_point(const PrepArgs& a, int64_t i, int& s, double& m0, double& m1, double& m2,
                                          double& t0, double& t1, double& t2) {
  int64_t src;
  s = 0;
  if (a.inline_meta) {
    src = i * a.ds;
  } else {
    s = a.S > 1 ? find_scan(a.scan_off, a.S, i) : 0;
    src = (a.scan_ptr ? 0 : a.src_off[s]) + (i - a.scan_off[s]) * a.ds;
  }
  const void* pts = a.scan_ptr && !a.inline_meta ? (const void*)a.scan_ptr[s] : a.pts;
  double p0, p1, p2;
  if (a.dtype == DBT_F32) {
    const float* q = (const float*)pts + 3 * src;
    p0 = q[0];
    p1 = q[1];
    p2 = q[2];
  } else {
    const double* q = (const double*)pts + 3 * src;
    p0 = q[0];
    p1 = q[1];
    p2 = q[2];
  }
  if (DESKEW) {
    // integrator.py:223-230: motion_compensate, then pts @ R.T + t below
    const double t = deskew::clip01(a.dk_ts ? a.dk_ts[src] : deskew::linspace01(i, a.n));
    double o[3];
    int rare = 0;
    deskew::apply(a.dk, t, p0, p1, p2, o, a.sincos, &rare);
    p0 = rare ? CUDART_NAN : o[0];  // (never for finite poses) discarded like a NaN return
    p1 = o[1];
    p2 = o[2];
  }
  if (a.map_mode) {
    m0 = p0;
    m1 = p1;
    m2 = p2;
    t0 = a.sensor[3 * src];
    t1 = a.sensor[3 * src + 1];
    t2 = a.sensor[3 * src + 2];
  } else {
    const double* P = a.inline_meta ? a.pose0 : a.poses + 12 * s;
    t0 = P[9];
    t1 = P[10];
    t2 = P[11];
    // pts @ R.T + t: OpenBLAS dgemm accumulates k = 0,1,2 with FMA
    // (probed on both the build and the GPU-box hosts), then numpy adds t.
    m0 = __dadd_rn(__fma_rn(p2, P[2], __fma_rn(p1, P[1], __dmul_rn(p0, P[0]))), t0);
    m1 = __dadd_rn(__fma_rn(p2, P[5], __fma_rn(p1, P[4], __dmul_rn(p0, P[3]))), t1);
    m2 = __dadd_rn(__fma_rn(p2, P[8], __fma_rn(p1, P[7], __dmul_rn(p0, P[6]))), t2);
  }
}

// np.linalg.norm(rays, axis=1): sqrt((x*x + y*y) + z*z), no FMA
__device__ __forceinline__ double ray_norm(double rx, double ry, double rz) {
  return __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(rx, rx), __dmul_rn(ry, ry)), __dmul_rn(rz, rz)));
}

// DESKEW: the motion-compensated variant (a separate instantiation keeps the
// default path's register budget)
template <bool DESKEW>
__global__ void __launch_bounds__(kPrepThreads) prep_kernel(PrepArgs a) {
  // the sweep (programmatic dependent launch) may be scheduled once every
  // prep block has started; it waits for this grid's completion before
  // reading anything (griddepcontrol.wait), so only its launch latency
  // overlaps preprocessing
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  const int lane = threadIdx.x & 31;
  bool live = i < a.n;
  int s = 0;
  int ok = 0, fallback = 0;
  bool append = false;  // this lane owns a new sweep work item (unique centre)
  bool claimed = false; // centre stamp already applied / claimed: no sweep
  bool relevant = false; // the return's cube touches this part's planes
  uint64_t packed = kEmptyKey;
  if (live) {
    double m0, m1, m2, t0, t1, t2;
    map_point<DESKEW>(a, i, s, m0, m1, m2, t0, t1, t2);
    double rx = __dsub_rn(m0, t0), ry = __dsub_rn(m1, t1), rz = __dsub_rn(m2, t2);
    double nrm = ray_norm(rx, ry, rz);
    ok = a.skip_norm ? 1 : (nrm >= a.vs);
    long long cx, cy, cz;
    bool fx = floor_index(m0, a.ox, a.vs, cx);
    bool fy = floor_index(m1, a.oy, a.vs, cy);
    bool fz = floor_index(m2, a.oz, a.vs, cz);
    ok = ok && fx && fy && fz && cx >= a.R && cy >= a.R && cz >= a.R && cx <= a.nx - 1 - a.R &&
         cy <= a.ny - 1 - a.R && cz <= a.nz - 1 - a.R;
    if (ok) {
      int ba = 0, be = 0;
      relevant = a.xm.touches(cx - a.R, cx + a.R);
      if (!relevant) {
        // a sharded part skips the bins of returns whose cube misses its
        // planes (only the shadow update of a relevant return needs one)
      } else if (a.bins) {
        bin_dev(rx, ry, rz, nrm, a.b_az, a.b_el, a.seeds, ba, be, fallback);
        a.bin[i] = (uint16_t)(ba * a.b_el + be);
      } else {
        // the shadow kernel bins the return from its ray (off the sweep's
        // critical path, and without re-reading a zero-copy host scan)
        a.ray[3 * i] = rx;
        a.ray[3 * i + 1] = ry;
        a.ray[3 * i + 2] = rz;
      }
      packed = pack_center(cx, cy, cz);
      if (a.dirty)  // replica merge bookkeeping (idempotent plain store)
        a.dirty[((cx >> kBrickShift) * a.dby + (cy >> kBrickShift)) * a.dbz + (cz >> kBrickShift)] = 1;
      // a part of a sharded grid ignores returns whose cube misses its planes
      // (still counted; the first-return choice below stays global)
      if (a.claim && relevant) {
        // claim the stamp certificate of the centre (one atomicOr): a bit
        // already set means the stamp is in the grid from an earlier launch
        // or owned by an earlier return of this launch; either way no sweep.
        // Certificates are indexed by the global centre (a part certifies
        // the centres whose cube touches its planes).
        const int64_t cidx = (cx * a.ny + cy) * a.nzp + cz;
        const uint32_t bit = 1u << (cidx & 31);
        claimed = (atomicOr(a.stamped + (cidx >> 5), bit) & bit) != 0;
        append = !claimed;
      }
      // the hash table dedups centres for the sweep when certificates are not
      // used (measurement flags) and picks the first return per centre for
      // the shadow update in first-return mode
      const bool use_hash = !a.claim || a.first_return;
      uint64_t key = (uint64_t)((cx * a.ny + cy) * a.nz + cz);
      if (a.key_scan_bits) key |= (uint64_t)s << 40;
      uint64_t h = mix64(key) & a.hmask;
      key |= a.epoch;
      if (!a.claim) append = a.no_dedup != 0;
      unsigned long long cur = use_hash ? __ldcg(&a.hkey[h]) : 0ull;
      while (use_hash) {
        if (cur == key) break;  // centre already inserted this launch
        if ((cur & ~kKeyMask) != a.epoch) {
          // slot is empty for this launch (older epoch): claim it
          unsigned long long prev = atomicCAS(&a.hkey[h], cur, (unsigned long long)key);
          if (prev == cur) {
            if (!a.claim && !a.no_dedup) append = true;
            break;
          }
          cur = prev;  // lost the race: re-examine the same slot
          continue;
        }
        h = (h + 1) & a.hmask;
        cur = __ldcg(&a.hkey[h]);
      }
      append = append && relevant;
      if (a.fuse_shadow && relevant) {
        // up to 8 shadow cells, their visits counted independently
        const int b0 = a.sstart[ba * a.b_el + be], nsh = a.sstart[ba * a.b_el + be + 1] - b0;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          if (k >= nsh) break;
          const char4 o = reinterpret_cast<const char4*>(a.sxyz)[b0 + k];
          const int64_t lgx = a.xm.local(cx + o.x);
          if (lgx >= 0)
            shadow_add(&a.cells.y[(lgx * a.ny + (cy + o.y)) * a.nzp + (cz + o.z)], (uint32_t)a.h_max,
                       (uint32_t)a.t_occ);
        }
      }
      if (a.first_return) atomicMin(&a.hmin[h], (uint32_t)i);
      a.slot[i] = (uint32_t)h;
      if (!relevant) packed |= kRemote;  // the shadow kernel counts it, visits nothing
    }
    a.center[i] = packed;
    if (a.outcome) a.outcome[i] = ok ? 1 : 0;
  }
  // Launch-wide counters are aggregated per block: one atomic per block and
  // counter instead of one per warp (same-address atomics serialise at L2).
  __shared__ unsigned w_app[kPrepThreads / 32], w_clm[kPrepThreads / 32], w_ok[kPrepThreads / 32],
      w_fb[kPrepThreads / 32];
  __shared__ int w_scan[kPrepThreads / 32];
  __shared__ unsigned long long blk_base;
  const int warp = threadIdx.x >> 5, nwarps = kPrepThreads / 32;
  const unsigned app = __ballot_sync(0xffffffffu, append);
  const unsigned clm = __ballot_sync(0xffffffffu, claimed);
  const unsigned act = __ballot_sync(0xffffffffu, live);
  const unsigned okm = __ballot_sync(0xffffffffu, live && ok);
  const unsigned fbm = __ballot_sync(0xffffffffu, live && ok && fallback);
  // the scan of this warp's returns, -1 when they span several scans
  const int s0 = act ? __shfl_sync(0xffffffffu, s, __ffs(act) - 1) : 0;
  const bool uniform = __all_sync(0xffffffffu, !live || s == s0);
  if (lane == 0) {
    w_app[warp] = __popc(app);
    w_clm[warp] = __popc(clm);
    w_ok[warp] = __popc(okm);
    w_fb[warp] = __popc(fbm);
    w_scan[warp] = !act ? -2 : (uniform ? s0 : -1);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned napp = 0, nclm = 0, nok = 0, nfb = 0;
    int sb = -2;
    bool same = true;
    for (int w = 0; w < nwarps; ++w) {
      napp += w_app[w];
      nclm += w_clm[w];
      nok += w_ok[w];
      nfb += w_fb[w];
      if (w_scan[w] == -2) continue;
      if (sb == -2) sb = w_scan[w];
      same = same && w_scan[w] == sb && sb >= 0;
    }
    blk_base = napp ? atomicAdd(&a.lc->n_unique, (unsigned long long)napp) : 0ull;
    if (nclm) atomicAdd(&a.lc->skipped, (unsigned long long)nclm);
    if (same && sb >= 0) {
      if (nok) atomicAdd(&a.sc[sb].n_ok, (unsigned long long)nok);
      if (nfb) atomicAdd(&a.sc[sb].n_fallback, (unsigned long long)nfb);
      w_scan[0] = -3;  // counted for the whole block
    }
  }
  __syncthreads();
  // sweep work items at this warp's offset inside the block's range
  if (append) {
    unsigned long long off = blk_base;
    for (int w = 0; w < warp; ++w) off += w_app[w];
    a.uniq[off + __popc(app & ((1u << lane) - 1u))] = packed;
  }
  if (w_scan[0] != -3 && live) {
    // the block spans several scans: per-scan counters per warp (or thread)
    if (uniform) {
      if (lane == __ffs(act) - 1) {
        if (okm) atomicAdd(&a.sc[s0].n_ok, (unsigned long long)__popc(okm));
        if (fbm) atomicAdd(&a.sc[s0].n_fallback, (unsigned long long)__popc(fbm));
      }
    } else {
      if (ok) atomicAdd(&a.sc[s].n_ok, 1ull);
      if (ok && fallback) atomicAdd(&a.sc[s].n_fallback, 1ull);
    }
  }
}

struct ShadowArgs {
  Cells cells;
  const uint64_t* center;
  const uint16_t* bin;
  const uint32_t* slot;
  const uint32_t* hmin;
  const int8_t* sxyz;
  const int32_t* sstart;
  int64_t n;
  int log2s;  // threads per return = 1 << log2s >= max shadow count
  int64_t x0, x1, ny, nzp;
  XMap xm;
  int h_max, t_occ;
  int first_return;
  int S;
  const int64_t* scan_off;
  ScanCounters* sc;
  LaunchCounters* lc;
  // shadow_bin_kernel: rays from prep, bin table geometry
  const double* ray;
  int b_az, b_el;
  const uint16_t* seeds;
};

__global__ void __launch_bounds__(256) shadow_kernel(ShadowArgs a) {
  const int64_t total = a.n << a.log2s;
  const int64_t smask = (1ll << a.log2s) - 1;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = t >> a.log2s;
    int k = (int)(t & smask);
    uint64_t c = a.center[i];
    if (c == kEmptyKey) continue;
    if (a.first_return) {
      if (a.hmin[a.slot[i]] != (uint32_t)i) continue;
      if (k == 0) {
        // one atomic per group of lanes counting the same scan
        const int s = a.S > 1 ? find_scan(a.scan_off, a.S, i) : 0;
        const unsigned grp = __match_any_sync(__activemask(), s);
        if ((threadIdx.x & 31) == __ffs(grp) - 1) atomicAdd(&a.sc[s].n_applied, (unsigned long long)__popc(grp));
      }
    }
    if (c & kRemote) continue;
    int b = a.bin[i];
    int st = a.sstart[b];
    if (k >= a.sstart[b + 1] - st) continue;
    char4 o = reinterpret_cast<const char4*>(a.sxyz)[st + k];
    int64_t cx, cy, cz;
    unpack_center(c, cx, cy, cz);
    const int64_t lgx = a.xm.local(cx + o.x);
    if (lgx < 0) continue;
    shadow_add(&a.cells.y[(lgx * a.ny + (cy + o.y)) * a.nzp + (cz + o.z)], (uint32_t)a.h_max,
               (uint32_t)a.t_occ);
  }
}

// Shadow update with the direction bins computed here (prep skips them, so
// the sweep starts earlier; this kernel runs beside the sweep). A block takes
// tiles of 256 >> log2s returns: phase 1, one thread per return, bins the
// ray prep stored (bin_dev on the same doubles) and applies the first-return
// choice; phase 2, one thread per (return, shadow offset), counts the visit
// as shadow_kernel does.
__global__ void __launch_bounds__(256) shadow_bin_kernel(ShadowArgs a) {
  __shared__ uint64_t s_c[256];
  __shared__ uint16_t s_b[256];
  // returns per tile: 256 >> log2s (one visit per thread), at least 64 (the
  // binning phase keeps two warps busy; the visits then take several passes)
  const int per = max(64, 256 >> a.log2s);
  const int smask = (1 << a.log2s) - 1;
  const int64_t tiles = (a.n + per - 1) / per;
  for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
    const int64_t r0 = tile * per;
    if ((int)threadIdx.x < per) {
      const int64_t i = r0 + threadIdx.x;
      uint64_t c = i < a.n ? a.center[i] : kEmptyKey;
      if (c != kEmptyKey && a.first_return) {
        if (a.hmin[a.slot[i]] != (uint32_t)i) {
          c = kEmptyKey;
        } else {
          // one atomic per group of lanes counting the same scan
          const int sc = a.S > 1 ? find_scan(a.scan_off, a.S, i) : 0;
          const unsigned grp = __match_any_sync(__activemask(), sc);
          if ((threadIdx.x & 31) == __ffs(grp) - 1) atomicAdd(&a.sc[sc].n_applied, (unsigned long long)__popc(grp));
        }
      }
      uint16_t bin = 0;
      if (c != kEmptyKey && (c & kRemote)) c = kEmptyKey;  // counted above; no visits here
      if (c != kEmptyKey) {
        const double rx = a.ray[3 * i], ry = a.ray[3 * i + 1], rz = a.ray[3 * i + 2];
        int ba, be, fb;
        bin_dev(rx, ry, rz, ray_norm(rx, ry, rz), a.b_az, a.b_el, a.seeds, ba, be, fb);
        bin = (uint16_t)(ba * a.b_el + be);
        if (fb) atomicAdd(&a.sc[a.S > 1 ? find_scan(a.scan_off, a.S, i) : 0].n_fallback, 1ull);  // rare
      }
      s_c[threadIdx.x] = c;
      s_b[threadIdx.x] = bin;
    }
    __syncthreads();
    for (int pair = threadIdx.x; pair < (per << a.log2s); pair += 256) {
      const int j = pair >> a.log2s, k = pair & smask;
      const uint64_t c = s_c[j];
      if (c == kEmptyKey) continue;
      const int b = s_b[j];
      const int st = a.sstart[b];
      if (k < a.sstart[b + 1] - st) {
        const char4 o = reinterpret_cast<const char4*>(a.sxyz)[st + k];
        int64_t cx, cy, cz;
        unpack_center(c, cx, cy, cz);
        const int64_t lgx = a.xm.local(cx + o.x);
        if (lgx >= 0)
          shadow_add(&a.cells.y[(lgx * a.ny + (cy + o.y)) * a.nzp + (cz + o.z)], (uint32_t)a.h_max,
                     (uint32_t)a.t_occ);
      }
    }
    __syncthreads();  // s_c / s_b are rewritten by the next tile
  }
}

// Length-cache lowering of one 8-voxel chunk of a kernel row (engine.cuh):
// w = the 8 cached lengths (16-bit lanes), d8 = the row's 8 run lengths + 1
// (bytes, 64 outside the kernel). Per 16-bit lane (L | 0x8000) - (d + 1)
// never borrows across lanes (L <= 32, d + 1 <= 64) and its bit 15 is set
// exactly when d < L: the return lowers that voxel. A chunk with a lowered
// voxel takes ONE REDG.MIN.F16x8 of its 8 run lengths (a lane that does not
// lower holds d >= L, a no-op under MIN); returns the lowered voxels.
__device__ __forceinline__ void red_min_len8(uint16_t* p, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
  asm volatile("red.global.min.noftz.v4.f16x2 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(a), "r"(b), "r"(c), "r"(d));
}
__device__ __forceinline__ unsigned lower_chunk(uint16_t* p, uint4 w, uint2 d8) {
  constexpr uint32_t H = 0x80008000u, O = 0x00010001u;
  // the table bytes as 16-bit lanes: d + 1
  const uint32_t t0 = __byte_perm(d8.x, 0u, 0x7170), t1 = __byte_perm(d8.x, 0u, 0x7372);
  const uint32_t t2 = __byte_perm(d8.y, 0u, 0x7170), t3 = __byte_perm(d8.y, 0u, 0x7372);
  const uint32_t l0 = ((w.x | H) - t0) & H, l1 = ((w.y | H) - t1) & H;
  const uint32_t l2 = ((w.z | H) - t2) & H, l3 = ((w.w | H) - t3) & H;
  const uint32_t lt = l0 | (l1 >> 1) | (l2 >> 2) | (l3 >> 3);
  if (!lt) return 0u;
  red_min_len8(p, t0 - O, t1 - O, t2 - O, t3 - O);
  return (unsigned)__popc(lt);
}

struct SweepArgs {
  Cells cells;
  uint16_t* dist;
  const uint64_t* uniq;
  const LaunchCounters* lc_in;
  unsigned long long* changed_out;
  const uint2* dtab;      // [8][nd][CH]
  const uint16_t* rowd;   // [rows] distinct id * CH
  const int32_t* rowoff;  // [rows]
  int K, R, nd;
  int64_t x0, x1, ny, nzp;
  XMap xm;
};

constexpr int kSweepUnroll = 4;

// Warp per unique centre. Chunks of 8 voxels along z, row-major over the
// K*K kernel rows (row = (dx+R)*K + (dy+R)); a 21-voxel row is 3 or 4 64-bit
// loads of the distance cache depending on the centre's z alignment. Each
// lane issues kSweepUnroll independent loads before testing any of them (the
// updates below could alias later loads, so the compiler would not hoist
// them). A byte lane with d < cached bit length marks a voxel this return
// lowers: RED.AND of run_mask(d) into its record's mask word, then d goes to
// the cache. Stale cache reads (L1) only cause redundant ANDs, never missed
// ones (cache >= bit length of the mask, see engine.cuh).
template <int CH>
__global__ void __launch_bounds__(256) sweep_kernel(SweepArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int rows = a.K * a.K;
  const int ntab = 8 * a.nd * CH;
  uint2* dtab = reinterpret_cast<uint2*>(smem_raw);
  // per kernel row: {voxel offset of the row, index of its d-row in the table}
  int2* rowinfo = reinterpret_cast<int2*>(dtab + ntab);
  for (int i = threadIdx.x; i < ntab; i += blockDim.x) dtab[i] = a.dtab[i];
  for (int i = threadIdx.x; i < rows; i += blockDim.x) rowinfo[i] = make_int2(a.rowoff[i], a.rowd[i]);
  __syncthreads();

  const int64_t n_unique = (int64_t)a.lc_in->n_unique;
  const int64_t per = (n_unique + gridDim.x - 1) / gridDim.x;
  const int64_t lo = blockIdx.x * per;
  const int64_t hi = min(lo + per, n_unique);
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  unsigned long long changed = 0;

  for (int64_t u = lo + warp; u < hi; u += nwarps) {
    int64_t cx, cy, cz;
    unpack_center(a.uniq[u], cx, cy, cz);
    const int64_t zs = cz - a.R;  // >= 0: boundary discard guarantees it
    const int sh = (int)(zs & 7);
    // chunks this alignment needs per row (3 or 4 for K = 21); j -> row by a
    // 16-bit reciprocal (exact for j < 2^15)
    const int nch = (sh + a.K + 7) >> 3;
    const uint32_t magic = (65536u + nch - 1) / nch;
    const bool ilv = a.xm.w != 0;  // interleaved slabs: x-planes mapped per row
    const int64_t sx = a.ny * a.nzp;
    const int64_t base0 = cy * a.nzp + (zs & ~int64_t(7));
    const int64_t base = ilv ? base0 : (cx - a.x0) * sx + base0;
    // slab clip (multi-GPU): rows are dx-major, so the owned dx range of a
    // contiguous slab is a contiguous range of chunk indices
    const int64_t dxlo = ilv ? -a.R : max((int64_t)-a.R, a.x0 - cx);
    const int64_t dxhi = ilv ? a.R : min((int64_t)a.R, a.x1 - 1 - cx);
    if (dxlo > dxhi) continue;
    const int jlo = (int)((dxlo + a.R) * a.K * nch);
    const int jhi = (int)((dxhi + a.R + 1) * a.K * nch);
    const uint2* dt = dtab + sh * a.nd * CH;
    for (int j0 = jlo + lane; j0 < jhi; j0 += 32 * kSweepUnroll) {
      uint4 w[kSweepUnroll];
      uint2 d8[kSweepUnroll];
      int64_t off[kSweepUnroll];
#pragma unroll
      for (int k = 0; k < kSweepUnroll; ++k) {
        const int j = j0 + 32 * k;
        bool v = j < jhi;
        const int jj = v ? j : jlo;
        const int row = (int)(((uint32_t)jj * magic) >> 16);
        const int ch = jj - row * nch;
        const int2 ri = rowinfo[row];
        off[k] = base + ri.x + 8 * ch;
        if (ilv) {
          // row offset = dx*sx + dy*nzp: swap the dx plane for its storage plane
          const int dx = row / a.K - a.R;
          const int64_t lgx = a.xm.local(cx + dx);
          v = v && lgx >= 0;
          off[k] = v ? lgx * sx + (ri.x - dx * sx) + base0 + 8 * ch : 0;
        }
        d8[k] = v ? dt[ri.y + ch] : make_uint2(0x40404040u, 0x40404040u);
        w[k] = *reinterpret_cast<const uint4*>(a.dist + off[k]);
      }
#pragma unroll
      for (int k = 0; k < kSweepUnroll; ++k) changed += lower_chunk(a.dist + off[k], w[k], d8[k]);
    }
  }
  for (int o = 16; o; o >>= 1) changed += __shfl_xor_sync(0xffffffffu, changed, o);
  if (lane == 0 && changed) atomicAdd(a.changed_out, changed);
}

// Culling sweep for isotropic kernels (run length = h(|o|^2), h
// non-decreasing: every bank build_kernel_bank makes). A centre c may skip
// voxel v when a neighbour centre e = c + delta (|delta|_inf = 1) whose stamp
// is applied or claimed (certificate bit set) covers v (v in e's K^3 window)
// and is strictly closer in real distance, |v - e| < |v - c|, i.e.
// 2 (v - c).delta > |delta|^2: then h(|v-e|^2) <= h(|v-c|^2), so e's AND
// already implies c's at v. Following "skips because of" strictly decreases
// the real distance to v, so the chain ends at a centre that does sweep v
// with a run length <= c's: the grid is exactly the unculled one. The
// certificate bits are static during the sweep (set by prep), so the rule is
// race-free.
//
// Per centre the surviving region is, for each kernel x-offset dx (lane), a
// dy interval (neighbours with delta_z = 0 cut whole rows) and per row a dz
// interval (delta_z = +-1 neighbours cut z prefixes/suffixes). A block takes
// kCullWarps centres at a time: phase A, one warp per centre, writes the
// surviving rows into a shared-memory queue of row tasks (row start, chunk
// range, d-table row), each lane its own column's rows at its prefix-sum
// offset; phase B, the whole block, sweeps the queued rows one thread
// per row (1-4 chunk loads in flight each), testing them as sweep_kernel
// does. Rows of a heavy centre (a fresh surface: nothing culled) thus spread
// over the block instead of serialising one warp.
struct CullArgs {
  Cells cells;
  uint16_t* dist;
  const uint64_t* uniq;
  LaunchCounters* lc;
  const uint2* dtab;     // [8][nd][CH]
  const uint16_t* rowd;  // [K*K] distinct id * CH
  const uint32_t* stamped;
  int K, R, nd, CH;
  int64_t x0, x1, nx, ny, nzp;
  XMap xm;
};

// L2 residency hints for the culling sweep: certificate words and
// distance-cache chunks are re-read by neighbouring centres, so their loads
// carry an evict_last policy (same-box A/B against no hints: config 4 +2.5 %,
// config 3 +5 %, config 2 +2.5 %). Tried and not kept: evict_first on the
// record RED.ANDs (config 4 -1.5 %), evict_last on prep's certificate claims
// (neutral).
__device__ __forceinline__ uint64_t l2_policy_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
// not volatile: the policy is a constant, so one CREATEPOLICY per thread is
// hoisted out of the loops (it was 6 % of the sweep's instructions re-created
// at every load)
__device__ __forceinline__ uint64_t l2_policy_last() {
  uint64_t p;
#ifdef DBT_POLICY_VOLATILE
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
#else
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
#endif
  return p;
}
__device__ __forceinline__ uint32_t ld_cert(const uint32_t* p) {
#ifndef DBT_NO_HINT_CERT_EL
  uint32_t v;
  asm volatile("ld.global.cg.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(v) : "l"(p), "l"(l2_policy_last()));
  return v;
#else
  return __ldcg(p);
#endif
}
__device__ __forceinline__ uint4 ld_dist(const uint16_t* p) {
#ifndef DBT_NO_HINT_DIST_EL
  uint4 v;
  asm volatile("ld.global.L2::cache_hint.v4.u32 {%0, %1, %2, %3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(l2_policy_last()));
  return v;
#else
  return *reinterpret_cast<const uint4*>(p);
#endif
}
constexpr int kFar = 1 << 20;
// phase A row emission: balanced over the warp's lanes when
// ceil(rows / 32) * NUM < max rows per column * DEN (A/B knobs)
#ifndef DBT_ROWS_BAL_NUM
#define DBT_ROWS_BAL_NUM 5
#endif
#ifndef DBT_ROWS_BAL_DEN
#define DBT_ROWS_BAL_DEN 3
#endif
#ifndef DBT_PLANE_GATHER_BELOW
#define DBT_PLANE_GATHER_BELOW 8
#endif
constexpr int kPlaneGatherBelow = DBT_PLANE_GATHER_BELOW;  // certified adjacent centres below which plane neighbours are read
// centres per block batch (one warp each), 32 resident warps per SM at 64
// registers. With the divergent certificate gather 8 (4 blocks per SM) beat 4
// (config 2 +8.5 %, config 3 +11 %); since the gather became one instruction
// stream, 4 centres per batch (8 blocks of 128 threads per SM: shorter
// barriers, finer work fetch) win: same-box A/B 4 vs 8: config 4 +3.2 %,
// config 5 (32 scans) +3.5 %, config 3 +0.7 %, configs 1-2 within 1 %; 2, 3,
// 5, 6 and 16 are slower (profiles/README.md, s5_ab4 / s5_ab5)
#ifndef DBT_CULL_WARPS
#define DBT_CULL_WARPS 4
#endif
constexpr int kCullWarps = DBT_CULL_WARPS;

// row task: bits 0-36 row start / 8 (cells), 37-38 first chunk, 39-40 last
// chunk, 41-54 d-table row offset
__device__ __forceinline__ uint64_t pack_task(int64_t rbase, int c0, int c1, int drow) {
  return (uint64_t)(rbase >> 3) | ((uint64_t)c0 << 37) | ((uint64_t)c1 << 39) | ((uint64_t)drow << 41);
}

// Row-task writers of phase A. Put64: one 64-bit task per surviving row
// (absolute row start, chunk range, d-table row); kEmptyKey for a row whose
// dz interval is empty.
struct Put64 {
  uint64_t* queue;
  // ch = row start / 8 (the low word of the task: a grid has < 2^35 cells,
  // checked at launch), built with 32-bit arithmetic per row
  __device__ __forceinline__ void operator()(int i, bool valid, int, int c0, int c1, uint32_t ch,
                                             const uint16_t* rowd, int drow0) const {
    const uint32_t hi = ((uint32_t)c0 << 5) | ((uint32_t)c1 << 7) | ((uint32_t)(drow0 + __ldg(rowd)) << 9);
    reinterpret_cast<uint2*>(queue)[i] = valid ? make_uint2(ch, hi) : make_uint2(~0u, ~0u);
  }
};
struct NoInfo {
  __device__ __forceinline__ void operator()(int, int64_t, int64_t, int) const {}
};

// Phase A of the culling sweep for one centre (one warp): neighbour
// certificates -> per-lane dy interval and per-row dz interval -> the
// surviving row tasks, reserved as one range of `total` slots through *q_n
// (lane 0) and written with put(slot, task) (kEmptyKey for a row whose dz
// interval is empty).
// The certificates phase A cuts with (one warp, every lane gets the same
// bits): the 26 adjacent centres (nb, bit (a+1)*9 + (b+1)*3 + (c+1), bit 13
// cleared), the axis neighbours at distance 2-5 (axm) and, for sparse
// neighbourhoods, the norm-2 plane neighbours (plm).
__device__ __forceinline__ void gather_certs(const CullArgs& a, int64_t cx, int64_t cy, int64_t cz, int lane,
                                             uint32_t& nb, uint32_t& axm, uint32_t& plm) {
  // neighbour certificates: 27 bits, bit (a+1)*9 + (b+1)*3 + (c+1)
  uint32_t nb3 = 0;
  if (lane < 9) {
    const int na = lane / 3 - 1, nbb = lane % 3 - 1;
    const int64_t gx = cx + na;  // certificates: global planes (boundary discard keeps it in the grid)
    {
      const int64_t idx = (gx * a.ny + (cy + nbb)) * a.nzp + (cz - 1);
      const uint32_t w0 = ld_cert(a.stamped + (idx >> 5));
      const uint32_t w1 = ((idx & 31) > 29) ? ld_cert(a.stamped + (idx >> 5) + 1) : 0u;
      nb3 = (__funnelshift_r(w0, w1, (int)(idx & 31)) & 7u) << (3 * lane);
    }
  }
  // axis neighbours at distance k = 2..5 (sparse returns: the next beam
  // or azimuth step is often several voxels away): c + k e_x (lanes
  // 9-16), c + k e_y (lanes 17-24), c + k e_z (lane 25: the centre row's
  // bits cz-5 .. cz+5). Each cuts the half-space 2 k o_axis > k^2, i.e.
  // o_axis >= k/2 + 1 on its side (inside its window: o_axis >= k - R).
  // Bits: 4 per direction (k = 2..5): x+ 0-3, x- 4-7, y+ 8-11, y- 12-15,
  // z+ 16-19, z- 20-23.
  uint32_t ax = 0;
  if (lane >= 9 && lane < 25) {
    const int j = (lane - 9) & 7, k = 2 + (j & 3), sg = j < 4 ? 1 : -1;
    const bool along_x = lane < 17;
    const int64_t qx = along_x ? cx + sg * k : cx, qy = along_x ? cy : cy + sg * k;
    if (qy >= 0 && qy < a.ny && qx >= 0 && qx < a.nx) {
      const int64_t idx = (qx * a.ny + qy) * a.nzp + cz;
      ax = ((ld_cert(a.stamped + (idx >> 5)) >> (idx & 31)) & 1u) << (lane - 9);
    }
  } else if (lane == 25 && cz >= 5 && cz + 5 < a.nzp) {  // padding bits are never set
    {
      const int64_t idx = (cx * a.ny + cy) * a.nzp + (cz - 5);
      const uint32_t w0 = ld_cert(a.stamped + (idx >> 5));
      const uint32_t w1 = ((idx & 31) > 21) ? ld_cert(a.stamped + (idx >> 5) + 1) : 0u;
      const uint32_t b11 = __funnelshift_r(w0, w1, (int)(idx & 31)) & 0x7FFu;  // bit i: cz - 5 + i
      const uint32_t up = (b11 >> 7) & 0xFu;                                // cz+2 .. cz+5
      const uint32_t dn = __brev(b11 & 0xFu) >> 28;                         // cz-2 .. cz-5
      ax = (up << 16) | (dn << 20);
    }
  }
  nb = __reduce_or_sync(0xffffffffu, nb3) & ~(1u << 13);  // not c itself
  axm = __reduce_or_sync(0xffffffffu, ax);
  // sparse neighbourhood (few of the 26 adjacent centres certified): also
  // gather the norm-2 plane neighbours below (a second round of loads,
  // skipped for dense surfaces where they add little)
  plm = 0;
  if (__popc(nb) < kPlaneGatherBelow) {
    // plane neighbours of norm 2 with one zero coordinate besides the
    // axes: (a, b, 0) (lanes 0-11, bit cz) and (a, 0, c) (lanes 12-15: rows
    // cx+1, cx-1, cx+2, cx-2 at bits cz-2 .. cz+2). Their cuts are
    // constant per lane (a dy interval or a dz threshold). Index i of
    // either list: |a|,|b| = (2,1) for i < 4, (1,2) for i < 8, (2,2) else;
    // first sign + for even i>>1, second sign + for even i.
    uint32_t plb = 0;
    if (lane < 12) {
      const int g = lane >> 2, sa = (lane & 2) ? -1 : 1, sb = (lane & 1) ? -1 : 1;
      const int pa = sa * (g == 1 ? 1 : 2), pb = sb * (g == 0 ? 1 : 2);
      const int64_t qy = cy + pb, qx = cx + pa;
      if (qy >= 0 && qy < a.ny && qx >= 0 && qx < a.nx) {
        const int64_t idx = (qx * a.ny + qy) * a.nzp + cz;
        plb = ((ld_cert(a.stamped + (idx >> 5)) >> (idx & 31)) & 1u) << lane;
      }
    } else if (lane < 16 && cz >= 2 && cz + 2 < a.nzp) {
      const int pa = lane == 12 ? 1 : lane == 13 ? -1 : lane == 14 ? 2 : -2;
      const int64_t qx = cx + pa;
      if (qx >= 0 && qx < a.nx) {
        const int64_t idx = (qx * a.ny + cy) * a.nzp + (cz - 2);
        const uint32_t w0 = ld_cert(a.stamped + (idx >> 5));
        const uint32_t w1 = ((idx & 31) > 27) ? ld_cert(a.stamped + (idx >> 5) + 1) : 0u;
        const uint32_t b5 = __funnelshift_r(w0, w1, (int)(idx & 31)) & 0x1Fu;  // bit i: cz - 2 + i
        const uint32_t cp1 = (b5 >> 3) & 1u, cm1 = (b5 >> 1) & 1u, cp2 = (b5 >> 4) & 1u, cm2 = b5 & 1u;
        uint32_t xz = 0;
        if (lane == 12) xz = (cp2 << 4) | (cm2 << 5);
        if (lane == 13) xz = (cp2 << 6) | (cm2 << 7);
        if (lane == 14) xz = cp1 | (cm1 << 1) | (cp2 << 8) | (cm2 << 9);
        if (lane == 15) xz = (cp1 << 2) | (cm1 << 3) | (cp2 << 10) | (cm2 << 11);
        plb = xz << 12;
      }
    }
    plm = __reduce_or_sync(0xffffffffu, plb);
  }
}

// The same gather with one instruction stream for all lanes (kernels with
// R >= 5, grids whose y-z plane offsets fit 32 bits): every neighbour read is
// "nbits certificate bits starting at voxel c + (ox, oy, oz)", so each lane
// derives its offset and width from its index and all lanes run the index
// arithmetic, the one or two loads and the extraction together, instead of
// the 3 + 2 divergent lane groups of gather_certs (15 % of the sweep's
// instructions at 12-15 active lanes). R >= 5 puts every neighbour read inside
// the grid (boundary discard: c +- R is in the grid), so no bounds checks.
// Returns the same nb / axm / plm.
__device__ __forceinline__ void gather_certs_uniform(const CullArgs& a, int64_t cx, int64_t cy, int64_t cz, int lane,
                                                     uint32_t& nb, uint32_t& axm, uint32_t& plm) {
  const int ny = (int)a.ny, nzp = (int)a.nzp;
  const int64_t base = (cx * a.ny + cy) * a.nzp + cz;
  // round 1: lanes 0-8 the 3x3 columns (3 bits from cz-1), lanes 9-24 the
  // x / y axis neighbours at k = 2..5 (1 bit), lane 25 the centre column
  // (11 bits from cz-5)
  int ox = 0, oy = 0, oz = 0, nbits = 1;
  if (lane < 9) {
    ox = lane / 3 - 1;
    oy = lane % 3 - 1;
    oz = -1;
    nbits = 3;
  } else if (lane < 25) {
    const int j = (lane - 9) & 7, k = 2 + (j & 3), sk = j < 4 ? k : -k;
    ox = lane < 17 ? sk : 0;
    oy = lane < 17 ? 0 : sk;
  } else {
    oz = -5;
    nbits = 11;
  }
  uint32_t bits = 0;
  if (lane < 26) {
    const int64_t idx = base + ((ox * ny + oy) * nzp + oz);
    const int sft = (int)(idx & 31);
    const uint32_t* wp = a.stamped + (idx >> 5);
    const uint32_t w0 = ld_cert(wp);
    const uint32_t w1 = sft + nbits > 32 ? ld_cert(wp + 1) : 0u;
    bits = __funnelshift_r(w0, w1, sft) & ((1u << nbits) - 1u);
  }
  const uint32_t nbc = lane < 9 ? bits << (3 * lane) : 0u;
  uint32_t axc = (lane >= 9 && lane < 25) ? bits << (lane - 9) : 0u;
  if (lane == 25) axc = (((bits >> 7) & 0xFu) << 16) | ((__brev(bits & 0xFu) >> 28) << 20);
  nb = __reduce_or_sync(0xffffffffu, nbc) & ~(1u << 13);  // not c itself
  axm = __reduce_or_sync(0xffffffffu, axc);
  plm = 0;
  if (__popc(nb) < kPlaneGatherBelow) {
    // round 2: lanes 0-11 the (a, b, 0) plane neighbours (1 bit at cz),
    // lanes 12-15 the columns cx+1, cx-1, cx+2, cx-2 (5 bits from cz-2)
    uint32_t plb = 0;
    if (lane < 16) {
      int px, py = 0, pz = 0, pbits = 1;
      if (lane < 12) {
        const int g = lane >> 2, sa = (lane & 2) ? -1 : 1, sb = (lane & 1) ? -1 : 1;
        px = sa * (g == 1 ? 1 : 2);
        py = sb * (g == 0 ? 1 : 2);
      } else {
        px = lane == 12 ? 1 : lane == 13 ? -1 : lane == 14 ? 2 : -2;
        pz = -2;
        pbits = 5;
      }
      const int64_t idx = base + ((px * ny + py) * nzp + pz);
      const int sft = (int)(idx & 31);
      const uint32_t* wp = a.stamped + (idx >> 5);
      const uint32_t w0 = ld_cert(wp);
      const uint32_t w1 = sft + pbits > 32 ? ld_cert(wp + 1) : 0u;
      const uint32_t b = __funnelshift_r(w0, w1, sft) & ((1u << pbits) - 1u);
      if (lane < 12) {
        plb = b << lane;
      } else {  // bit i of b: cz - 2 + i
        const uint32_t cp1 = (b >> 3) & 1u, cm1 = (b >> 1) & 1u, cp2 = (b >> 4) & 1u, cm2 = b & 1u;
        const uint32_t xz = lane == 12   ? (cp2 << 4) | (cm2 << 5)
                            : lane == 13 ? (cp2 << 6) | (cm2 << 7)
                            : lane == 14 ? cp1 | (cm1 << 1) | (cp2 << 8) | (cm2 << 9)
                                         : (cp1 << 2) | (cm1 << 3) | (cp2 << 10) | (cm2 << 11);
        plb = xz << 12;
      }
    }
    plm = __reduce_or_sync(0xffffffffu, plb);
  }
}

template <typename Put, typename Info>
__device__ __forceinline__ void cull_centre(const CullArgs& a, uint64_t centre, int lane, int* q_n, Put put, Info info) {
  const int R = a.R, K = a.K;
  const int64_t sx = a.ny * a.nzp;
  const uint16_t* rowd = a.rowd;
  int64_t cx, cy, cz;
  unpack_center(centre, cx, cy, cz);
  uint32_t nb, axm, plm;
#if defined(DBT_GATHER_DIVERGENT)
  gather_certs(a, cx, cy, cz, lane, nb, axm, plm);
#else
  if (a.R >= 5 && a.ny * a.nzp < (int64_t(1) << 28)) {
    gather_certs_uniform(a, cx, cy, cz, lane, nb, axm, plm);
#if defined(DBT_GATHER_CHECK)
    uint32_t nb2, axm2, plm2;
    gather_certs(a, cx, cy, cz, lane, nb2, axm2, plm2);
    if (nb != nb2 || axm != axm2 || plm != plm2) __trap();
#endif
  } else {
    gather_certs(a, cx, cy, cz, lane, nb, axm, plm);
  }
#endif
#define NB(A, B, C) ((nb >> (((A) + 1) * 9 + ((B) + 1) * 3 + ((C) + 1))) & 1u)
  // per lane: kernel x-offset dx, its dy interval and z-cut terms
  const int dx = lane - R;
  const int64_t lgx = lane < K ? a.xm.local(cx + dx) : -1;
  bool dead = lgx < 0;
  const int64_t xbase = dead ? 0 : lgx * sx;  // storage offset of this lane's x-plane
  int ylo = -R, yhi = R;
  int mp[3] = {kFar, kFar, kFar}, mm[3] = {-kFar, -kFar, -kFar};  // index b + 1
#pragma unroll
  for (int na = -1; na <= 1; ++na) {
    const bool xw = na == 0 || (na > 0 ? dx >= -R + 1 : dx <= R - 1);  // v in e's x-window
    if (!xw) continue;
    const int s = na * dx;
    if (na != 0 && NB(na, 0, 0) && s >= 1) dead = true;  // delta_z = 0: whole rows
    const int t2 = na == 0 ? 1 : 2;                     // floor(|delta|^2 / 2) + 1
    if (NB(na, 1, 0)) yhi = min(yhi, max(t2 - s, -R + 1) - 1);
    if (NB(na, -1, 0)) ylo = max(ylo, min(s - t2, R - 1) + 1);
#pragma unroll
    for (int b = -1; b <= 1; ++b) {
      const int t3 = (na * na + b * b + 1) / 2 + 1;
      if (NB(na, b, 1)) mp[b + 1] = min(mp[b + 1], t3 - s);
      if (NB(na, b, -1)) mm[b + 1] = max(mm[b + 1], s - t3);
    }
  }
#undef NB
  // axis neighbours: per direction the nearest present k gives the cut
  // threshold thr = max(k / 2 + 1, k - R) (0 when none)
  int thr[6];
#pragma unroll
  for (int d = 0; d < 6; ++d) {
    const uint32_t bits = (axm >> (4 * d)) & 0xFu;
    const int k = bits ? 2 + (__ffs(bits) - 1) : 0;
    thr[d] = k ? max(k / 2 + 1, k - R) : 0;
  }
  if (thr[0] && dx >= thr[0]) dead = true;
  if (thr[1] && dx <= -thr[1]) dead = true;
  if (thr[2]) yhi = min(yhi, thr[2] - 1);
  if (thr[3]) ylo = max(ylo, 1 - thr[3]);
  if (thr[4]) mp[1] = min(mp[1], thr[4]);   // dz >= thr culled
  if (thr[5]) mm[1] = max(mm[1], -thr[5]);  // dz <= -thr culled
  // plane neighbours: (a, b, 0) cut b dy >= T - a dx, (a, 0, c) cut
  // c dz >= T - a dx, T = |delta|^2 / 2 + 1, each inside its window
#if defined(DBT_PLM_UNROLLED)
  if (plm) {
#pragma unroll
    for (int i = 0; i < 12; ++i) {
      const int g = i >> 2, s1 = (i & 2) ? -1 : 1, s2 = (i & 1) ? -1 : 1;
      const int pa = s1 * (g == 1 ? 1 : 2), q = s2 * (g == 0 ? 1 : 2);
      const bool xw = dx - pa <= R && pa - dx <= R;  // v inside e's x-window
      const int num = (g == 2 ? 5 : 3) - pa * dx;
      const int cdiv = g == 0 ? num : (num + 1) >> 1;  // ceil(num / |q|)
      if (xw && ((plm >> i) & 1u)) {  // (pa, q, 0): dy cut
        if (q > 0) yhi = min(yhi, max(cdiv, q - R) - 1);
        else ylo = max(ylo, min(-cdiv, R + q) + 1);
      }
      if (xw && ((plm >> (12 + i)) & 1u)) {  // (pa, 0, q): dz cut
        if (q > 0) mp[1] = min(mp[1], max(cdiv, q - R));
        else mm[1] = max(mm[1], min(-cdiv, R + q));
      }
    }
  }
#else
  // one pass per certified plane neighbour (plm is the same in every lane, so
  // the loop and the decode of its bit are warp-uniform; the unrolled,
  // predicated form ran all 24 cuts for every sparse centre)
  for (uint32_t m = plm; m; m &= m - 1) {
    const int bit = __ffs(m) - 1;
    const bool zcut = bit >= 12;  // (pa, 0, q): dz cut; else (pa, q, 0): dy cut
    const int i = zcut ? bit - 12 : bit;
    const int g = i >> 2, s1 = (i & 2) ? -1 : 1, s2 = (i & 1) ? -1 : 1;
    const int pa = s1 * (g == 1 ? 1 : 2), q = s2 * (g == 0 ? 1 : 2);
    const bool xw = dx - pa <= R && pa - dx <= R;  // v inside e's x-window
    const int num = (g == 2 ? 5 : 3) - pa * dx;
    const int cdiv = g == 0 ? num : (num + 1) >> 1;  // ceil(num / |q|)
    if (!xw) continue;
    if (!zcut) {
      if (q > 0) yhi = min(yhi, max(cdiv, q - R) - 1);
      else ylo = max(ylo, min(-cdiv, R + q) + 1);
    } else {
      if (q > 0) mp[1] = min(mp[1], max(cdiv, q - R));
      else mm[1] = max(mm[1], min(-cdiv, R + q));
    }
  }
#endif
  const int cnt = dead ? 0 : max(0, yhi - ylo + 1);
  int pre = cnt;  // inclusive scan
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, pre, o);
    if (lane >= o) pre += v;
  }
  const int total = __shfl_sync(0xffffffffu, pre, 31);
  pre -= cnt;  // exclusive
  const int64_t zs = cz - R;
  const int sh = (int)(zs & 7);
  const int64_t zb = zs >> 3;  // chunk index of the kernel's first chunk
  const int64_t cbase = cy * a.nzp + (zb << 3);
  // each lane writes its own column's rows at its prefix offset (no owner
  // search, no per-row shuffles); a row with an empty dz interval fills
  // its reserved slot with kEmptyKey
  int qb = 0;
  if (lane == 0 && total) qb = atomicAdd(q_n, total);
  qb = __shfl_sync(0xffffffffu, qb, 0);
  const int zhi0 = min(R, max(mp[1], -R + 1) - 1), zlo0 = max(-R, min(mm[1], R - 1) + 1);
  const int drow0 = sh * a.nd * a.CH;
  info(lane, xbase, cbase, drow0);
  // one row of column `col` (kernel x-offset col - R): its dz interval —
  // delta_z = +1 neighbours cut dz >= max(mp - b dy, -R+1), delta_z = -1
  // ones cut dz <= min(mm + b dy, R-1) (b = delta_y, only when v is in
  // their y-window) — and its task
  const int nzp8 = (int)(a.nzp >> 3);
  // chunk index of this lane's column at dy = 0 (xbase and cbase are multiples of 8)
  const uint32_t colch = (uint32_t)((xbase + cbase) >> 3);
  auto emit = [&](int slot, int col, int rdy, int z_hi0, int z_lo0, int mp0, int mm0, int mp2, int mm2,
                  uint32_t cch) {
    int zhi = z_hi0, zlo = z_lo0;
    if (rdy <= R - 1) {  // b = -1
      zhi = min(zhi, max(mp0 + rdy, -R + 1) - 1);
      zlo = max(zlo, min(mm0 - rdy, R - 1) + 1);
    }
    if (rdy >= -R + 1) {  // b = +1
      zhi = min(zhi, max(mp2 - rdy, -R + 1) - 1);
      zlo = max(zlo, min(mm2 + rdy, R - 1) + 1);
    }
    const bool valid = zlo <= zhi;
    const int c0 = (int)(((cz + zlo) >> 3) - zb), c1 = (int)(((cz + zhi) >> 3) - zb);
    put(qb + slot, valid, rdy, c0, c1, cch + (uint32_t)(rdy * nzp8), rowd + col * K + R + rdy, drow0);
  };
  const int cmax = __reduce_max_sync(0xffffffffu, (unsigned)cnt);
  if (((total + 31) >> 5) * DBT_ROWS_BAL_NUM < cmax * DBT_ROWS_BAL_DEN) {
    // few rows spread unevenly over the columns (a culled centre): the
    // warp's lanes take consecutive rows of the whole list, each finding its
    // column by a binary search over the inclusive prefix sums, instead of
    // every lane walking its own column (the loop would run max(cnt) times
    // with most lanes idle)
    const int incl = pre + cnt;
    for (int base = 0; base < total; base += 32) {
      const int j = base + lane;
      int col = 0;
#pragma unroll
      for (int step = 16; step; step >>= 1) {
        const int v = __shfl_sync(0xffffffffu, incl, col + step - 1);
        if (v <= j) col += step;
      }
      col &= 31;
      const int o_ylo = __shfl_sync(0xffffffffu, ylo, col), o_pre = __shfl_sync(0xffffffffu, pre, col);
      const int o_zhi0 = __shfl_sync(0xffffffffu, zhi0, col), o_zlo0 = __shfl_sync(0xffffffffu, zlo0, col);
      const int o_mp0 = __shfl_sync(0xffffffffu, mp[0], col), o_mm0 = __shfl_sync(0xffffffffu, mm[0], col);
      const int o_mp2 = __shfl_sync(0xffffffffu, mp[2], col), o_mm2 = __shfl_sync(0xffffffffu, mm[2], col);
      const uint32_t o_ch = __shfl_sync(0xffffffffu, colch, col);
      if (j < total) emit(j, col, o_ylo + (j - o_pre), o_zhi0, o_zlo0, o_mp0, o_mm0, o_mp2, o_mm2, o_ch);
    }
  } else {
    // each lane writes its own column's rows at its prefix offset
    for (int k = 0; k < cnt; ++k) emit(pre + k, lane, ylo + k, zhi0, zlo0, mp[0], mm[0], mp[2], mm[2], colch);
  }
}

// A decoded row task: row start (cells), first / last chunk (c1 = -1: no
// row), d-table row offset.
struct RowTask {
  int64_t rb;
  int c0, c1, drow;
};

__device__ __forceinline__ RowTask decode_task64(uint64_t task) {
  RowTask r;
  r.rb = (int64_t)(task & ((1ull << 37) - 1)) << 3;
  r.c0 = (int)((task >> 37) & 3);
  r.c1 = task != kEmptyKey ? (int)((task >> 39) & 3) : -1;
  r.drow = (int)(task >> 41);
  return r;
}

// Phase B of the culling sweep: one thread, two row tasks (c1 = -1: none)
// with their chunk loads in flight together; a cached length above the row's
// run length marks a voxel this centre lowers: one MIN reduction per lowered
// chunk on the length cache (lower_chunk).
__device__ __forceinline__ void sweep_rows2(const CullArgs& a, const RowTask rows[2], unsigned long long& changed,
                                            unsigned long long& rows_done) {
  uint4 w[2][4];
  int64_t rb[2];
  int cb[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    rows_done += rows[r].c1 >= 0;
    rb[r] = rows[r].rb;
    const int c0 = rows[r].c0, c1 = rows[r].c1;
    cb[r] = c0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      // inactive chunks read one shared dummy sector (predicated-off loads
      // measured 6 % slower on config 4: profiles/README.md, s5)
      w[r][j] = ld_dist(c0 + j <= c1 ? a.dist + rb[r] + 8 * (c0 + j) : a.dist);
    }
  }
  // the d-table (L1-resident) is read after the cache loads are in flight
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const uint2* drow = a.dtab + rows[r].drow + cb[r];
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (cb[r] + j > rows[r].c1) continue;
#if !defined(DBT_DIAG_NO_RED)
      changed += lower_chunk(a.dist + rb[r] + 8 * (cb[r] + j), w[r][j], __ldg(drow + j));
#endif
    }
  }
}

// 32 resident warps per SM (64 registers, a few bytes spilled): same-box A/B
// vs 28 (72 registers): config 2 +2.7 %, config 1 +5 %, config 3 neutral;
// 36 or 40 warps (56 / 48 registers) spill more and are slower
#ifndef DBT_CULL_MIN_BLOCKS
#define DBT_CULL_MIN_BLOCKS (32 / DBT_CULL_WARPS)
#endif
__global__ void __launch_bounds__(kCullWarps * 32, DBT_CULL_MIN_BLOCKS) sweep_cull_kernel(CullArgs a) {
  // launched programmatically behind prep_kernel: wait for its results
  asm volatile("griddepcontrol.wait;" ::: "memory");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  uint64_t* queue = reinterpret_cast<uint64_t*>(smem_raw);  // kCullWarps * K * K
  __shared__ int q_n;
  __shared__ long long batch0, batch_next;
  // the d-table (17 KB for K = 21) is read through L1 (__ldg), not staged
  if (threadIdx.x == 0) batch_next = (long long)atomicAdd(&a.lc->work, (unsigned long long)kCullWarps);

  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t n_items = (int64_t)a.lc->n_unique;
  unsigned long long changed = 0, rows_done = 0;
  while (true) {
    if (threadIdx.x == 0) {
      batch0 = batch_next;
      q_n = 0;
    }
    __syncthreads();
    const int64_t item = batch0 + warp;
    if (batch0 >= n_items) break;
    if (item < n_items) {
      cull_centre(a, a.uniq[item], lane, &q_n, Put64{queue}, NoInfo{});
    }
    __syncthreads();
    // next batch index: its atomic overlaps phase B
    if (threadIdx.x == 0) batch_next = (long long)atomicAdd(&a.lc->work, (unsigned long long)kCullWarps);
    // ===== phase B: the block sweeps the queued rows, one thread per row,
    // two rows' chunk loads in flight per thread =====
    const int nq = q_n;
    for (int i = threadIdx.x; i < nq; i += 2 * blockDim.x) {
      const RowTask rows[2] = {decode_task64(i < nq ? queue[i] : kEmptyKey),
                               decode_task64(i + (int)blockDim.x < nq ? queue[i + blockDim.x] : kEmptyKey)};
      sweep_rows2(a, rows, changed, rows_done);
    }
    __syncthreads();  // queue and batch0 are rewritten by the next batch
  }
  // one atomic per block and counter (same-address atomics serialise at L2)
  __shared__ unsigned long long blk_changed, blk_rows;
  if (threadIdx.x == 0) blk_changed = blk_rows = 0;
  for (int o = 16; o; o >>= 1) {
    changed += __shfl_xor_sync(0xffffffffu, changed, o);
    rows_done += __shfl_xor_sync(0xffffffffu, rows_done, o);
  }
  __syncthreads();
  if (lane == 0 && changed) atomicAdd(&blk_changed, changed);
  if (lane == 0 && rows_done) atomicAdd(&blk_rows, rows_done);
  __syncthreads();
  if (threadIdx.x == 0 && blk_changed) atomicAdd(&a.lc->changed, blk_changed);
  if (threadIdx.x == 0 && blk_rows) atomicAdd(&a.lc->rows, blk_rows);
}

// Warp-independent variant of the culling sweep (A/B: -DDBT_SWEEP_WARP): each
// warp fetches groups of centres and runs phase A and phase B for one centre
// at a time on its own shared-memory queue, with no block barrier (a heavy
// centre is swept by its own 32 lanes).
__global__ void __launch_bounds__(kCullWarps * 32, DBT_CULL_MIN_BLOCKS) sweep_warp_kernel(CullArgs a) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t* queue = reinterpret_cast<uint64_t*>(smem_raw) + warp * a.K * a.K;
  __shared__ int q_n[kCullWarps];
  const int64_t n_items = (int64_t)a.lc->n_unique;
  unsigned long long changed = 0, rows_done = 0;
  constexpr int G = 4;  // centres per work fetch
  long long next = 0;
  if (lane == 0) next = (long long)atomicAdd(&a.lc->work, (unsigned long long)G);
  next = __shfl_sync(0xffffffffu, next, 0);
  while (next < n_items) {
    const long long cur = next;
    if (lane == 0) next = (long long)atomicAdd(&a.lc->work, (unsigned long long)G);  // overlaps this group
    for (int k = 0; k < G && cur + k < n_items; ++k) {
      if (lane == 0) q_n[warp] = 0;
      __syncwarp();
      cull_centre(a, a.uniq[cur + k], lane, &q_n[warp], Put64{queue}, NoInfo{});
      __syncwarp();
      const int nq = q_n[warp];
      for (int i = lane; i < nq; i += 64) {
        const RowTask rows[2] = {decode_task64(queue[i]), decode_task64(i + 32 < nq ? queue[i + 32] : kEmptyKey)};
        sweep_rows2(a, rows, changed, rows_done);
      }
      __syncwarp();
    }
    next = __shfl_sync(0xffffffffu, next, 0);
  }
  __shared__ unsigned long long blk_changed, blk_rows;
  if (threadIdx.x == 0) blk_changed = blk_rows = 0;
  for (int o = 16; o; o >>= 1) {
    changed += __shfl_xor_sync(0xffffffffu, changed, o);
    rows_done += __shfl_xor_sync(0xffffffffu, rows_done, o);
  }
  __syncthreads();
  if (lane == 0 && changed) atomicAdd(&blk_changed, changed);
  if (lane == 0 && rows_done) atomicAdd(&blk_rows, rows_done);
  __syncthreads();
  if (threadIdx.x == 0 && blk_changed) atomicAdd(&a.lc->changed, blk_changed);
  if (threadIdx.x == 0 && blk_rows) atomicAdd(&a.lc->rows, blk_rows);
}

#if defined(DBT_SWEEP_WARP)
#define DBT_ISO_SWEEP sweep_warp_kernel
#else
#define DBT_ISO_SWEEP sweep_cull_kernel
#endif

typedef void (*SweepFn)(SweepArgs);

SweepFn sweep_fn(int CH) {
  switch (CH) {
    case 1: return sweep_kernel<1>;
    case 2: return sweep_kernel<2>;
    case 3: return sweep_kernel<3>;
    case 4: return sweep_kernel<4>;
    case 5: return sweep_kernel<5>;
    case 6: return sweep_kernel<6>;
  }
  return nullptr;
}

size_t sweep_smem_bytes(int K, int CH, int nd) {
  return (size_t)8 * nd * CH * sizeof(uint2) + (size_t)K * K * sizeof(int2);
}

__global__ void bin_kernel(const double* __restrict__ dirs, int64_t n, int b_az, int b_el,
                           const uint16_t* __restrict__ seeds, int64_t* __restrict__ oa,
                           int64_t* __restrict__ oe) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double x = dirs[3 * i], y = dirs[3 * i + 1], z = dirs[3 * i + 2];
    double nrm = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), __dmul_rn(z, z)));
    int ba, be, kn;
    bin_dev(x, y, z, nrm, b_az, b_el, seeds, ba, be, kn);
    oa[i] = ba;
    oe[i] = be;
  }
}

// ---------------------------------------------------------------- host side

// SVML seed table, uploaded once per device
const uint16_t* device_seeds(int device, int* rc) {
  static std::mutex mu;
  static uint16_t* tabs[64] = {nullptr};
  *rc = DBT_OK;
  if (device < 0 || device >= 64) {
    *rc = set_error(DBT_ERR_CONFIG, "device ordinal out of range");
    return nullptr;
  }
  std::lock_guard<std::mutex> lock(mu);
  if (!tabs[device]) {
    uint16_t* p = nullptr;
    cudaError_t e = cudaMalloc(&p, sizeof(dbt_svml_seeds));
    if (e == cudaSuccess) e = cudaMemcpy(p, dbt_svml_seeds, sizeof(dbt_svml_seeds), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      *rc = cuda_error(e, "svml seed table");
      return nullptr;
    }
    tabs[device] = p;
  }
  return tabs[device];
}

// The C library's sin/cos table for the deskew restatement (libm_emu.cuh):
// located in this process's libm, checked against its sin/cos on 200 000
// arguments, uploaded once per device. nullptr (and *rc) when the library
// cannot be matched (another libm build or dispatch variant).
const double* device_sincostab(int device, int* rc) {
  static std::mutex mu;
  static double* tabs[64] = {nullptr};
  static int host_state = 0;  // 0 unknown, 1 matched, -1 not matched
  static const double* host_tab = nullptr;
  *rc = DBT_OK;
  if (device < 0 || device >= 64) {
    *rc = set_error(DBT_ERR_CONFIG, "device ordinal out of range");
    return nullptr;
  }
  std::lock_guard<std::mutex> lock(mu);
  if (host_state == 0) {
    host_tab = libm_emu::find_sincostab();
    host_state = (host_tab && libm_emu::check_sincostab(host_tab) == 0) ? 1 : -1;
  }
  if (host_state < 0) {
    *rc = set_error(DBT_ERR_CONFIG, "device deskew unavailable: the C library's sin/cos do not match the restatement");
    return nullptr;
  }
  if (!tabs[device]) {
    double* p = nullptr;
    cudaError_t e = cudaMalloc(&p, libm_emu::kTabEntries * sizeof(double));
    if (e == cudaSuccess)
      e = cudaMemcpy(p, host_tab, libm_emu::kTabEntries * sizeof(double), cudaMemcpyHostToDevice);
    if (e != cudaSuccess) {
      *rc = cuda_error(e, "sin/cos table");
      return nullptr;
    }
    tabs[device] = p;
  }
  return tabs[device];
}

// deskewed float64 points of a (downsampled) scan (dbt_deskew_points)
__global__ void deskew_points_kernel(const void* pts, int dtype, int64_t n, int ds, const double* ts, dbt_deskew dk,
                                     const double* tab, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t src = i * ds;
    double p0, p1, p2;
    if (dtype == DBT_F32) {
      const float* q = (const float*)pts + 3 * src;
      p0 = q[0];
      p1 = q[1];
      p2 = q[2];
    } else {
      const double* q = (const double*)pts + 3 * src;
      p0 = q[0];
      p1 = q[1];
      p2 = q[2];
    }
    const double t = deskew::clip01(ts ? ts[src] : deskew::linspace01(i, n));
    int rare = 0;
    deskew::apply(dk, t, p0, p1, p2, out + 3 * i, tab, &rare);
    if (rare) out[3 * i] = CUDART_NAN;
  }
}

int check_deskew(const dbt_deskew* d) {
  if (!d) return set_error(DBT_ERR_CONFIG, "null deskew parameters");
  if (d->mode != DBT_DESKEW_YAW && d->mode != DBT_DESKEW_SE3)
    return set_error(DBT_ERR_CONFIG, "deskew mode must be DBT_DESKEW_YAW or DBT_DESKEW_SE3");
  return DBT_OK;
}

int grow(void** p, int64_t* cap, int64_t need, size_t elem) {
  if (need <= *cap) return DBT_OK;
  int64_t c = std::max<int64_t>(need, *cap + *cap / 2);
  if (*p) cudaFree(*p);
  *p = nullptr;
  *cap = 0;
  DBT_CUDA(cudaMalloc(p, (size_t)c * elem));
  *cap = c;
  return DBT_OK;
}

int ensure_points(dbt_grid* g, int64_t n) {
  if (n <= g->cap_pts) return DBT_OK;
  int64_t c = std::max<int64_t>(n, g->cap_pts + g->cap_pts / 2);
  void* ptrs[] = {g->d_center, g->d_bin, g->d_slot, g->d_ray};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (g->d_uniq) cudaFree(g->d_uniq);
  g->d_center = nullptr;
  g->d_bin = nullptr;
  g->d_slot = nullptr;
  g->d_uniq = nullptr;
  g->d_ray = nullptr;
  g->cap_pts = 0;
  DBT_CUDA(cudaMalloc(&g->d_center, c * sizeof(uint64_t)));
  DBT_CUDA(cudaMalloc(&g->d_bin, c * sizeof(uint16_t)));
  DBT_CUDA(cudaMalloc(&g->d_slot, c * sizeof(uint32_t)));
  DBT_CUDA(cudaMalloc(&g->d_uniq, c * sizeof(uint64_t)));
  DBT_CUDA(cudaMalloc(&g->d_ray, c * 3 * sizeof(double)));
  g->cap_pts = c;
  return DBT_OK;
}

int ensure_hash(dbt_grid* g, int64_t n) {
  int64_t want = 1024;
  while (want < 2 * n) want <<= 1;
  if (want <= g->cap_hash) return DBT_OK;
  if (g->d_hkey) cudaFree(g->d_hkey);
  if (g->d_hmin) cudaFree(g->d_hmin);
  g->d_hkey = nullptr;
  g->d_hmin = nullptr;
  g->cap_hash = 0;
  DBT_CUDA(cudaMalloc(&g->d_hkey, want * sizeof(unsigned long long)));
  DBT_CUDA(cudaMalloc(&g->d_hmin, want * sizeof(uint32_t)));
  DBT_CUDA(cudaMemset(g->d_hkey, 0, want * sizeof(unsigned long long)));  // epoch 0: never live
  g->hash_epoch = 0;
  g->cap_hash = want;
  return DBT_OK;
}

int ensure_rows(dbt_grid* g, const dbt_bank* b) {
  if (g->tab_bank == b->serial && g->d_rowoff) return DBT_OK;
  const int K = b->K, R = b->R, rows = K * K;
  std::vector<int32_t> ro(rows);
  for (int r = 0; r < rows; ++r) {
    int dx = r / K - R, dy = r % K - R;
    int64_t v = ((int64_t)dx * g->ny + dy) * g->nzp;
    if (v > INT32_MAX || v < INT32_MIN)
      return set_error(DBT_ERR_CONFIG, "grid too large in y*z for 32-bit kernel row offsets");
    ro[r] = (int32_t)v;
  }
  if (g->d_rowoff) cudaFree(g->d_rowoff);
  g->d_rowoff = nullptr;
  DBT_CUDA(cudaMalloc(&g->d_rowoff, rows * sizeof(int32_t)));
  DBT_CUDA(cudaMemcpy(g->d_rowoff, ro.data(), rows * sizeof(int32_t), cudaMemcpyHostToDevice));
  g->tab_bank = b->serial;
  g->tab_K = K;
  return DBT_OK;
}

int validate_params(const dbt_params* p) {
  if (!p) return set_error(DBT_ERR_CONFIG, "null params");
  if (!(1 <= p->t_occ && p->t_occ <= p->h_max && p->h_max <= 255))
    return set_error(DBT_ERR_CONFIG, "need 1 <= T <= H_max <= 255 (integrator.py:64-67)");
  if (p->downsample < 1) return set_error(DBT_ERR_CONFIG, "downsample factor must be >= 1");
  return DBT_OK;
}

// Core launch sequence. Points are already on the device (d_pts). counts /
// poses are host arrays. map_sensor (device) selects the map-frame mode.
// Graph mode of a single-scan launch (integrate_host_graph): the host-side
// bookkeeping and the conditional pre-steps (fold on a parameter change,
// epoch wrap, certificate reset) always run here, issued directly; the core
// sequence — counter memset, prep, shadow fork/join, PDL sweep — is captured
// once into a CUDA graph (capture) and afterwards only the prep / shadow
// kernel arguments of the instantiated graph change per call (replay).
struct GraphCtl {
  bool capture = false;  // issue the core under stream capture
  bool replay = false;   // do not issue the core: fill the arguments below
  PrepArgs pa;
  ShadowArgs sa;
  unsigned prep_blocks = 0, shadow_blocks = 0;
  bool shadow_bin = false;  // shadow_bin_kernel (else shadow_kernel)
  bool has_shadow = false;
};

struct DeskewArgs {
  dbt_deskew dk;
  const double* d_ts;    // device times by raw index, or null (linspace)
  const double* sincos;  // device copy of the C library's sin/cos table
};

int launch_integrate(dbt_grid* g, const dbt_bank* b, const void* d_pts, int dtype,
                     const int64_t* counts, int S, const double* poses, const dbt_params* p,
                     const double* d_map_sensor, int8_t* d_outcome, cudaStream_t st,
                     const void* const* scan_ptrs, GraphCtl* gc = nullptr, const DeskewArgs* dka = nullptr) {
  if (dka && (S != 1 || d_map_sensor)) return set_error(DBT_ERR_CONFIG, "device deskew needs one scan per launch");
  if (S < 1 || S > kMaxScansPerLaunch) return set_error(DBT_ERR_CONFIG, "scan count per launch out of range");
  if (b->device != g->device) return set_error(DBT_ERR_CONFIG, "bank and grid live on different devices");
  if (dtype != DBT_F32 && dtype != DBT_F64) return set_error(DBT_ERR_CONFIG, "points dtype must be f32 or f64");
  if (b->K > g->nx || b->K > g->ny || b->K > g->nz) {
    // every return is discarded by the boundary rule; nothing to launch
  }
  const int ds = d_map_sensor ? 1 : p->downsample;
  if (g->nx * g->ny * g->nz >= (1ll << 40))
    return set_error(DBT_ERR_CONFIG, "grid has 2^40 voxels or more (hash key width)");
  if (g->last_st != st) {
    // the per-grid scratch (counters, work list, hash, rays) may still be in
    // use by a launch on another stream: order behind it. A device-wide sync
    // (rare: only when the caller switches streams) rather than an event on
    // the old stream, which the caller may have destroyed meanwhile.
    DBT_CUDA(cudaDeviceSynchronize());
    g->last_st = st;
  }
  g->last_points_in.assign(S, 0);
  int64_t n = 0;
  for (int s = 0; s < S; ++s) {
    if (counts[s] < 0) return set_error(DBT_ERR_CONFIG, "negative point count");
    g->last_points_in[s] = (counts[s] + ds - 1) / ds;
    n += g->last_points_in[s];
  }
  g->last_scans = S;
  g->last_first_return = p->first_return ? 1 : 0;
  int rc = ensure_points(g, std::max<int64_t>(n, 1));
  if (!rc) rc = ensure_hash(g, std::max<int64_t>(n, 1));
  if (!rc) rc = ensure_rows(g, b);
  if (rc) return rc;
  const bool inline_meta = (S == 1);
  if (!inline_meta) {
    // one H2D copy of [scan_off (S+1) | src_off (S+1) | poses (12 S) |
    // scan pointers (S)] from pinned staging; wait until the previous launch
    // consumed it
    DBT_CUDA(cudaEventSynchronize(g->ev_meta));
    int64_t* h_scan = g->h_meta;
    int64_t* h_src = h_scan + (S + 1);
    double* h_pose = reinterpret_cast<double*>(h_src + (S + 1));
    h_scan[0] = 0;
    h_src[0] = 0;
    for (int s = 0; s < S; ++s) {
      h_scan[s + 1] = h_scan[s] + g->last_points_in[s];
      h_src[s + 1] = h_src[s] + counts[s];
      if (!d_map_sensor) {
        const double* P = poses + 16 * s;
        double* D = h_pose + 12 * s;
        for (int r = 0; r < 3; ++r)
          for (int c = 0; c < 3; ++c) D[3 * r + c] = P[4 * r + c];
        D[9] = P[3];
        D[10] = P[7];
        D[11] = P[11];
      }
    }
    if (scan_ptrs) {
      uint64_t* h_ptr = reinterpret_cast<uint64_t*>(h_pose + 12 * S);
      for (int s = 0; s < S; ++s) h_ptr[s] = (uint64_t)(uintptr_t)scan_ptrs[s];
    }
    const size_t bytes = (size_t)(2 * (S + 1) + (d_map_sensor ? 0 : 12 * S) + (scan_ptrs ? S : 0)) * 8;
    DBT_CUDA(cudaMemcpyAsync(g->d_scan_off, h_scan, bytes, cudaMemcpyHostToDevice, st));
    DBT_CUDA(cudaEventRecord(g->ev_meta, st));
  }
  if (n == 0) {
    DBT_CUDA(cudaMemsetAsync(g->d_lcnt, 0, sizeof(LaunchCounters) + S * sizeof(ScanCounters), st));
    return DBT_OK;
  }
  // pending shadow visits were counted under other (h_max, T): fold them first
  if (g->pend && (g->pend_h_max != p->h_max || g->pend_t_occ != p->t_occ)) {
    rc = fold_pending(g, st);
    if (rc) return rc;
  }
  if (b->max_shadow > 0) {
    g->pend = true;
    g->pend_h_max = p->h_max;
    g->pend_t_occ = p->t_occ;
  }
  g->lazy_m = true;  // the sweep lowers the length cache; masks folded before reads
  const int64_t hcap = [&] {
    int64_t w = 1024;
    while (w < 2 * n) w <<= 1;
    return w;
  }();
  // epoch-tagged hash keys: slots of older launches count as empty, so the
  // table is cleared only when the 12-bit epoch wraps
  if (g->hash_epoch >= kMaxEpoch) {
    DBT_CUDA(cudaMemsetAsync(g->d_hkey, 0, g->cap_hash * sizeof(unsigned long long), st));
    g->hash_epoch = 0;
  }
  ++g->hash_epoch;
  if (p->first_return) DBT_CUDA(cudaMemsetAsync(g->d_hmin, 0xFF, hcap * sizeof(uint32_t), st));
  if (g->cert_dk != b->dk_hash) {
    // certificates of another distance kernel say nothing about this one
    if (g->cert_dk != 0)
      DBT_CUDA(cudaMemsetAsync(g->stamped, 0, (size_t)((g->n_cert + 63) / 32) * 4, st));
    g->cert_dk = b->dk_hash;
  }
  // the core sequence starts here (graph mode: captured once, then replayed)
  if (gc && gc->capture) DBT_CUDA(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
  const bool issue = !(gc && gc->replay);
  // launch + per-scan counters: one contiguous block, one memset (zeroing
  // them behind the previous launch's read-back instead measured 2 us per
  // step slower device-resident)
  if (issue) DBT_CUDA(cudaMemsetAsync(g->d_lcnt, 0, sizeof(LaunchCounters) + S * sizeof(ScanCounters), st));
  // claim mode: centre dedup and cross-launch skip through the certificates
  // (the stamp of a centre is the same for every return there, so this holds
  // in first-return mode too; the hash then only picks the shadow return)
  const bool claim = !(p->flags & (DBT_FLAG_NO_SKIP | DBT_FLAG_NO_DEDUP));
  // the shadow update runs as its own kernel on the aux stream, concurrent
  // with the sweep (one is atomic-latency bound, the other L1 bound); fusing
  // it into preprocessing is kept as a measurement option
  const bool fuse_shadow =
      !p->first_return && b->max_shadow > 0 && b->max_shadow <= 8 && (p->flags & DBT_FLAG_FUSE_SHADOW);
  int shadow_l2 = 0;
  while ((1 << shadow_l2) < b->max_shadow) ++shadow_l2;
  // bins in the shadow kernel (off the critical path) for a single-scan
  // sized launch (tiles of >= 64 returns, |S| <= 32); big batched launches
  // keep them in prep, where the latency-bound shadow tile loop would become
  // the critical path (same-box A/B, config 5: 8 scans per launch +7 %, 32
  // scans +16 % with the bins in prep)
#ifndef DBT_SHADOW_BIN_MAX_L2
#define DBT_SHADOW_BIN_MAX_L2 5
#endif
  const bool shadow_bins = b->max_shadow > 0 && !fuse_shadow && shadow_l2 <= DBT_SHADOW_BIN_MAX_L2 && n <= (1 << 19);

  PrepArgs pa;
  pa.pts = d_pts;
  pa.sensor = d_map_sensor;
  pa.dtype = dtype;
  pa.S = S;
  pa.ds = ds;
  pa.map_mode = d_map_sensor != nullptr;
  pa.n = n;
  pa.scan_off = g->d_scan_off;
  pa.src_off = g->d_scan_off + (S + 1);
  pa.poses = reinterpret_cast<const double*>(g->d_scan_off + 2 * (S + 1));
  pa.scan_ptr = scan_ptrs ? reinterpret_cast<const uint64_t*>(g->d_scan_off + 2 * (S + 1) + 12 * S) : nullptr;
  pa.inline_meta = inline_meta ? 1 : 0;
  if (inline_meta && !d_map_sensor) {
    for (int r = 0; r < 3; ++r)
      for (int c = 0; c < 3; ++c) pa.pose0[3 * r + c] = poses[4 * r + c];
    pa.pose0[9] = poses[3];
    pa.pose0[10] = poses[7];
    pa.pose0[11] = poses[11];
  }
  pa.epoch = (uint64_t)g->hash_epoch << kEpochShift;
  pa.fuse_shadow = fuse_shadow ? 1 : 0;
  pa.cells = g->cells;
  pa.sxyz = b->d_shadow_xyz;
  pa.sstart = b->d_shadow_start;
  pa.x0 = g->x0;
  pa.x1 = g->x1;
  pa.xm = g->xm;
  pa.nzp = g->nzp;
  pa.h_max = p->h_max;
  pa.t_occ = p->t_occ;
  pa.claim = claim ? 1 : 0;
  pa.stamped = g->stamped;
  pa.nx = g->nx;
  pa.ny = g->ny;
  pa.nz = g->nz;
  pa.vs = g->vs;
  pa.ox = g->org[0];
  pa.oy = g->org[1];
  pa.oz = g->org[2];
  pa.R = b->R;
  pa.b_az = b->b_az;
  pa.b_el = b->b_el;
  pa.skip_norm = (p->flags & DBT_FLAG_SKIP_NORM_CHECK) ? 1 : 0;
  pa.first_return = p->first_return ? 1 : 0;
  pa.key_scan_bits = (p->first_return && S > 1) ? 1 : 0;
  pa.no_dedup = ((p->flags & DBT_FLAG_NO_DEDUP) && !p->first_return) ? 1 : 0;
  pa.center = g->d_center;
  pa.bin = g->d_bin;
  pa.slot = g->d_slot;
  pa.hkey = g->d_hkey;
  pa.hmin = g->d_hmin;
  pa.hmask = (uint64_t)(hcap - 1);
  pa.uniq = g->d_uniq;
  pa.lc = g->d_lcnt;
  pa.sc = g->d_scnt;
  pa.outcome = d_outcome;
  pa.seeds = device_seeds(g->device, &rc);
  pa.bins = shadow_bins ? 0 : 1;
  pa.ray = g->d_ray;
  pa.dirty = g->d_dirty;
  pa.dby = g->dby;
  pa.dbz = g->dbz;
  pa.deskew = dka ? 1 : 0;
  if (dka) pa.dk = dka->dk;
  pa.dk_ts = dka ? dka->d_ts : nullptr;
  pa.sincos = dka ? dka->sincos : nullptr;
  if (g->d_dirty) g->dirty_reach = std::max(g->dirty_reach, b->R);
  if (rc) return rc;
  int tok;
  const unsigned prep_blocks = (unsigned)((n + kPrepThreads - 1) / kPrepThreads);
  if (gc) {
    gc->pa = pa;
    gc->prep_blocks = prep_blocks;
    gc->has_shadow = false;
  }
  if (issue) {
    prof_begin(g, "prep_kernel", st, &tok);
    if (pa.deskew)
      prep_kernel<true><<<prep_blocks, kPrepThreads, 0, st>>>(pa);
    else
      prep_kernel<false><<<prep_blocks, kPrepThreads, 0, st>>>(pa);
    prof_end(g, st, tok);
    DBT_CHECK_LAUNCH("prep_kernel");
  }

  bool joined = false;
#ifdef DBT_DIAG_NO_SHADOW
  if (false) {
#else
  if (b->max_shadow > 0 && !fuse_shadow) {
#endif
    ShadowArgs sa;
    sa.cells = g->cells;
    sa.center = g->d_center;
    sa.bin = g->d_bin;
    sa.slot = g->d_slot;
    sa.hmin = g->d_hmin;
    sa.sxyz = b->d_shadow_xyz;
    sa.sstart = b->d_shadow_start;
    sa.n = n;
    const int l2 = shadow_l2;
    sa.log2s = l2;
    sa.x0 = g->x0;
    sa.x1 = g->x1;
    sa.xm = g->xm;
    sa.ny = g->ny;
    sa.nzp = g->nzp;
    sa.h_max = p->h_max;
    sa.t_occ = p->t_occ;
    sa.first_return = p->first_return ? 1 : 0;
    sa.S = S;
    sa.scan_off = g->d_scan_off;  // only read when S > 1 (first-return)
    sa.sc = g->d_scnt;
    sa.lc = g->d_lcnt;
    int64_t total = n << l2;
    unsigned blocks = (unsigned)std::min<int64_t>((total + 255) / 256, 148 * 64);
    if (shadow_bins) {
      const int per = std::max(64, 256 >> l2);
      const int64_t tiles = (n + per - 1) / per;
      sa.ray = g->d_ray;
      sa.b_az = b->b_az;
      sa.b_el = b->b_el;
      sa.seeds = pa.seeds;
      blocks = (unsigned)std::min<int64_t>(tiles, 148 * 64);
    }
    if (gc) {
      gc->sa = sa;
      gc->shadow_blocks = blocks;
      gc->shadow_bin = shadow_bins;
      gc->has_shadow = true;
    }
    if (issue) {
      // fork: aux waits for prep, runs the shadow kernel; joined before the
      // counters are read back
      DBT_CUDA(cudaEventRecord(g->ev_fork, st));
      DBT_CUDA(cudaStreamWaitEvent(g->aux, g->ev_fork, 0));
      prof_begin(g, "shadow_kernel", g->aux, &tok);
      if (shadow_bins)
        shadow_bin_kernel<<<blocks, 256, 0, g->aux>>>(sa);
      else
        shadow_kernel<<<blocks, 256, 0, g->aux>>>(sa);
      prof_end(g, g->aux, tok);
      DBT_CHECK_LAUNCH("shadow_kernel");
      DBT_CUDA(cudaEventRecord(g->ev_join, g->aux));
      joined = true;
    }
  }

  if (p->flags & DBT_FLAG_EXACT_WRITTEN) {
    // the reference's serial count needs the masks before this launch's stamps
    // (saved here for the touched cells; counted after the sweep)
    if (S != 1 || d_map_sensor) return set_error(DBT_ERR_CONFIG, "exact voxels_written needs one scan per launch");
    rc = launch_exact_pre(g, b, st);
    if (rc) return rc;
  }

  if (b->iso && !(p->flags & DBT_FLAG_GENERIC_SWEEP)) {
    // row tasks carry the row start / 8 in 32 bits (Put64)
    if (g->n_cells >> 35) return set_error(DBT_ERR_CONFIG, "grid part above 2^35 cells: unsupported by the culling sweep");
    const size_t smem = (size_t)kCullWarps * b->K * b->K * sizeof(uint64_t);
    if (g->sweep_ch != -b->K) {
      DBT_CUDA(cudaFuncSetAttribute(DBT_ISO_SWEEP, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      int per_sm = 0, sms = 0;
      DBT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, DBT_ISO_SWEEP, kCullWarps * 32, smem));
      DBT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device));
      g->sweep_blocks = std::max(per_sm, 1) * sms;
      g->sweep_ch = -b->K;
    }
    CullArgs wa;
    wa.cells = g->cells;
    wa.dist = g->dist;
    wa.uniq = g->d_uniq;
    wa.lc = g->d_lcnt;
    wa.dtab = b->d_dtab;
    wa.rowd = b->d_rowd;
    wa.stamped = g->stamped;
    wa.K = b->K;
    wa.R = b->R;
    wa.nd = b->n_distinct;
    wa.CH = b->chunks_per_row;
    wa.x0 = g->x0;
    wa.x1 = g->x1;
    wa.xm = g->xm;
    wa.nx = g->nx;
    wa.ny = g->ny;
    wa.nzp = g->nzp;
    if (!issue) {
      g->last_st = st;
      return DBT_OK;
    }
    // persistent blocks fetching kCullWarps centres at a time (a graph keeps
    // the full persistent grid: its shape cannot follow n)
    unsigned blocks = gc ? (unsigned)g->sweep_blocks
                         : (unsigned)std::min<int64_t>(g->sweep_blocks,
                                                       std::max<int64_t>(1, (n + 2 * kCullWarps - 1) / (2 * kCullWarps)));
    prof_begin(g, "sweep_kernel", st, &tok);
    if (p->flags & DBT_FLAG_EXACT_WRITTEN) {
      // exact_pre sits between prep and the sweep: plain stream order
      DBT_ISO_SWEEP<<<blocks, kCullWarps * 32, smem, st>>>(wa);
    } else {
      // programmatic dependent launch: the sweep's launch latency overlaps
      // the tail of preprocessing (the kernel waits for prep's completion)
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(blocks);
      cfg.blockDim = dim3(kCullWarps * 32);
      cfg.dynamicSmemBytes = smem;
      cfg.stream = st;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      attr[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      DBT_CUDA(cudaLaunchKernelEx(&cfg, DBT_ISO_SWEEP, wa));
    }
    prof_end(g, st, tok);
    DBT_CHECK_LAUNCH("sweep_cull_kernel");
    if (p->flags & DBT_FLAG_EXACT_WRITTEN) {
      rc = launch_exact_post(g, b, st);
      if (rc) return rc;
    }
    if (joined) DBT_CUDA(cudaStreamWaitEvent(st, g->ev_join, 0));
    g->last_st = st;
    return DBT_OK;
  }
  const int CH = b->chunks_per_row;
  SweepFn fn = sweep_fn(CH);
  if (!fn) return set_error(DBT_ERR_CONFIG, "unsupported kernel size for the sweep");
  const size_t smem = sweep_smem_bytes(b->K, CH, b->n_distinct);
  const int shape_key = CH;
  if (g->sweep_ch != shape_key) {
    DBT_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    // keep shared memory to what 8 resident blocks need; the rest stays L1
    int carve = (int)std::min<size_t>(100, (smem * 8 * 100 + 233471) / 233472 + 1);
    DBT_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, carve));
    int per_sm = 0, sms = 0;
    DBT_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 256, smem));
    DBT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device));
    g->sweep_blocks = std::max(per_sm, 1) * sms;
    g->sweep_ch = shape_key;
  }
  SweepArgs wa;
  wa.cells = g->cells;
  wa.dist = g->dist;
  wa.uniq = g->d_uniq;
  wa.lc_in = g->d_lcnt;
  wa.changed_out = &g->d_lcnt->changed;
  wa.dtab = b->d_dtab;
  wa.rowd = b->d_rowd;
  wa.rowoff = g->d_rowoff;
  wa.nd = b->n_distinct;
  wa.K = b->K;
  wa.R = b->R;
  wa.x0 = g->x0;
  wa.x1 = g->x1;
  wa.xm = g->xm;
  wa.ny = g->ny;
  wa.nzp = g->nzp;
  unsigned blocks = (unsigned)std::min<int64_t>(g->sweep_blocks, std::max<int64_t>(1, (n + 7) / 8));
  prof_begin(g, "sweep_kernel", st, &tok);
  fn<<<blocks, 256, smem, st>>>(wa);
  prof_end(g, st, tok);
  DBT_CHECK_LAUNCH("sweep_kernel");
  if (p->flags & DBT_FLAG_EXACT_WRITTEN) {
    rc = launch_exact_post(g, b, st);
    if (rc) return rc;
  }
  if (joined) DBT_CUDA(cudaStreamWaitEvent(st, g->ev_join, 0));
  g->last_st = st;
  return DBT_OK;
}

int fetch_counters(dbt_grid* g, cudaStream_t st) {
  DBT_CUDA(cudaMemcpyAsync(g->h_lcnt, g->d_lcnt, sizeof(LaunchCounters) + g->last_scans * sizeof(ScanCounters),
                           cudaMemcpyDeviceToHost, st));
  return DBT_OK;
}

void fill_stats(dbt_grid* g, const dbt_params* p, dbt_stats* out, int S) {
  for (int s = 0; s < S; ++s) {
    dbt_stats& o = out[s];
    std::memset(&o, 0, sizeof(o));
    o.points_in = g->last_points_in[s];
    int64_t nok = (int64_t)g->h_scnt[s].n_ok;
    o.points_discarded = o.points_in - nok;
    o.points_applied = p->first_return ? (int64_t)g->h_scnt[s].n_applied : nok;
    o.bin_fallbacks = (int64_t)g->h_scnt[s].n_fallback;
    if (s == 0) {
      o.voxels_written = (int64_t)((p->flags & DBT_FLAG_EXACT_WRITTEN) ? g->h_lcnt->exact_written
                                                                        : g->h_lcnt->changed);
      o.unique_centers = (int64_t)g->h_lcnt->n_unique;
      o.centers_skipped = (int64_t)g->h_lcnt->skipped;
      o.rows_swept = (int64_t)g->h_lcnt->rows;
    }
  }
}

int check(dbt_grid* g, const dbt_bank* b) {
  if (!g) return set_error(DBT_ERR_CONFIG, "null grid handle");
  if (!b) return set_error(DBT_ERR_CONFIG, "null bank handle");
  return grid_set_device(g);
}

int stage_raw(dbt_grid* g, int64_t bytes) { return grow(&g->d_raw, &g->cap_raw_bytes, bytes, 1); }

// Synchronous entry points poll the completion event instead of sleeping in
// cudaStreamSynchronize: the call is about to return anyway, and polling
// answers within ~1 us of completion (a blocking wake-up can take ~10 us).
// Completion of a synchronous call: poll the event (answers within ~1 us;
// a blocking wake-up costs ~10 us, a quarter of a config-2 step) for up to
// 1 ms, then poll every 50 us with the thread asleep in between, so long
// batched calls do not keep a host core spinning. (A blocking-sync event
// instead made every config-2 call ~14 us slower, even when polled.)
cudaError_t wait_event(cudaEvent_t ev) {
  const auto t0 = std::chrono::steady_clock::now();
  cudaError_t e;
  while ((e = cudaEventQuery(ev)) == cudaErrorNotReady) {
    if (std::chrono::steady_clock::now() - t0 > std::chrono::microseconds(1000))
      std::this_thread::sleep_for(std::chrono::microseconds(50));
  }
  return e;
}

// Synchronous calls: device_ms (two timing events + cudaEventElapsedTime,
// ~4 us of host time) only when profiling or $DBT_DEVICE_MS asks for it;
// otherwise one timing-free completion event.
void call_begin(dbt_grid* g, cudaStream_t st, bool timed) {
  if (timed) cudaEventRecord(g->ev_a, st);
}

int call_end(dbt_grid* g, cudaStream_t st, bool timed, double* device_ms) {
  cudaEvent_t e = timed ? g->ev_b : g->ev_done;
  DBT_CUDA(cudaEventRecord(e, st));
  DBT_CUDA(wait_event(e));
  *device_ms = 0.0;
  if (timed) {
    float dms = 0.f;
    cudaEventElapsedTime(&dms, g->ev_a, g->ev_b);
    *device_ms = dms;
  }
  return DBT_OK;
}

double now_ms() {
  return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// The synchronous single-scan sequence as a CUDA graph: one cudaGraphLaunch
// (plus two kernel-argument updates) instead of ~10 stream calls, and no
// launch gaps between the kernels. Eligible: default-path launches (claim
// mode, isotropic kernel, no first-return / exact / measurement flags), not
// under profiling. The graph is re-captured when the launch shape changes
// (bank, dtype, flags, parameters, scratch buffers, stream, shadow mode).
// Returns DBT_OK after enqueueing the graph (counters D2H included).
bool graph_eligible(const dbt_grid* g, const dbt_bank* b, const dbt_params* p) {
  static const bool off = getenv("DBT_NO_GRAPH") != nullptr;
  const uint32_t bad = DBT_FLAG_NO_DEDUP | DBT_FLAG_NO_SKIP | DBT_FLAG_FUSE_SHADOW | DBT_FLAG_GENERIC_SWEEP |
                       DBT_FLAG_EXACT_WRITTEN | DBT_FLAG_MAP_FRAME;
  return !off && !g->gdisabled && !g->profiling && b->iso && !p->first_return && !(p->flags & bad);
}

int integrate_graph(dbt_grid* g, const dbt_bank* b, const void* d_src, int dtype, int64_t n_raw, const double* pose,
                    const dbt_params* p, cudaStream_t st, int exec_slot = -1) {
  const int64_t n = (n_raw + p->downsample - 1) / p->downsample;
  if (g->sweep_ch != -b->K || n > g->cap_pts || 2 * n > g->cap_hash) {
    // first launch with this bank / growth of the scratch buffers: the one-time
    // setup (allocations, sweep shape, seed table) runs outside any capture
    int rc = launch_integrate(g, b, d_src, dtype, &n_raw, 1, pose, p, nullptr, nullptr, st, nullptr);
    return rc ? rc : fetch_counters(g, st);
  }
  uint64_t key[12] = {b->serial, (uint64_t)dtype, (uint64_t)p->flags,
                      (uint64_t)p->h_max | ((uint64_t)p->t_occ << 8) | ((uint64_t)p->downsample << 16),
                      (uint64_t)(uintptr_t)g->d_center, (uint64_t)g->cap_pts, (uint64_t)(uintptr_t)st,
                      (uint64_t)(n <= (1 << 19)), (uint64_t)g->sweep_blocks, (uint64_t)(uintptr_t)g->d_raw,
                      (uint64_t)g->cap_hash, (uint64_t)(uintptr_t)b};
  GraphCtl gc;
  const bool fresh = !g->gexec || std::memcmp(key, g->gkey, sizeof(key)) != 0;
  if (fresh) {
    if (g->gexec) cudaGraphExecDestroy(g->gexec);
    if (g->ggraph) cudaGraphDestroy(g->ggraph);
    g->gexec = nullptr;
    g->ggraph = nullptr;
    for (auto& e : g->aexec) {
      if (e) cudaGraphExecDestroy(e);  // stale shape (a running launch completes first)
      e = nullptr;
    }
    // the persistent sweep grid size is measured on first use: make sure it
    // is known before the key is stored
    gc.capture = true;
    const int64_t c0 = dbt_launch_count();
    int rc = launch_integrate(g, b, d_src, dtype, &n_raw, 1, pose, p, nullptr, nullptr, st, nullptr, &gc);
    if (!rc) rc = fetch_counters(g, st);
    cudaGraph_t graph = nullptr;
    const cudaError_t ec = cudaStreamEndCapture(st, &graph);
    add_launches(-(dbt_launch_count() - c0));  // nothing ran yet
    if (rc) {
      if (graph) cudaGraphDestroy(graph);
      return rc;
    }
    cudaGraphExec_t exec = nullptr;
    cudaError_t ei = ec == cudaSuccess ? cudaGraphInstantiate(&exec, graph, 0) : ec;
    if (ei != cudaSuccess) {
      // capture of this sequence is not supported here: direct launches
      cudaGetLastError();
      if (graph) cudaGraphDestroy(graph);
      g->gdisabled = true;
      rc = launch_integrate(g, b, d_src, dtype, &n_raw, 1, pose, p, nullptr, nullptr, st, nullptr);
      if (!rc) rc = fetch_counters(g, st);
      return rc;
    }
    size_t nn = 0;
    DBT_CUDA(cudaGraphGetNodes(graph, nullptr, &nn));
    std::vector<cudaGraphNode_t> nodes(nn);
    DBT_CUDA(cudaGraphGetNodes(graph, nodes.data(), &nn));
    g->gprep = g->gshadow = nullptr;
    g->gkernels = 0;
    for (cudaGraphNode_t nd : nodes) {
      cudaGraphNodeType t;
      DBT_CUDA(cudaGraphNodeGetType(nd, &t));
      if (t != cudaGraphNodeTypeKernel) continue;
      ++g->gkernels;
      cudaKernelNodeParams kp;
      DBT_CUDA(cudaGraphKernelNodeGetParams(nd, &kp));
      if (kp.func == (void*)prep_kernel<false>) g->gprep = nd;
      if (kp.func == (void*)shadow_kernel || kp.func == (void*)shadow_bin_kernel) g->gshadow = nd;
    }
    g->ggraph = graph;
    g->gexec = exec;
    std::memcpy(g->gkey, key, sizeof(key));
    if (!g->gprep) return set_error(DBT_ERR_GENERIC, "graph capture lost the prep kernel");
  } else {
    gc.replay = true;
    int rc = launch_integrate(g, b, d_src, dtype, &n_raw, 1, pose, p, nullptr, nullptr, st, nullptr, &gc);
    if (rc) return rc;
    cudaGraphExec_t ex = g->gexec;
    if (exec_slot >= 0) {
      if (!g->aexec[exec_slot]) DBT_CUDA(cudaGraphInstantiate(&g->aexec[exec_slot], g->ggraph, 0));
      ex = g->aexec[exec_slot];
    }
    cudaKernelNodeParams kp = {};
    void* pargs[] = {&gc.pa};
    kp.func = (void*)prep_kernel<false>;
    kp.gridDim = dim3(gc.prep_blocks);
    kp.blockDim = dim3(kPrepThreads);
    kp.kernelParams = pargs;
    DBT_CUDA(cudaGraphExecKernelNodeSetParams(ex, g->gprep, &kp));
    if (gc.has_shadow != (g->gshadow != nullptr)) return set_error(DBT_ERR_GENERIC, "graph shape changed");
    if (gc.has_shadow) {
      void* sargs[] = {&gc.sa};
      kp.func = gc.shadow_bin ? (void*)shadow_bin_kernel : (void*)shadow_kernel;
      kp.gridDim = dim3(gc.shadow_blocks);
      kp.blockDim = dim3(256);
      kp.kernelParams = sargs;
      DBT_CUDA(cudaGraphExecKernelNodeSetParams(ex, g->gshadow, &kp));
    }
    DBT_CUDA(cudaGraphLaunch(ex, st));
    add_launches(g->gkernels);
    return DBT_OK;
  }
  DBT_CUDA(cudaGraphLaunch(g->gexec, st));
  add_launches(g->gkernels);
  return DBT_OK;
}

int integrate_host(dbt_grid* g, const dbt_bank* b, const void* points, int dtype, const int64_t* counts,
                   int S, const double* poses, const dbt_params* p, dbt_stats* out, const dbt_deskew* dk = nullptr,
                   const double* timestamps = nullptr) {
  double t0 = now_ms();
  int rc = check(g, b);
  if (!rc) rc = validate_params(p);
  if (!rc && dk) rc = check_deskew(dk);
  if (rc) return rc;
  int64_t total = 0;
  for (int s = 0; s < S; ++s) total += counts[s];
  if (total == 0) {
    // empty scan: zeroed stats, no device work (integrator.py:219-221)
    for (int s = 0; s < S; ++s) std::memset(&out[s], 0, sizeof(dbt_stats));
    out[0].elapsed_ms = now_ms() - t0;
    return DBT_OK;
  }
  const size_t esz = dtype == DBT_F32 ? 12 : 24;
  cudaStream_t st = g->stream;
  // Pinned (page-locked, device-mapped) host scans are read by the prep
  // kernel straight over the host link (zero-copy): the transfer overlaps
  // preprocessing instead of preceding it. Pageable memory is staged with
  // one H2D copy.
  const void* d_src = nullptr;
  if (!(p->flags & DBT_FLAG_STAGE_COPY)) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, points) == cudaSuccess && at.type == cudaMemoryTypeHost &&
        at.devicePointer != nullptr)
      d_src = at.devicePointer;
    else
      cudaGetLastError();  // pageable pointers report an error on some drivers
  }
  const bool timed = g->time_calls || g->profiling;
  // pageable scans: multi-threaded host copy into pinned staging, read by
  // prep over the host link like a pinned scan (the driver's pageable copy
  // is single-threaded)
  if (!d_src && !(p->flags & DBT_FLAG_STAGE_COPY)) {
    const int64_t bytes = total * (int64_t)esz;
    if (!stage_pageable(g, &points, &bytes, 1, &d_src)) d_src = nullptr;
  }
  call_begin(g, st, timed);
  if (!d_src) {
    rc = stage_raw(g, total * (int64_t)esz);
    if (rc) return rc;
    DBT_CUDA(cudaMemcpyAsync(g->d_raw, points, total * esz, cudaMemcpyHostToDevice, st));
    d_src = g->d_raw;
  }
  if (dk) {
    // device deskew: the C library's sin/cos table, the per-point times
    DeskewArgs dka;
    dka.dk = *dk;
    dka.d_ts = nullptr;
    dka.sincos = device_sincostab(g->device, &rc);
    if (rc) return rc;
    if (timestamps) {
      rc = grow((void**)&g->d_ts, &g->cap_ts, counts[0], sizeof(double));
      if (rc) return rc;
      DBT_CUDA(cudaMemcpyAsync(g->d_ts, timestamps, counts[0] * sizeof(double), cudaMemcpyHostToDevice, st));
      dka.d_ts = g->d_ts;
    }
    rc = launch_integrate(g, b, d_src, dtype, counts, 1, poses, p, nullptr, nullptr, st, nullptr, nullptr, &dka);
    if (!rc) rc = fetch_counters(g, st);
  } else if (S == 1 && graph_eligible(g, b, p)) {
    rc = integrate_graph(g, b, d_src, dtype, counts[0], poses, p, st);
  } else {
    rc = launch_integrate(g, b, d_src, dtype, counts, S, poses, p, nullptr, nullptr, st, nullptr);
    if (!rc) rc = fetch_counters(g, st);
  }
  if (rc) return rc;
  double dms = 0.0;
  rc = call_end(g, st, timed, &dms);
  if (rc) return rc;
  fill_stats(g, p, out, S);
  out[0].device_ms = dms;
  out[0].elapsed_ms = now_ms() - t0;
  return DBT_OK;
}

// S scans given as S host pointers (no concatenation on the host): pinned
// scans are read zero-copy by the prep kernel through a device table of scan
// pointers, pageable ones are staged each with one H2D copy.
int integrate_scans_host(dbt_grid* g, const dbt_bank* b, const void* const* points, int dtype,
                         const int64_t* counts, int S, const double* poses, const dbt_params* p, dbt_stats* out) {
  double t0 = now_ms();
  int rc = check(g, b);
  if (!rc) rc = validate_params(p);
  if (rc) return rc;
  if (S < 1 || S > kMaxScansPerLaunch) return set_error(DBT_ERR_CONFIG, "scan count per launch out of range");
  int64_t total = 0;
  for (int s = 0; s < S; ++s) {
    if (counts[s] < 0) return set_error(DBT_ERR_CONFIG, "negative point count");
    total += counts[s];
  }
  if (total == 0) {
    for (int s = 0; s < S; ++s) std::memset(&out[s], 0, sizeof(dbt_stats));
    out[0].elapsed_ms = now_ms() - t0;
    return DBT_OK;
  }
  const size_t esz = dtype == DBT_F32 ? 12 : 24;
  cudaStream_t st = g->stream;
  std::vector<const void*> dptr(S, nullptr);
  int64_t staged = 0;
  for (int s = 0; s < S; ++s) {
    if (counts[s] == 0 || (p->flags & DBT_FLAG_STAGE_COPY)) continue;
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, points[s]) == cudaSuccess && at.type == cudaMemoryTypeHost &&
        at.devicePointer != nullptr)
      dptr[s] = at.devicePointer;
    else
      cudaGetLastError();
  }
  if (!(p->flags & DBT_FLAG_STAGE_COPY)) {
    // pageable scans: multi-threaded host copy into pinned staging
    std::vector<const void*> src;
    std::vector<int64_t> bytes;
    std::vector<int> idx;
    for (int s = 0; s < S; ++s)
      if (!dptr[s] && counts[s]) {
        src.push_back(points[s]);
        bytes.push_back(counts[s] * (int64_t)esz);
        idx.push_back(s);
      }
    std::vector<const void*> out(src.size());
    if (!src.empty() && stage_pageable(g, src.data(), bytes.data(), (int)src.size(), out.data()))
      for (size_t i = 0; i < idx.size(); ++i) dptr[idx[i]] = out[i];
  }
  for (int s = 0; s < S; ++s)
    if (!dptr[s]) staged += counts[s];
  const bool timed = g->time_calls || g->profiling;
  call_begin(g, st, timed);
  if (staged) {
    rc = stage_raw(g, staged * (int64_t)esz);
    if (rc) return rc;
    int64_t off = 0;
    for (int s = 0; s < S; ++s) {
      if (dptr[s]) continue;
      char* d = (char*)g->d_raw + off * esz;
      if (counts[s]) DBT_CUDA(cudaMemcpyAsync(d, points[s], counts[s] * esz, cudaMemcpyHostToDevice, st));
      dptr[s] = d;
      off += counts[s];
    }
  }
  if (S == 1)
    rc = launch_integrate(g, b, dptr[0], dtype, counts, 1, poses, p, nullptr, nullptr, st, nullptr);
  else
    rc = launch_integrate(g, b, nullptr, dtype, counts, S, poses, p, nullptr, nullptr, st, dptr.data());
  if (rc) return rc;
  rc = fetch_counters(g, st);
  if (rc) return rc;
  double dms = 0.0;
  rc = call_end(g, st, timed, &dms);
  if (rc) return rc;
  fill_stats(g, p, out, S);
  out[0].device_ms = dms;
  out[0].elapsed_ms = now_ms() - t0;
  return DBT_OK;
}

}  // namespace

extern "C" {

int dbt_integrate_scans(dbt_grid* g, const dbt_bank* b, const void* const* points, int dtype,
                        const int64_t* counts, int32_t n_scans, const double* poses, const dbt_params* p,
                        dbt_stats* out) {
  return integrate_scans_host(g, b, points, dtype, counts, n_scans, poses, p, out);
}

int dbt_integrate_frame(dbt_grid* g, const dbt_bank* b, const void* points, int dtype, int64_t n,
                        const double pose[16], const dbt_params* p, dbt_stats* out) {
  return integrate_host(g, b, points, dtype, &n, 1, pose, p, out);
}

// Asynchronous single-scan call: the scan is copied into a device buffer
// of its slot on a copy stream (overlapping the previous calls' kernels),
// the launch sequence (graph) follows on the grid stream, and the counters
// land in the slot's pinned block; dbt_frame_wait collects them. Up to
// kAsyncSlots calls are in flight; a fifth call waits for the oldest slot's
// completion (its stats stay readable until the slot is reused).
int dbt_integrate_frame_async(dbt_grid* g, const dbt_bank* b, const void* points, int dtype, int64_t n,
                              const double pose[16], const dbt_params* p, int64_t* ticket) {
  const double t0 = now_ms();
  int rc = check(g, b);
  if (!rc) rc = validate_params(p);
  if (rc) return rc;
  if (!ticket) return set_error(DBT_ERR_CONFIG, "null ticket");
  if (dtype != DBT_F32 && dtype != DBT_F64) return set_error(DBT_ERR_CONFIG, "points dtype must be f32 or f64");
  if (n < 0) return set_error(DBT_ERR_CONFIG, "negative point count");
  cudaStream_t st = g->stream;
  if (g->last_st != st) {
    DBT_CUDA(cudaDeviceSynchronize());
    g->last_st = st;
  }
  if (!g->cstream) DBT_CUDA(cudaStreamCreateWithFlags(&g->cstream, cudaStreamNonBlocking));
  const int64_t tk = g->a_next++;
  AsyncSlot& sl = g->aslot[tk % kAsyncSlots];
  if (!sl.done) {
    DBT_CUDA(cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming));
    DBT_CUDA(cudaEventCreateWithFlags(&sl.copied, cudaEventDisableTiming));
    DBT_CUDA(cudaHostAlloc((void**)&sl.h, sizeof(LaunchCounters) + sizeof(ScanCounters), cudaHostAllocDefault));
  }
  if (sl.ticket >= 0) DBT_CUDA(wait_event(sl.done));  // the slot's previous call (buffer and counters free)
  const size_t esz = dtype == DBT_F32 ? 12 : 24;
  if (n * (int64_t)esz > sl.cap) {
    // with headroom (scan sizes vary by their dropouts) and geometric
    // growth: cudaFree / cudaMalloc synchronise the device
    if (sl.d_buf) DBT_CUDA(cudaFree(sl.d_buf));
    sl.d_buf = nullptr;
    sl.cap = std::max<int64_t>(n * (int64_t)esz * 5 / 4, sl.cap + sl.cap / 2);
    DBT_CUDA(cudaMalloc(&sl.d_buf, sl.cap));
  }
  sl.ticket = tk;
  sl.p = *p;
  sl.points_in = (n + p->downsample - 1) / p->downsample;
  sl.t0 = t0;
  if (n == 0) {
    std::memset(sl.h, 0, sizeof(LaunchCounters) + sizeof(ScanCounters));
    DBT_CUDA(cudaEventRecord(sl.done, st));
    *ticket = tk;
    return DBT_OK;
  }
  // a pageable scan (plain numpy) goes through the slot's pinned staging with
  // the host copy pool: cudaMemcpyAsync from pageable memory would block this
  // thread on the driver's single-threaded bounce buffer (hostcopy.cu)
  const void* h_src = points;
  if ((int64_t)(n * esz) >= (64 << 10) && !getenv("DBT_NO_HOST_STAGE")) {
    cudaPointerAttributes at;
    const bool registered = cudaPointerGetAttributes(&at, points) == cudaSuccess &&
                            (at.type == cudaMemoryTypeHost || at.type == cudaMemoryTypeManaged);
    if (!registered) {
      cudaGetLastError();  // pageable pointers report an error on some drivers
      if ((int64_t)(n * esz) > sl.cap_hstage) {
        if (sl.h_stage) cudaFreeHost(sl.h_stage);
        sl.h_stage = nullptr;
        sl.cap_hstage = 0;
        const int64_t cap = (int64_t)(n * esz) * 5 / 4;
        if (cudaHostAlloc(&sl.h_stage, (size_t)cap, cudaHostAllocDefault) == cudaSuccess)
          sl.cap_hstage = cap;
        else
          cudaGetLastError();
      }
      if (sl.h_stage) {
        // the slot's previous copy has completed (its `done` event was waited on above)
        pooled_host_copy(sl.h_stage, points, n * esz);
        h_src = sl.h_stage;
      }
    }
  }
  DBT_CUDA(cudaMemcpyAsync(sl.d_buf, h_src, n * esz, cudaMemcpyHostToDevice, g->cstream));
  DBT_CUDA(cudaEventRecord(sl.copied, g->cstream));
  DBT_CUDA(cudaStreamWaitEvent(st, sl.copied, 0));
  // the default path replays the slot's own executable graph; other launch
  // shapes (first-return, exact count, measurement flags, profiling) are
  // issued directly
  if (graph_eligible(g, b, p))
    rc = integrate_graph(g, b, sl.d_buf, dtype, n, pose, p, st, (int)(tk % kAsyncSlots));
  else
    rc = launch_integrate(g, b, sl.d_buf, dtype, &n, 1, pose, p, nullptr, nullptr, st, nullptr);
  if (rc) return rc;
  DBT_CUDA(cudaMemcpyAsync(sl.h, g->d_lcnt, sizeof(LaunchCounters) + sizeof(ScanCounters), cudaMemcpyDeviceToHost,
                           st));
  DBT_CUDA(cudaEventRecord(sl.done, st));
  *ticket = tk;
  return DBT_OK;
}

int dbt_frame_wait(dbt_grid* g, int64_t ticket, dbt_stats* out) {
  if (!g) return set_error(DBT_ERR_CONFIG, "null grid handle");
  if (!out) return set_error(DBT_ERR_CONFIG, "null stats");
  if (ticket < 0 || ticket >= g->a_next) return set_error(DBT_ERR_CONFIG, "unknown ticket");
  AsyncSlot& sl = g->aslot[ticket % kAsyncSlots];
  if (sl.ticket != ticket) return set_error(DBT_ERR_CONFIG, "ticket expired (more than 4 calls issued since)");
  DBT_CUDA(wait_event(sl.done));
  const LaunchCounters& lc = *sl.h;
  const ScanCounters& sc = *reinterpret_cast<const ScanCounters*>(sl.h + 1);
  std::memset(out, 0, sizeof(*out));
  out->points_in = sl.points_in;
  out->points_discarded = sl.points_in - (int64_t)sc.n_ok;
  out->points_applied = sl.p.first_return ? (int64_t)sc.n_applied : (int64_t)sc.n_ok;
  out->bin_fallbacks = (int64_t)sc.n_fallback;
  out->voxels_written = (int64_t)((sl.p.flags & DBT_FLAG_EXACT_WRITTEN) ? lc.exact_written : lc.changed);
  out->unique_centers = (int64_t)lc.n_unique;
  out->centers_skipped = (int64_t)lc.skipped;
  out->rows_swept = (int64_t)lc.rows;
  out->elapsed_ms = now_ms() - sl.t0;
  return DBT_OK;
}

int dbt_deskew_available(int32_t* ok) {
  if (!ok) return set_error(DBT_ERR_CONFIG, "null output");
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n < 1) {
    cudaGetLastError();
    *ok = 0;
    return DBT_OK;
  }
  int cur = 0;
  cudaGetDevice(&cur);
  int rc = DBT_OK;
  *ok = device_sincostab(cur, &rc) != nullptr ? 1 : 0;
  return DBT_OK;
}

int dbt_integrate_frame_deskew(dbt_grid* g, const dbt_bank* b, const void* points, int dtype, int64_t n,
                               const double* timestamps, const double pose[16], const dbt_deskew* d,
                               const dbt_params* p, dbt_stats* out) {
  return integrate_host(g, b, points, dtype, &n, 1, pose, p, out, d, timestamps);
}

int dbt_deskew_points(int device, const void* points, int dtype, int64_t n, const double* timestamps,
                      int32_t downsample, const dbt_deskew* d, double* out) {
  int rc = check_deskew(d);
  if (rc) return rc;
  if (dtype != DBT_F32 && dtype != DBT_F64) return set_error(DBT_ERR_CONFIG, "points dtype must be f32 or f64");
  if (downsample < 1 || n < 0) return set_error(DBT_ERR_CONFIG, "bad point count or downsample factor");
  if (n == 0) return DBT_OK;
  DBT_CUDA(cudaSetDevice(device));
  const double* tab = device_sincostab(device, &rc);
  if (rc) return rc;
  const int64_t m = (n + downsample - 1) / downsample;
  const size_t esz = dtype == DBT_F32 ? 12 : 24;
  void* dp = nullptr;
  double *dts = nullptr, *dout = nullptr;
  cudaError_t e = cudaMalloc(&dp, n * esz);
  if (e == cudaSuccess) e = cudaMalloc((void**)&dout, m * 24);
  if (e == cudaSuccess && timestamps) e = cudaMalloc((void**)&dts, n * 8);
  if (e == cudaSuccess) e = cudaMemcpy(dp, points, n * esz, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && timestamps) e = cudaMemcpy(dts, timestamps, n * 8, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    deskew_points_kernel<<<(unsigned)std::min<int64_t>((m + 255) / 256, 148 * 8), 256>>>(dp, dtype, m, downsample,
                                                                                       dts, *d, tab, dout);
    e = cudaGetLastError();
    if (e == cudaSuccess) count_launch();
  }
  if (e == cudaSuccess) e = cudaMemcpy(out, dout, m * 24, cudaMemcpyDeviceToHost);
  cudaFree(dp);
  cudaFree(dout);
  if (dts) cudaFree(dts);
  if (e != cudaSuccess) return cuda_error(e, "dbt_deskew_points");
  return DBT_OK;
}

int dbt_integrate_batch(dbt_grid* g, const dbt_bank* b, const void* points, int dtype,
                        const int64_t* counts, int32_t n_scans, const double* poses,
                        const dbt_params* p, dbt_stats* out) {
  return integrate_host(g, b, points, dtype, counts, n_scans, poses, p, out);
}

int dbt_integrate_points_map(dbt_grid* g, const dbt_bank* b, const double* p_map, const double* sensor,
                             int64_t n, const dbt_params* p, dbt_stats* out, int8_t* outcome) {
  double t0 = now_ms();
  int rc = check(g, b);
  if (!rc) rc = validate_params(p);
  if (rc) return rc;
  std::memset(out, 0, sizeof(dbt_stats));
  if (n == 0) return DBT_OK;
  dbt_params q = *p;
  q.downsample = 1;
  q.first_return = 0;
  rc = stage_raw(g, n * 24);
  if (!rc) rc = grow((void**)&g->d_sensor, &g->cap_sensor, n * 3, sizeof(double));
  if (!rc && outcome) rc = grow((void**)&g->d_outcome, &g->cap_outcome, n, 1);
  if (rc) return rc;
  cudaStream_t st = g->stream;
  const bool timed = g->time_calls || g->profiling;
  call_begin(g, st, timed);
  DBT_CUDA(cudaMemcpyAsync(g->d_raw, p_map, n * 24, cudaMemcpyHostToDevice, st));
  DBT_CUDA(cudaMemcpyAsync(g->d_sensor, sensor, n * 24, cudaMemcpyHostToDevice, st));
  rc = launch_integrate(g, b, g->d_raw, DBT_F64, &n, 1, nullptr, &q, g->d_sensor,
                        outcome ? g->d_outcome : nullptr, st, nullptr);
  if (rc) return rc;
  rc = fetch_counters(g, st);
  if (rc) return rc;
  if (outcome) DBT_CUDA(cudaMemcpyAsync(outcome, g->d_outcome, n, cudaMemcpyDeviceToHost, st));
  double dms = 0.0;
  rc = call_end(g, st, timed, &dms);
  if (rc) return rc;
  fill_stats(g, &q, out, 1);
  out->device_ms = dms;
  out->elapsed_ms = now_ms() - t0;
  return DBT_OK;
}

int dbt_integrate_device(dbt_grid* g, const dbt_bank* b, const void* d_points, int dtype,
                         const int64_t* counts, int32_t n_scans, const double* poses,
                         const dbt_params* p, void* stream) {
  int rc = check(g, b);
  if (!rc) rc = validate_params(p);
  if (rc) return rc;
  cudaStream_t st = (cudaStream_t)stream;  // NULL = legacy default stream
  // single scans on a capturable stream go through the launch-sequence graph
  if (n_scans == 1 && st != nullptr && counts[0] > 0 && graph_eligible(g, b, p))
    return integrate_graph(g, b, d_points, dtype, counts[0], poses, p, st);
  rc = launch_integrate(g, b, d_points, dtype, counts, n_scans, poses, p, nullptr, nullptr, st, nullptr);
  if (rc) return rc;
  return fetch_counters(g, st);
}

int dbt_stats_read(dbt_grid* g, dbt_stats* out, int32_t n_scans) {
  if (!g) return set_error(DBT_ERR_CONFIG, "null grid handle");
  DBT_CUDA(cudaSetDevice(g->device));
  DBT_CUDA(cudaDeviceSynchronize());
  if (n_scans != g->last_scans) return set_error(DBT_ERR_CONFIG, "scan count differs from the last launch");
  dbt_params q{};
  q.first_return = g->last_first_return;
  fill_stats(g, &q, out, n_scans);
  return DBT_OK;
}

int dbt_grid_stream(dbt_grid* g, void** stream) {
  if (!g) return set_error(DBT_ERR_CONFIG, "null grid handle");
  *stream = (void*)g->stream;
  return DBT_OK;
}

int dbt_synchronize(dbt_grid* g) {
  if (!g) return set_error(DBT_ERR_CONFIG, "null grid handle");
  DBT_CUDA(cudaSetDevice(g->device));
  DBT_CUDA(cudaStreamSynchronize(g->stream));
  return DBT_OK;
}

int dbt_bin_index_array(const double* dirs, int64_t n, int32_t b_az, int32_t b_el, int64_t* b_a,
                        int64_t* b_e, int device) {
  if (n == 0) return DBT_OK;
  DBT_CUDA(cudaSetDevice(device));
  double* d_dirs = nullptr;
  int64_t* d_out = nullptr;
  DBT_CUDA(cudaMalloc(&d_dirs, n * 24));
  cudaError_t e = cudaMalloc(&d_out, n * 16);
  if (e != cudaSuccess) {
    cudaFree(d_dirs);
    return cuda_error(e, "cudaMalloc(bins)");
  }
  e = cudaMemcpy(d_dirs, dirs, n * 24, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) {
    unsigned blocks = (unsigned)std::min<int64_t>((n + 255) / 256, 148 * 32);
    int rc2 = DBT_OK;
    const uint16_t* seeds = device_seeds(device, &rc2);
    if (rc2) {
      cudaFree(d_dirs);
      cudaFree(d_out);
      return rc2;
    }
    bin_kernel<<<blocks, 256>>>(d_dirs, n, b_az, b_el, seeds, d_out, d_out + n);
    e = cudaGetLastError();
    dbt::count_launch();
  }
  if (e == cudaSuccess) e = cudaMemcpy(b_a, d_out, n * 8, cudaMemcpyDeviceToHost);
  if (e == cudaSuccess) e = cudaMemcpy(b_e, d_out + n, n * 8, cudaMemcpyDeviceToHost);
  cudaFree(d_dirs);
  cudaFree(d_out);
  if (e != cudaSuccess) return cuda_error(e, "dbt_bin_index_array");
  return DBT_OK;
}

}  // extern "C"
