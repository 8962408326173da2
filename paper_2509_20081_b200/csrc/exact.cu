// exact.cu — the reference's serial FrameStats.voxels_written on the device
// (DBT_FLAG_EXACT_WRITTEN; reference integrator.py:139-160, 268-285).
//
// The reference stamps the applied returns one by one in ascending centre
// order (stable argsort of the C-order centre index, integrator.py:268-274)
// and counts, per stamp, the K^3 cells whose mask the AND changed. The final
// grid does not depend on that order, but the count does. It is recovered
// exactly from three facts:
//  * a return whose centre was already stamped (same scan or a certified
//    earlier one, engine.cuh "stamp certificates") changes nothing and leaves
//    the state unchanged, so only this launch's new centres (the sweep's work
//    list) matter, each once;
//  * cell v sees the new centres c with v in box(c), i.e. c in box(v), in
//    lexicographic (cx, cy, cz) order — rows (cx, cy) ascending, cz ascending;
//  * a stamp changes v iff (m & k) != m for the running mask m, starting from
//    v's mask before the launch.
// Before the sweep the new centres are marked (centre, centre-row and
// touched-cell bitmaps) and the touched cells' masks saved; after it, one
// lane per touched cell that changed replays the centres of its box in that
// order until its mask reaches the final value (exact_count_kernel).
// Costs ~ms per scan (every cell of every new centre's box is visited), so it
// is opt-in; the default path reports the concurrent change count.
#include "engine.cuh"

using namespace dbt;

namespace {

struct ExactArgs {
  const uint32_t* cm;     // masks (Cells::m), lazily lowered:
  const uint16_t* lc;     // effective mask = cm[v] & run_mask(lc[v]) (engine.cuh length cache)
  const uint64_t* uniq;
  const LaunchCounters* lc_in;
  unsigned long long* out;
  uint32_t* cbits;        // centre bitmap (storage index)
  uint32_t* tbits;        // touched-cell bitmap (storage index)
  uint32_t* rbits;        // centre-row bitmap (x*ny + y): rows holding a new centre
  uint32_t* m0;           // masks before the launch, touched cells only
  const uint8_t* len;     // K^3 kernel run lengths
  int64_t nx, ny, nzp, nz, n_words;
  int K, R;
};

__device__ __forceinline__ uint32_t run_mask(int len) { return len >= 32 ? 0xFFFFFFFFu : ((1u << len) - 1u); }

// bits [b, b + w) of a bitmap (w <= 32)
__device__ __forceinline__ uint32_t bits_at(const uint32_t* bm, int64_t b, int w) {
  const int64_t q = b >> 5;
  const int s = (int)(b & 31);
  const uint64_t v = (uint64_t)bm[q] | ((uint64_t)bm[q + 1] << 32);
  return (uint32_t)(v >> s) & (w >= 32 ? 0xFFFFFFFFu : ((1u << w) - 1u));
}

__device__ __forceinline__ void set_bits(uint32_t* bm, int64_t b, int w) {
  const int64_t q = b >> 5;
  const int s = (int)(b & 31);
  const uint64_t v = (uint64_t)((w >= 32 ? 0xFFFFFFFFull : ((1ull << w) - 1ull))) << s;
  if ((uint32_t)v) atomicOr(bm + q, (uint32_t)v);
  if ((uint32_t)(v >> 32)) atomicOr(bm + q + 1, (uint32_t)(v >> 32));
}

// warp per new centre: its bit in cbits and rbits, its K^3 box in tbits
__global__ void exact_mark_kernel(ExactArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t n = (int64_t)a.lc_in->n_unique;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t u = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); u < n; u += warps) {
    int64_t cx, cy, cz;
    unpack_center(a.uniq[u], cx, cy, cz);
    if (lane == 0) {
      const int64_t ci = (cx * a.ny + cy) * a.nzp + cz, ri = cx * a.ny + cy;
      atomicOr(a.cbits + (ci >> 5), 1u << (ci & 31));
      atomicOr(a.rbits + (ri >> 5), 1u << (ri & 31));
    }
    for (int r = lane; r < a.K * a.K; r += 32) {
      const int dx = r / a.K - a.R, dy = r % a.K - a.R;
      set_bits(a.tbits, ((cx + dx) * a.ny + (cy + dy)) * a.nzp + cz - a.R, a.K);
    }
  }
}

// masks of the touched cells before the sweep changes them
__global__ void exact_snap_kernel(ExactArgs a) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < a.n_words;
       w += (int64_t)gridDim.x * blockDim.x) {
    for (uint32_t bits = a.tbits[w]; bits; bits &= bits - 1) {
      const int64_t v = w * 32 + (__ffs(bits) - 1);
      a.m0[v] = a.cm[v] & run_mask(a.lc[v]);
    }
  }
}

__global__ void exact_clear_kernel(ExactArgs a) {
  const int64_t n = (int64_t)a.lc_in->n_unique;
  for (int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x) {
    int64_t cx, cy, cz;
    unpack_center(a.uniq[u], cx, cy, cz);
    const int64_t ci = (cx * a.ny + cy) * a.nzp + cz, ri = cx * a.ny + cy;
    a.cbits[ci >> 5] = 0u;  // every centre bit of these words is being cleared
    a.rbits[ri >> 5] = 0u;
  }
}

// After the sweep. Warps walk the touched bitmap 32 words at a time
// (clearing it); every non-zero word is processed with one lane per cell. A
// cell the launch did not change contributes 0; otherwise its lane replays
// the new centres of its box in lexicographic order — centre rows (cx, cy)
// from the row bitmap, their centres in z order from the centre bitmap —
// from the pre-launch mask, counting changes, and stops once the running
// mask reaches the final one (masks only lose bits). Run lengths in shared
// memory.
__global__ void exact_count_kernel(ExactArgs a) {
  extern __shared__ uint8_t s_len[];
  const int K = a.K, R = a.R, K3 = K * K * K;
  for (int i = threadIdx.x; i < K3; i += blockDim.x) s_len[i] = a.len[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  unsigned long long tot = 0;
  for (int64_t w0 = (blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5)) * 32; w0 < a.n_words;
       w0 += warps * 32) {
    uint32_t word = 0;
    if (w0 + lane < a.n_words) {
      word = a.tbits[w0 + lane];
      if (word) a.tbits[w0 + lane] = 0u;
    }
    for (unsigned todo = __ballot_sync(0xffffffffu, word != 0); todo; todo &= todo - 1) {
      const int src = __ffs(todo) - 1;
      const uint32_t bits = __shfl_sync(0xffffffffu, word, src);
      if (!((bits >> lane) & 1u)) continue;
      const int64_t v = (w0 + src) * 32 + lane;
      const uint32_t fin = a.cm[v] & run_mask(a.lc[v]);
      uint32_t m = a.m0[v];
      if (m == fin) continue;  // not changed by this launch
      const int64_t row = v / a.nzp, z = v - row * a.nzp;
      const int64_t x = row / a.ny, y = row - x * a.ny;
      const int64_t zlo = z - R < 0 ? 0 : z - R;
      const int64_t zhi = z + R > a.nz - 1 ? a.nz - 1 : z + R;
      const int w = (int)(zhi - zlo + 1);
      const int zoff = (int)(z - zlo);  // window bit j is centre z = zlo + j: kernel z index R + zoff - j
      const int64_t ylo = y - R < 0 ? 0 : y - R;
      const int64_t yhi = y + R > a.ny - 1 ? a.ny - 1 : y + R;
      const int wy = (int)(yhi - ylo + 1);
      unsigned cnt = 0;
      for (int ia = 0; ia < K && m != fin; ++ia) {
        const int64_t cx = x - R + ia;
        if (cx < 0 || cx >= a.nx) continue;
        for (uint32_t rows = bits_at(a.rbits, cx * a.ny + ylo, wy); rows && m != fin; rows &= rows - 1) {
          const int64_t cy = ylo + (__ffs(rows) - 1);
          const int ib = (int)(cy - (y - R));
          uint32_t win = bits_at(a.cbits, (cx * a.ny + cy) * a.nzp + zlo, w);
          // kernel offset v - c = (R - ia, R - ib, z - cz)
          const uint8_t* lrow = s_len + ((2 * R - ia) * K + (2 * R - ib)) * K + R + zoff;
          for (; win; win &= win - 1) {
            const uint32_t k = run_mask(lrow[-(__ffs(win) - 1)]);
            if ((m & k) != m) {
              ++cnt;
              m &= k;
            }
          }
        }
      }
      tot += cnt;
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, o);
  __shared__ unsigned long long s[32];
  if (lane == 0) s[threadIdx.x >> 5] = tot;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s[w];
    if (t) atomicAdd(a.out, t);
  }
}

ExactArgs exact_args(dbt_grid* g, const dbt_bank* b, int64_t n_words) {
  ExactArgs a;
  a.cm = g->cells.m;
  a.lc = g->dist;
  a.uniq = g->d_uniq;
  a.lc_in = g->d_lcnt;
  a.out = &g->d_lcnt->exact_written;
  a.cbits = g->d_exact_bits;
  a.tbits = g->d_exact_bits + n_words;
  a.rbits = g->d_exact_bits + 2 * n_words;
  a.m0 = g->d_exact_m0;
  a.len = b->d_len;
  a.nx = g->nx;
  a.ny = g->ny;
  a.nzp = g->nzp;
  a.nz = g->nz;
  a.n_words = n_words - 2;
  a.K = b->K;
  a.R = b->R;
  return a;
}

int64_t exact_words(const dbt_grid* g) { return (g->n_cells + 31) / 32 + 2; }

}  // namespace

namespace dbt {

// before the sweep: centre / row / touched bitmaps and the touched masks
int launch_exact_pre(dbt_grid* g, const dbt_bank* b, cudaStream_t st) {
  if (g->xm.w != 0 || g->xm.x0 != 0 || g->xm.x1 != g->nx)
    return set_error(DBT_ERR_CONFIG, "exact voxels_written needs a whole (unsharded) grid");
  const int64_t n_words = exact_words(g);
  const int64_t r_words = (g->nx * g->ny + 31) / 32 + 2;
  if (!g->d_exact_bits) {
    const size_t bytes = (size_t)(2 * n_words + r_words) * 4;
    DBT_CUDA(cudaMalloc(&g->d_exact_bits, bytes));
    DBT_CUDA(cudaMemsetAsync(g->d_exact_bits, 0, bytes, st));
    DBT_CUDA(cudaMalloc(&g->d_exact_m0, (size_t)g->n_cells * 4));
  }
  ExactArgs a = exact_args(g, b, n_words);
  int tok;
  prof_begin(g, "exact_mark_kernel", st, &tok);
  exact_mark_kernel<<<148 * 8, 256, 0, st>>>(a);
  prof_end(g, st, tok);
  DBT_CHECK_LAUNCH("exact_mark_kernel");
  exact_snap_kernel<<<148 * 8, 256, 0, st>>>(a);
  DBT_CHECK_LAUNCH("exact_snap_kernel");
  return DBT_OK;
}

// after the sweep: count the changes of the touched cells, clear the bitmaps
int launch_exact_post(dbt_grid* g, const dbt_bank* b, cudaStream_t st) {
  ExactArgs a = exact_args(g, b, exact_words(g));
  int tok;
  prof_begin(g, "exact_count_kernel", st, &tok);
  exact_count_kernel<<<148 * 8, 256, (size_t)b->K * b->K * b->K, st>>>(a);
  prof_end(g, st, tok);
  DBT_CHECK_LAUNCH("exact_count_kernel");
  exact_clear_kernel<<<148 * 4, 256, 0, st>>>(a);
  DBT_CHECK_LAUNCH("exact_clear_kernel");
  return DBT_OK;
}

}  // namespace dbt
