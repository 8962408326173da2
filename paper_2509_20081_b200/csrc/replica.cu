// replica.cu — data-parallel replicas of one grid and their exact merge
// (multi-GPU alternative to slab sharding).
//
// Every rank holds the whole grid and integrates its own scans. Because each
// update commutes, the sequential result over all ranks' scans is recovered
// from the replicas alone, given the state B they shared at the last merge
// (dbt_replica_mark keeps B's masks and hit counts):
//  * mask: replica r holds m_r = B.mask & run(L_r) (L_r its shortest stamp
//    run at the voxel), which equals B.mask & run(bitlen(m_r)); the AND over
//    replicas is B.mask & run(min_r bitlen(m_r)) — an all-reduce MIN of one
//    byte per voxel;
//  * hits: h_r = h0 >= h_max ? h0 : min(h0 + n_r, h_max) for n_r visits on
//    replica r (fold_meta), so h = h0 >= h_max ? h0 : min(h0 + sum(h_r - h0),
//    h_max) — an all-reduce SUM of the deltas (<= 255 each) as float16, exact
//    below 2048 and >= 2048 (saturated anyway) above, whatever the order;
//  * sign: a visit that leaves h' >= T clears it; the replicas' signs are B's
//    or 0, so sign = (sum of deltas > 0 && h >= T) ? 0 : MIN(sign_r).
// 4 bytes per voxel travel. Distance-cache entries stay upper bounds (masks
// only lost bits) and are rebuilt; stamp certificates stay valid (each says
// its stamp was applied).
//
// Sparse merge (dbt_replica_dirty / _select / _pack_bricks / _apply_bricks):
// a voxel can change only inside the K^3 cube of a return some rank applied
// since the last merge (mask ANDs and shadow visits both stay within R of
// the centre). prep_kernel flags the 16^3 brick of every applied centre; the
// ranks OR their flags (all-reduce MAX of one byte per brick), every rank
// dilates them by ceil(R / 16) bricks and lists the result in brick order
// (identical lists on every rank), and only those bricks are packed, reduced
// and applied: 4 bytes per voxel of the selected bricks instead of the whole
// grid. Unselected bricks are unchanged since the last merge on every rank,
// so they already agree.
#include <cub/device/device_scan.cuh>
#include <cuda_fp16.h>

#include "engine.cuh"

using namespace dbt;

namespace {

__global__ void replica_mark_kernel(const Cells cells, uint32_t* __restrict__ bmask,
                                    uint8_t* __restrict__ bhits, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint2 c = cells.get(i);
    bmask[i] = c.x;
    bhits[i] = meta_hits(c.y);
  }
}

// compact C-order buffers over (nx, ny, nz) (no z padding)
__global__ void replica_pack_kernel(const Cells cells, const uint8_t* __restrict__ bhits,
                                    uint8_t* __restrict__ mlen, uint8_t* __restrict__ sign,
                                    __half* __restrict__ delta, int64_t n, int64_t nz, int64_t nzp) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / nz, v = row * nzp + (i - row * nz);
    const uint2 c = cells.get(v);
    mlen[i] = (uint8_t)mask_bitlen(c.x);
    sign[i] = meta_sign(c.y);
    delta[i] = __int2half_rn((int)meta_hits(c.y) - (int)bhits[v]);
  }
}

__global__ void replica_apply_kernel(Cells cells, uint16_t* __restrict__ dist,
                                     uint32_t* __restrict__ bmask, uint8_t* __restrict__ bhits,
                                     const uint8_t* __restrict__ mlen, const uint8_t* __restrict__ sign,
                                     const __half* __restrict__ delta, int64_t n, int64_t nz, int64_t nzp, int h_max,
                                     int t_occ) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / nz, v = row * nzp + (i - row * nz);
    const int len = mlen[i];
    const uint32_t m = bmask[v] & (len >= 32 ? 0xFFFFFFFFu : ((1u << len) - 1u));
    const int h0 = bhits[v];
    const int d = (int)fminf(__half2float(delta[i]), 4096.f);
    const int h = h0 >= h_max ? h0 : min(h0 + d, h_max);
    const uint32_t s = (d > 0 && h >= t_occ) ? 0u : (uint32_t)sign[i];
    cells.put(v, make_uint2(m, make_meta(s, (uint32_t)h)));
    dist[v] = (uint16_t)mask_bitlen(m);
    bmask[v] = m;
    bhits[v] = (uint8_t)h;
  }
}

constexpr int kBrick = 1 << kBrickShift;
constexpr int kBrickCells = kBrick * kBrick * kBrick;

// brick b is selected when a flagged brick lies within D bricks on every axis
__global__ void replica_select_kernel(const uint8_t* __restrict__ flags, int32_t* __restrict__ sel, int64_t bx,
                                      int64_t by, int64_t bz, int D) {
  const int64_t nb = bx * by * bz;
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x) {
    const int64_t x = b / (by * bz), y = (b / bz) % by, z = b % bz;
    int hit = 0;
    for (int64_t i = max((int64_t)0, x - D); i <= min(bx - 1, x + D) && !hit; ++i)
      for (int64_t j = max((int64_t)0, y - D); j <= min(by - 1, y + D) && !hit; ++j)
        for (int64_t k = max((int64_t)0, z - D); k <= min(bz - 1, z + D); ++k)
          if (flags[(i * by + j) * bz + k]) {
            hit = 1;
            break;
          }
    sel[b] = hit;
  }
}

__global__ void replica_compact_kernel(const int32_t* __restrict__ sel, const int32_t* __restrict__ pre,
                                       int32_t* __restrict__ out, int64_t nb) {
  for (int64_t b = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; b < nb; b += (int64_t)gridDim.x * blockDim.x)
    if (sel[b]) out[pre[b]] = (int32_t)b;
}

// voxel t (0..4095) of selected brick j: x-major, z fastest (16 consecutive
// z of a row per half warp)
struct BrickMap {
  int64_t by, bz, nx, ny, nz, nzp;
  __device__ __forceinline__ bool voxel(int32_t brick, int t, int64_t& v) const {
    const int64_t bxi = brick / (by * bz), byi = (brick / bz) % by, bzi = brick % bz;
    const int64_t x = (bxi << kBrickShift) + (t >> (2 * kBrickShift));
    const int64_t y = (byi << kBrickShift) + ((t >> kBrickShift) & (kBrick - 1));
    const int64_t z = (bzi << kBrickShift) + (t & (kBrick - 1));
    v = (x * ny + y) * nzp + z;
    return x < nx && y < ny && z < nz;
  }
};

// packed buffers of the selected bricks: mls = [n_sel * 4096 mask bit
// lengths | n_sel * 4096 signs], delta = n_sel * 4096 hit deltas; pending
// shadow visits and lazily lowered masks are folded on the fly (pend: the
// launch parameters)
__global__ void replica_pack_bricks_kernel(const Cells cells, const uint16_t* __restrict__ dist,
                                           const uint8_t* __restrict__ bhits,
                                           const int32_t* __restrict__ sel, int64_t n_sel, BrickMap bm, int pend,
                                           uint32_t ph, uint32_t pt, uint8_t* __restrict__ mls,
                                           __half* __restrict__ delta) {
  const int64_t tot = n_sel * kBrickCells;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t v;
    uint8_t ml = 0, sg = 0;
    int d = 0;
    if (bm.voxel(sel[i >> (3 * kBrickShift)], (int)(i & (kBrickCells - 1)), v)) {
      const uint32_t m = cells.m[v] & run_mask_of(dist[v]);  // the effective (lazily lowered) mask
      const uint32_t y = pend ? fold_meta(cells.y[v], ph, pt) : cells.y[v];
      ml = (uint8_t)mask_bitlen(m);
      sg = meta_sign(y);
      d = (int)meta_hits(y) - (int)bhits[v];
    }
    mls[i] = ml;
    mls[tot + i] = sg;
    delta[i] = __int2half_rn(d);
  }
}

__global__ void replica_apply_bricks_kernel(Cells cells, uint16_t* __restrict__ dist, uint32_t* __restrict__ bmask,
                                            uint8_t* __restrict__ bhits, const int32_t* __restrict__ sel,
                                            int64_t n_sel, BrickMap bm, const uint8_t* __restrict__ mls,
                                            const __half* __restrict__ delta, int h_max, int t_occ) {
  const int64_t tot = n_sel * kBrickCells;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    int64_t v;
    if (!bm.voxel(sel[i >> (3 * kBrickShift)], (int)(i & (kBrickCells - 1)), v)) continue;
    const int len = mls[i];
    const uint32_t m = bmask[v] & (len >= 32 ? 0xFFFFFFFFu : ((1u << len) - 1u));
    const int h0 = bhits[v];
    const int d = (int)fminf(__half2float(delta[i]), 4096.f);
    const int h = h0 >= h_max ? h0 : min(h0 + d, h_max);
    const uint32_t s = (d > 0 && h >= t_occ) ? 0u : (uint32_t)mls[tot + i];
    cells.put(v, make_uint2(m, make_meta(s, (uint32_t)h)));
    dist[v] = (uint16_t)mask_bitlen(m);
    bmask[v] = m;
    bhits[v] = (uint8_t)h;
  }
}

int blocks_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 16));
}

int check_whole(dbt_grid* g) {
  if (!g) return set_error(DBT_ERR_CONFIG, "null grid handle");
  if (g->xm.w != 0 || g->xm.x0 != 0 || g->xm.x1 != g->nx)
    return set_error(DBT_ERR_CONFIG, "replicas are whole (unsharded) grids");
  return grid_set_device(g);
}

}  // namespace

extern "C" {

int dbt_replica_mark(dbt_grid* g) {
  int rc = check_whole(g);
  if (!rc) rc = fold_pending(g, g->stream);
  if (rc) return rc;
  if (!g->d_base_hits) DBT_CUDA(cudaMalloc(&g->d_base_hits, (size_t)g->n_cells));
  if (!g->d_base_mask) DBT_CUDA(cudaMalloc(&g->d_base_mask, (size_t)g->n_cells * 4));
  replica_mark_kernel<<<blocks_for(g->n_cells), 256, 0, g->stream>>>(g->cells, g->d_base_mask, g->d_base_hits,
                                                                     g->n_cells);
  DBT_CHECK_LAUNCH("replica_mark_kernel");
  if (!g->d_dirty) {
    g->dbx = (g->nx + kBrick - 1) >> kBrickShift;
    g->dby = (g->ny + kBrick - 1) >> kBrickShift;
    g->dbz = (g->nz + kBrick - 1) >> kBrickShift;
    DBT_CUDA(cudaMalloc(&g->d_dirty, (size_t)(g->dbx * g->dby * g->dbz)));
  }
  DBT_CUDA(cudaMemsetAsync(g->d_dirty, 0, (size_t)(g->dbx * g->dby * g->dbz), g->stream));
  g->dirty_reach = 0;
  g->n_sel = 0;
  DBT_CUDA(cudaStreamSynchronize(g->stream));
  g->base_valid = true;
  return DBT_OK;
}

int dbt_replica_pack(dbt_grid* g, uint8_t* mask_len, uint8_t* sign, uint16_t* delta_f16, void* stream) {
  int rc = check_whole(g);
  if (rc) return rc;
  if (!g->base_valid)
    return set_error(DBT_ERR_CONFIG, "no replica base: call dbt_replica_mark after creating, resetting or writing the grid");
  cudaStream_t st = stream ? (cudaStream_t)stream : g->stream;
  rc = fold_pending(g, st);
  if (rc) return rc;
  const int64_t n = g->nx * g->ny * g->nz;
  replica_pack_kernel<<<blocks_for(n), 256, 0, st>>>(g->cells, g->d_base_hits, mask_len, sign,
                                                     reinterpret_cast<__half*>(delta_f16), n, g->nz, g->nzp);
  DBT_CHECK_LAUNCH("replica_pack_kernel");
  g->last_st = st;
  return DBT_OK;
}

int dbt_replica_apply(dbt_grid* g, const uint8_t* mask_len_min, const uint8_t* sign_min,
                      const uint16_t* delta_sum_f16, int32_t h_max, int32_t t_occ, void* stream) {
  int rc = check_whole(g);
  if (rc) return rc;
  if (!g->base_valid)
    return set_error(DBT_ERR_CONFIG, "no replica base: call dbt_replica_mark after creating, resetting or writing the grid");
  if (!(1 <= t_occ && t_occ <= h_max && h_max <= 255))
    return set_error(DBT_ERR_CONFIG, "need 1 <= T <= H_max <= 255");
  cudaStream_t st = stream ? (cudaStream_t)stream : g->stream;
  rc = fold_pending(g, st);
  if (rc) return rc;
  const int64_t n = g->nx * g->ny * g->nz;
  replica_apply_kernel<<<blocks_for(n), 256, 0, st>>>(g->cells, g->dist, g->d_base_mask, g->d_base_hits,
                                                      mask_len_min, sign_min,
                                                      reinterpret_cast<const __half*>(delta_sum_f16), n, g->nz,
                                                      g->nzp, h_max, t_occ);
  DBT_CHECK_LAUNCH("replica_apply_kernel");
  if (g->d_dirty) DBT_CUDA(cudaMemsetAsync(g->d_dirty, 0, (size_t)(g->dbx * g->dby * g->dbz), st));
  g->dirty_reach = 0;
  g->last_st = st;
  return DBT_OK;
}

int dbt_replica_bricks(dbt_grid* g, int64_t* n_bricks, int32_t* reach) {
  int rc = check_whole(g);
  if (rc) return rc;
  if (!g->base_valid || !g->d_dirty)
    return set_error(DBT_ERR_CONFIG, "no replica base: call dbt_replica_mark after creating, resetting or writing the grid");
  if (n_bricks) *n_bricks = g->dbx * g->dby * g->dbz;
  if (reach) *reach = g->dirty_reach;
  return DBT_OK;
}

int dbt_replica_dirty(dbt_grid* g, uint8_t* flags, void* stream) {
  int rc = dbt_replica_bricks(g, nullptr, nullptr);
  if (rc) return rc;
  cudaStream_t st = stream ? (cudaStream_t)stream : g->stream;
  if (g->last_st != st) {
    DBT_CUDA(cudaDeviceSynchronize());  // the last launch ran on another stream
    g->last_st = st;
  }
  DBT_CUDA(cudaMemcpyAsync(flags, g->d_dirty, (size_t)(g->dbx * g->dby * g->dbz), cudaMemcpyDeviceToDevice, st));
  return DBT_OK;
}

int dbt_replica_select(dbt_grid* g, const uint8_t* flags, int32_t reach, int64_t* n_sel, void* stream) {
  int rc = dbt_replica_bricks(g, nullptr, nullptr);
  if (rc) return rc;
  if (reach < 0) return set_error(DBT_ERR_CONFIG, "negative reach");
  cudaStream_t st = stream ? (cudaStream_t)stream : g->stream;
  const int64_t nb = g->dbx * g->dby * g->dbz;
  if (nb >= (1ll << 31)) return set_error(DBT_ERR_CONFIG, "too many bricks for a sparse merge");
  const int D = (reach + kBrick - 1) >> kBrickShift;
  int32_t *sel = nullptr, *pre = nullptr;
  void* tmp = nullptr;
  size_t tb = 0;
  DBT_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, (int32_t*)nullptr, (int32_t*)nullptr, (int)nb + 1, st));
  DBT_CUDA(cudaMallocAsync((void**)&sel, (size_t)(nb + 1) * 4, st));
  DBT_CUDA(cudaMallocAsync((void**)&pre, (size_t)(nb + 1) * 4, st));
  DBT_CUDA(cudaMallocAsync(&tmp, std::max<size_t>(tb, 1), st));
  DBT_CUDA(cudaMemsetAsync(sel + nb, 0, 4, st));
  replica_select_kernel<<<blocks_for(nb), 256, 0, st>>>(flags, sel, g->dbx, g->dby, g->dbz, D);
  DBT_CHECK_LAUNCH("replica_select_kernel");
  DBT_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tb, sel, pre, (int)nb + 1, st));
  int32_t cnt = 0;
  DBT_CUDA(cudaMemcpyAsync(&cnt, pre + nb, 4, cudaMemcpyDeviceToHost, st));
  DBT_CUDA(cudaStreamSynchronize(st));
  if (cnt > g->cap_sel) {
    if (g->d_sel) DBT_CUDA(cudaFree(g->d_sel));
    g->d_sel = nullptr;
    DBT_CUDA(cudaMalloc(&g->d_sel, (size_t)cnt * 4));
    g->cap_sel = cnt;
  }
  if (cnt) {
    replica_compact_kernel<<<blocks_for(nb), 256, 0, st>>>(sel, pre, g->d_sel, nb);
    DBT_CHECK_LAUNCH("replica_compact_kernel");
  }
  DBT_CUDA(cudaFreeAsync(sel, st));
  DBT_CUDA(cudaFreeAsync(pre, st));
  DBT_CUDA(cudaFreeAsync(tmp, st));
  g->n_sel = cnt;
  g->last_st = st;
  if (n_sel) *n_sel = cnt;
  return DBT_OK;
}

int dbt_replica_pack_bricks(dbt_grid* g, uint8_t* mask_len_sign, uint16_t* delta_f16, void* stream) {
  int rc = dbt_replica_bricks(g, nullptr, nullptr);
  if (rc) return rc;
  cudaStream_t st = stream ? (cudaStream_t)stream : g->stream;
  if (g->last_st != st) {
    DBT_CUDA(cudaDeviceSynchronize());
    g->last_st = st;
  }
  if (!g->n_sel) return DBT_OK;
  const BrickMap bm{g->dby, g->dbz, g->nx, g->ny, g->nz, g->nzp};
  replica_pack_bricks_kernel<<<blocks_for(g->n_sel * kBrickCells), 256, 0, st>>>(
      g->cells, g->dist, g->d_base_hits, g->d_sel, g->n_sel, bm, g->pend ? 1 : 0, (uint32_t)g->pend_h_max,
      (uint32_t)g->pend_t_occ, mask_len_sign, reinterpret_cast<__half*>(delta_f16));
  DBT_CHECK_LAUNCH("replica_pack_bricks_kernel");
  return DBT_OK;
}

int dbt_replica_apply_bricks(dbt_grid* g, const uint8_t* mask_len_sign_min, const uint16_t* delta_sum_f16,
                             int32_t h_max, int32_t t_occ, void* stream) {
  int rc = dbt_replica_bricks(g, nullptr, nullptr);
  if (rc) return rc;
  if (!(1 <= t_occ && t_occ <= h_max && h_max <= 255))
    return set_error(DBT_ERR_CONFIG, "need 1 <= T <= H_max <= 255");
  cudaStream_t st = stream ? (cudaStream_t)stream : g->stream;
  if (g->last_st != st) {
    DBT_CUDA(cudaDeviceSynchronize());
    g->last_st = st;
  }
  if (g->n_sel) {
    const BrickMap bm{g->dby, g->dbz, g->nx, g->ny, g->nz, g->nzp};
    replica_apply_bricks_kernel<<<blocks_for(g->n_sel * kBrickCells), 256, 0, st>>>(
        g->cells, g->dist, g->d_base_mask, g->d_base_hits, g->d_sel, g->n_sel, bm, mask_len_sign_min,
        reinterpret_cast<const __half*>(delta_sum_f16), h_max, t_occ);
    DBT_CHECK_LAUNCH("replica_apply_bricks_kernel");
  }
  // every pending visit and every lowering since the mark lay in a selected
  // brick: the records are final and the base is the merged grid again
  g->pend = false;
  g->lazy_m = false;
  DBT_CUDA(cudaMemsetAsync(g->d_dirty, 0, (size_t)(g->dbx * g->dby * g->dbz), st));
  g->dirty_reach = 0;
  g->n_sel = 0;
  return DBT_OK;
}

}  // extern "C"
