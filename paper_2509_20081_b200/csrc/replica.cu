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

__global__ void replica_apply_kernel(Cells cells, uint8_t* __restrict__ dist,
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
    dist[v] = (uint8_t)mask_bitlen(m);
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
  g->last_st = st;
  return DBT_OK;
}

}  // extern "C"
