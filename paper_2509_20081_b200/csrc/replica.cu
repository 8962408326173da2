// replica.cu — data-parallel replicas of one grid and their exact merge
// (multi-GPU alternative to slab sharding).
//
// Every rank holds the whole grid and integrates its own scans. Because each
// update commutes, the sequential result over all ranks' scans is recovered
// from the replicas alone, given the state B they shared at the last merge:
//  * mask: every replica holds B.mask & run(L_r) with L_r its shortest stamp
//    run at the voxel; x -> B.mask & run(x) is monotone, so the AND over
//    replicas is the numeric MIN of the replica masks (an all-reduce MIN on
//    the order-preserving key mask ^ 0x80000000 as int32);
//  * hits: h_r = h0 >= h_max ? h0 : min(h0 + n_r, h_max) for n_r visits on
//    replica r (fold_meta), so h = h0 >= h_max ? h0 : min(h0 + sum(h_r - h0),
//    h_max) (an all-reduce SUM of the deltas h_r - h0);
//  * sign: a visit that leaves h' >= T clears it; the replicas' signs are B's
//    or 0, so sign = (sum of deltas > 0 && h >= T) ? 0 : MIN(sign_r).
// Distance-cache entries stay upper bounds (masks only lost bits) and are
// rebuilt; stamp certificates stay valid (each says its stamp was applied).
// dbt_replica_mark snapshots h0; pack writes the three reduce buffers; apply
// combines the reduced buffers into the record and re-marks.
#include "engine.cuh"

using namespace dbt;

namespace {

__global__ void replica_mark_kernel(const uint2* __restrict__ cells, uint8_t* __restrict__ base, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    base[i] = meta_hits(cells[i].y);
}

// compact C-order buffers over (lx, ny, nz) (no z padding)
__global__ void replica_pack_kernel(const uint2* __restrict__ cells, const uint8_t* __restrict__ base,
                                    int32_t* __restrict__ mkey, uint8_t* __restrict__ sign,
                                    int32_t* __restrict__ delta, int64_t n, int64_t nz, int64_t nzp) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / nz, v = row * nzp + (i - row * nz);
    const uint2 c = cells[v];
    mkey[i] = (int32_t)(c.x ^ 0x80000000u);
    sign[i] = meta_sign(c.y);
    delta[i] = (int32_t)meta_hits(c.y) - (int32_t)base[v];
  }
}

__global__ void replica_apply_kernel(uint2* __restrict__ cells, uint8_t* __restrict__ dist,
                                     uint8_t* __restrict__ base, const int32_t* __restrict__ mkey,
                                     const uint8_t* __restrict__ sign, const int32_t* __restrict__ delta,
                                     int64_t n, int64_t nz, int64_t nzp, int h_max, int t_occ) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / nz, v = row * nzp + (i - row * nz);
    const uint32_t m = (uint32_t)mkey[i] ^ 0x80000000u;
    const int h0 = base[v], d = delta[i];
    const int h = h0 >= h_max ? h0 : min(h0 + d, h_max);
    const uint32_t s = (d > 0 && h >= t_occ) ? 0u : (uint32_t)sign[i];
    cells[v] = make_uint2(m, make_meta(s, (uint32_t)h));
    dist[v] = (uint8_t)mask_bitlen(m);
    base[v] = (uint8_t)h;
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
  replica_mark_kernel<<<blocks_for(g->n_cells), 256, 0, g->stream>>>(g->cells, g->d_base_hits, g->n_cells);
  DBT_CHECK_LAUNCH("replica_mark_kernel");
  DBT_CUDA(cudaStreamSynchronize(g->stream));
  g->base_valid = true;
  return DBT_OK;
}

int dbt_replica_pack(dbt_grid* g, int32_t* mask_key, uint8_t* sign, int32_t* delta, void* stream) {
  int rc = check_whole(g);
  if (rc) return rc;
  if (!g->base_valid)
    return set_error(DBT_ERR_CONFIG, "no replica base: call dbt_replica_mark after creating, resetting or writing the grid");
  cudaStream_t st = stream ? (cudaStream_t)stream : g->stream;
  rc = fold_pending(g, st);
  if (rc) return rc;
  const int64_t n = g->nx * g->ny * g->nz;
  replica_pack_kernel<<<blocks_for(n), 256, 0, st>>>(g->cells, g->d_base_hits, mask_key, sign, delta, n, g->nz,
                                                     g->nzp);
  DBT_CHECK_LAUNCH("replica_pack_kernel");
  g->last_st = st;
  return DBT_OK;
}

int dbt_replica_apply(dbt_grid* g, const int32_t* mask_key_min, const uint8_t* sign_min, const int32_t* delta_sum,
                      int32_t h_max, int32_t t_occ, void* stream) {
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
  replica_apply_kernel<<<blocks_for(n), 256, 0, st>>>(g->cells, g->dist, g->d_base_hits, mask_key_min, sign_min,
                                                      delta_sum, n, g->nz, g->nzp, h_max, t_occ);
  DBT_CHECK_LAUNCH("replica_apply_kernel");
  g->last_st = st;
  return DBT_OK;
}

}  // extern "C"
