// grid.cu — device voxel store: allocation, host sync, DBTSDF01 records and
// the distance readout kernels (reference: grid.py:39-202).
#include <cstdlib>
#include <algorithm>
#include <cstring>

#include "engine.cuh"

using namespace dbt;

namespace dbt {

int grid_set_device(const dbt_grid* g) {
  DBT_CUDA(cudaSetDevice(g->device));
  return DBT_OK;
}

int ensure_stage(dbt_grid* g, int64_t bytes) {
  if (bytes <= g->cap_stage) return DBT_OK;
  if (g->d_stage) cudaFree(g->d_stage);
  g->d_stage = nullptr;
  g->cap_stage = 0;
  DBT_CUDA(cudaMalloc(&g->d_stage, (size_t)bytes));
  g->cap_stage = bytes;
  return DBT_OK;
}

}  // namespace dbt

namespace {

constexpr int64_t kStageBytes = 256ll << 20;

__global__ void fill_cells_kernel(Cells cells, uint16_t* __restrict__ dist, int64_t n) {
  // n is a multiple of 8 (allocation is padded); 128-bit stores of four
  // fresh masks and four fresh meta words, and of eight fresh cache lengths
  const uint4 vm = make_uint4(kFullMask, kFullMask, kFullMask, kFullMask);
  const uint4 vy = make_uint4(kFreshMeta, kFreshMeta, kFreshMeta, kFreshMeta);
  const uint4 vd = make_uint4(0x00200020u, 0x00200020u, 0x00200020u, 0x00200020u);
  uint4* pm = reinterpret_cast<uint4*>(cells.m);
  uint4* py = reinterpret_cast<uint4*>(cells.y);
  uint4* pd = reinterpret_cast<uint4*>(dist);
  int64_t n4 = n / 4;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4;
       i += (int64_t)gridDim.x * blockDim.x) {
    pm[i] = vm;
    py[i] = vy;
    if (!(i & 1)) pd[i >> 1] = vd;
  }
}

// Host C-order slice (xs, ny, nz) of mask/sign/hits -> device records. Any
// mask and sign byte the reference can hold is stored as is.
__global__ void encode_kernel(Cells cells, const uint32_t* __restrict__ mask,
                              const uint8_t* __restrict__ sign, const uint8_t* __restrict__ hits,
                              int64_t n, int64_t nz, int64_t nzp) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t row = i / nz, z = i - row * nz;
    cells.put(row * nzp + z, make_uint2(mask[i], make_meta(sign[i], hits[i])));
  }
}

// dist[v] = bit length of the mask of cells[v] over the whole slab (after host writes)
__global__ void rebuild_dist_kernel(const uint32_t* __restrict__ cm, uint16_t* __restrict__ dist, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    dist[i] = (uint16_t)mask_bitlen(cm[i]);
}

// pending shadow visits -> final sign/hits (pend), lazily lowered masks ->
// final masks (lazy: m &= run_mask(len)); no concurrent writers
__global__ void fold_kernel(Cells cells, const uint16_t* __restrict__ dist, int64_t n, int pend, int lazy,
                            uint32_t h_max, uint32_t t_occ) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (pend) {
      const uint32_t y = cells.y[i];
      if (y >> kPendShift) cells.y[i] = fold_meta(y, h_max, t_occ);
    }
    if (lazy) {
      const uint32_t m = cells.m[i], f = m & run_mask_of(dist[i]);
      if (f != m) cells.m[i] = f;
    }
  }
}

// distance cache of the z-range [z0, z1) only (chunked record loads)
__global__ void rebuild_dist_range_kernel(const uint32_t* __restrict__ cm, uint16_t* __restrict__ dist, int64_t rows,
                                          int64_t nzp, int64_t z0, int64_t z1) {
  const int64_t zc = z1 - z0, n = rows * zc;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t row = i / zc, off = row * nzp + z0 + (i - row * zc);
    dist[off] = (uint16_t)mask_bitlen(cm[off]);
  }
}

__global__ void decode_kernel(const Cells cells, uint32_t* __restrict__ mask,
                              uint8_t* __restrict__ sign, uint8_t* __restrict__ hits, int64_t n,
                              int64_t nz, int64_t nzp) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t row = i / nz, z = i - row * nz;
    const uint2 c = cells.get(row * nzp + z);
    mask[i] = c.x;
    sign[i] = meta_sign(c.y);
    hits[i] = meta_hits(c.y);
  }
}

// Readout (grid.py:161-175). mode 0: popcount int32; 1: observed u8;
// 2: signed distance f64 (+ observed u8). Decode = __popc of the mask
// (grid.py:124-129, 166-167).
__global__ void readout_kernel(const Cells cells, int mode, int32_t* __restrict__ pop,
                               uint8_t* __restrict__ obs, double* __restrict__ sdf, double vs,
                               int64_t n, int64_t nz, int64_t nzp) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t row = i / nz, z = i - row * nz;
    const uint2 c = cells.get(row * nzp + z);
    const int len = __popc(c.x);
    if (mode == 0) {
      pop[i] = len;
    } else {
      obs[i] = !(c.x == kFullMask && meta_hits(c.y) == 0);
      if (mode == 2) {
        // sigma * (popcount * voxel_size), sigma = -1 where sign == occupied:
        // keeps -0.0 like numpy
        double dist = __dmul_rn((double)len, vs);
        double sigma = meta_sign(c.y) == 0 ? -1.0 : 1.0;
        sdf[i] = __dmul_rn(sigma, dist);
      }
    }
  }
}

__global__ void count_kernel(const Cells cells, int64_t n, int64_t nz, int64_t nzp,
                             unsigned long long* __restrict__ out) {
  unsigned long long obs = 0, occ = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t row = i / nz, z = i - row * nz;
    const uint2 c = cells.get(row * nzp + z);
    obs += !(c.x == kFullMask && meta_hits(c.y) == 0);
    occ += meta_sign(c.y) == 0;
  }
  for (int o = 16; o; o >>= 1) {
    obs += __shfl_xor_sync(0xffffffffu, obs, o);
    occ += __shfl_xor_sync(0xffffffffu, occ, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicAdd(out, obs);
    atomicAdd(out + 1, occ);
  }
}

// F-order record transpose (grid.py:178-185): records of iz slab [z0, z0+zc)
// rec[(iz-z0)*nx*ny + iy*nx + ix] <- cell(ix, iy, iz). The device record IS
// the serialized record (reserved bytes 0); tile 32 (x) x 32 (z) per block at
// fixed iy so both the cell reads (along z) and the record writes (along x)
// are coalesced.
__global__ void to_records_kernel(const Cells cells, uint2* __restrict__ rec, int64_t nx,
                                  int64_t ny, int64_t nzp, int64_t z0, int64_t zc) {
  __shared__ uint2 tile[32][33];
  int64_t iy = blockIdx.y;
  int64_t xb = blockIdx.x * 32, zb = blockIdx.z * 32;
  int tx = threadIdx.x, ty = threadIdx.y;  // 32 x 8
  for (int k = ty; k < 32; k += 8) {
    int64_t ix = xb + k, iz = zb + tx;
    uint2 v = make_uint2(0, 0);
    if (ix < nx && iz < zc) v = cells.get((ix * ny + iy) * nzp + z0 + iz);
    tile[k][tx] = v;
  }
  __syncthreads();
  for (int k = ty; k < 32; k += 8) {
    int64_t iz = zb + k, ix = xb + tx;
    if (ix < nx && iz < zc) rec[iz * nx * ny + iy * nx + ix] = tile[tx][k];
  }
}

__global__ void from_records_kernel(Cells cells, const uint2* __restrict__ rec, int64_t nx,
                                    int64_t ny, int64_t nzp, int64_t z0, int64_t zc) {
  __shared__ uint2 tile[32][33];
  int64_t iy = blockIdx.y;
  int64_t xb = blockIdx.x * 32, zb = blockIdx.z * 32;
  int tx = threadIdx.x, ty = threadIdx.y;
  for (int k = ty; k < 32; k += 8) {
    int64_t iz = zb + k, ix = xb + tx;
    uint2 v = make_uint2(0, 0);
    if (ix < nx && iz < zc) {
      v = rec[iz * nx * ny + iy * nx + ix];
      v.y &= 0xFFFFu;  // reserved bytes are ignored (grid.py:188-202)
    }
    tile[tx][k] = v;
  }
  __syncthreads();
  for (int k = ty; k < 32; k += 8) {
    int64_t ix = xb + k, iz = zb + tx;
    if (ix < nx && iz < zc) cells.put((ix * ny + iy) * nzp + z0 + iz, tile[k][tx]);
  }
}

__global__ void gather_kernel(const Cells cells, const int64_t* __restrict__ xyz, int64_t n,
                              XMap xm, int64_t ny, int64_t nzp, uint32_t* __restrict__ mask,
                              uint8_t* __restrict__ sign, uint8_t* __restrict__ hits) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint2 c = cells.get((xm.local(xyz[3 * i]) * ny + xyz[3 * i + 1]) * nzp + xyz[3 * i + 2]);
    mask[i] = c.x;
    sign[i] = meta_sign(c.y);
    hits[i] = meta_hits(c.y);
  }
}

int grid_blocks(int64_t n) {
  int64_t b = (n + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 16));
}

int check_grid(const dbt_grid* g) {
  if (!g) return set_error(DBT_ERR_CONFIG, "null grid handle");
  return grid_set_device(g);
}

}  // namespace

// the records read back are final: order after the last integration launch
// (it may have run on a caller's stream) and fold pending shadow visits
int dbt::fold_pending(dbt_grid* g, cudaStream_t st) {
  if (g->last_st != st) {
    // the last launch ran on a caller's stream (which may be gone by now)
    DBT_CUDA(cudaDeviceSynchronize());
    g->last_st = st;
  }
  if (!g->pend && !g->lazy_m) return DBT_OK;
  fold_kernel<<<grid_blocks(g->n_cells), 256, 0, st>>>(g->cells, g->dist, g->n_cells, g->pend ? 1 : 0,
                                                      g->lazy_m ? 1 : 0, (uint32_t)g->pend_h_max,
                                                      (uint32_t)g->pend_t_occ);
  DBT_CHECK_LAUNCH("fold_kernel");
  g->pend = false;
  g->lazy_m = false;
  return DBT_OK;
}

namespace {

// after host data replaced the records: rebuild the distance cache, drop
// every stamp certificate (host writes carry no stamp history)
int finish_host_write(dbt_grid* g) {
  g->base_valid = false;  // replica base: host data replaced the records
  g->lazy_m = false;      // every mask replaced; the cache is rebuilt from them
  rebuild_dist_kernel<<<grid_blocks(g->n_cells), 256, 0, g->stream>>>(g->cells.m, g->dist, g->n_cells);
  DBT_CHECK_LAUNCH("rebuild_dist_kernel");
  DBT_CUDA(cudaMemsetAsync(g->stamped, 0, (size_t)((g->n_cert + 63) / 32) * 4, g->stream));
  DBT_CUDA(cudaStreamSynchronize(g->stream));
  g->cert_dk = 0;
  g->base_valid = false;
  return DBT_OK;
}

}  // namespace

extern "C" {

static int create_grid(const int64_t dims[3], double voxel_size, const double origin[3], int device,
                       const XMap& xm, dbt_grid** out) {
  *out = nullptr;
  for (int i = 0; i < 3; ++i)
    if (dims[i] < 1) return set_error(DBT_ERR_CONFIG, "grid dims must be three positive counts");
  for (int i = 0; i < 3; ++i)
    if (dims[i] > kMaxDim)
      return set_error(DBT_ERR_CONFIG, "grid dim exceeds 2^21-1 voxels (packed centre encoding)");
  if (!(voxel_size > 0.0)) return set_error(DBT_ERR_CONFIG, "voxel_size must be positive");
  if (xm.x0 < 0 || xm.x1 > dims[0] || xm.x0 >= xm.x1)
    return set_error(DBT_ERR_CONFIG, "slab [x0, x1) must be a non-empty range inside [0, nx)");
  if (xm.w < 0 || xm.p < 1 || xm.r < 0 || xm.r >= xm.p)
    return set_error(DBT_ERR_CONFIG, "interleave needs width >= 1 and 0 <= part < parts");
  if (xm.planes() < 1) return set_error(DBT_ERR_CONFIG, "this part owns no x-plane of the grid");
  dbt_grid* g = new dbt_grid();
  g->device = device;
  g->nx = dims[0];
  g->ny = dims[1];
  g->nz = dims[2];
  g->nzp = (dims[2] + 7) & ~int64_t(7);
  g->x0 = xm.x0;
  g->x1 = xm.x1;
  g->xm = xm;
  g->lx = xm.planes();
  g->vs = voxel_size;
  for (int i = 0; i < 3; ++i) g->org[i] = origin[i];
  g->n_cells = g->lx * g->ny * g->nzp;
  g->n_cert = g->nx * g->ny * g->nzp;
  int rc = grid_set_device(g);
  if (rc) {
    delete g;
    return rc;
  }
  // +64 cells of slack: the sweep's aligned 4-cell chunks may read up to 3
  // cells past the last row of the slab (never written).
  // masks and meta words in one allocation: m = [0, n + 64), y = [n + 64, 2 (n + 64))
  uint32_t* base = nullptr;
  cudaError_t e = cudaMalloc(&base, (size_t)(g->n_cells + 64) * 2 * sizeof(uint32_t));
  if (e == cudaSuccess) g->cells = Cells{base, base + (g->n_cells + 64)};
  if (e == cudaSuccess) e = cudaMalloc(&g->dist, (size_t)(g->n_cells + 64) * sizeof(uint16_t));
  if (e == cudaSuccess) e = cudaMalloc(&g->stamped, (size_t)((g->n_cert + 63) / 32) * 4);
  if (e != cudaSuccess) {
    if (g->cells.m) cudaFree(g->cells.m);
    delete g;
    return cuda_error(e, "cudaMalloc(voxel grid)");
  }
  cudaStreamCreateWithFlags(&g->stream, cudaStreamNonBlocking);
  cudaEventCreate(&g->ev_a);
  cudaEventCreate(&g->ev_b);
  cudaEventCreateWithFlags(&g->ev_done, cudaEventDisableTiming);
  g->time_calls = getenv("DBT_DEVICE_MS") != nullptr;
  cudaEventCreateWithFlags(&g->ev_meta, cudaEventDisableTiming);
  cudaStreamCreateWithFlags(&g->aux, cudaStreamNonBlocking);
  cudaEventCreateWithFlags(&g->ev_fork, cudaEventDisableTiming);
  cudaEventCreateWithFlags(&g->ev_join, cudaEventDisableTiming);
  g->last_st = g->stream;
  static_assert(sizeof(LaunchCounters) % 32 == 0, "counter block alignment");
  const size_t cnt_bytes = sizeof(LaunchCounters) + sizeof(ScanCounters) * kMaxScansPerLaunch;
  e = cudaMalloc(&g->d_lcnt, cnt_bytes);
  if (e == cudaSuccess) g->d_scnt = reinterpret_cast<ScanCounters*>(g->d_lcnt + 1);
  // per-launch metadata, packed: scan_off (S+1) | src_off (S+1) | poses (12 S)
  // scan_off (S+1) | src_off (S+1) | poses (12 S) | scan pointers (S)
  const size_t meta_bytes = sizeof(int64_t) * (2 * (kMaxScansPerLaunch + 1) + 13 * kMaxScansPerLaunch);
  if (e == cudaSuccess) e = cudaMalloc(&g->d_scan_off, meta_bytes);
  if (e == cudaSuccess) e = cudaHostAlloc(&g->h_lcnt, cnt_bytes, cudaHostAllocDefault);
  if (e == cudaSuccess) g->h_scnt = reinterpret_cast<ScanCounters*>(g->h_lcnt + 1);
  if (e == cudaSuccess) e = cudaHostAlloc(&g->h_meta, meta_bytes, cudaHostAllocDefault);
  if (e != cudaSuccess) {
    int code = cuda_error(e, "grid metadata allocation");
    dbt_grid_destroy(g);
    return code;
  }
  rc = dbt_grid_reset(g);
  if (rc) {
    dbt_grid_destroy(g);
    return rc;
  }
  *out = g;
  return DBT_OK;
}

int dbt_grid_create(const int64_t dims[3], double voxel_size, const double origin[3], int device,
                    int64_t slab_x0, int64_t slab_x1, dbt_grid** out) {
  XMap xm;
  xm.x0 = slab_x0;
  xm.x1 = slab_x1;
  return create_grid(dims, voxel_size, origin, device, xm, out);
}

int dbt_grid_create_interleaved(const int64_t dims[3], double voxel_size, const double origin[3], int device,
                                int64_t width, int32_t parts, int32_t part, dbt_grid** out) {
  *out = nullptr;
  if (width < 1) return set_error(DBT_ERR_CONFIG, "interleave width must be >= 1");
  XMap xm;
  xm.x0 = 0;
  xm.x1 = dims[0];
  xm.w = width;
  xm.p = parts;
  xm.r = part;
  return create_grid(dims, voxel_size, origin, device, xm, out);
}

int dbt_grid_layout(const dbt_grid* g, int64_t* owned_planes, int64_t xmap[5]) {
  if (!g) return set_error(DBT_ERR_CONFIG, "null grid handle");
  *owned_planes = g->lx;
  xmap[0] = g->xm.x0;
  xmap[1] = g->xm.x1;
  xmap[2] = g->xm.w;
  xmap[3] = g->xm.p;
  xmap[4] = g->xm.r;
  return DBT_OK;
}

int dbt_grid_destroy(dbt_grid* g) {
  if (!g) return DBT_OK;
  cudaSetDevice(g->device);
  if (g->stream) cudaStreamSynchronize(g->stream);
  dbt::prof_flush(g);
  for (auto e : g->event_pool) cudaEventDestroy(e);
  void* dev[] = {g->cells.m, g->dist,  g->stamped, g->d_raw,  g->d_center, g->d_bin,     g->d_slot,    g->d_uniq,
                 g->d_hkey, g->d_hmin, g->d_sensor, g->d_outcome, g->d_scan_off,
                 g->d_lcnt, g->d_stage, g->d_rowoff, g->d_exact_bits, g->d_exact_m0, g->d_base_hits, g->d_base_mask,
                 g->d_ray, g->d_dirty, g->d_sel, g->d_ts};
  for (void* p : dev)
    if (p) cudaFree(p);
  void* host[] = {g->h_lcnt, g->h_meta};
  for (void* p : host)
    if (p) cudaFreeHost(p);
  if (g->ev_a) cudaEventDestroy(g->ev_a);
  if (g->ev_b) cudaEventDestroy(g->ev_b);
  if (g->ev_done) cudaEventDestroy(g->ev_done);
  if (g->ev_meta) cudaEventDestroy(g->ev_meta);
  if (g->h_stage) cudaFreeHost(g->h_stage);
  if (g->gexec) cudaGraphExecDestroy(g->gexec);
  if (g->ggraph) cudaGraphDestroy(g->ggraph);
  if (g->ev_fork) cudaEventDestroy(g->ev_fork);
  if (g->ev_join) cudaEventDestroy(g->ev_join);
  if (g->aux) cudaStreamDestroy(g->aux);
  for (auto& sl : g->aslot) {
    if (sl.copied) cudaEventDestroy(sl.copied);
    if (sl.done) cudaEventDestroy(sl.done);
    if (sl.d_buf) cudaFree(sl.d_buf);
    if (sl.h) cudaFreeHost(sl.h);
    if (sl.h_stage) cudaFreeHost(sl.h_stage);
  }
  if (g->cstream) cudaStreamDestroy(g->cstream);
  for (auto& e : g->aexec)
    if (e) cudaGraphExecDestroy(e);
  if (g->stream && g->own_stream) cudaStreamDestroy(g->stream);
  delete g;
  return DBT_OK;
}

int dbt_grid_reset(dbt_grid* g) {
  int rc = check_grid(g);
  if (rc) return rc;
  if (g->last_st != g->stream) {
    DBT_CUDA(cudaDeviceSynchronize());
    g->last_st = g->stream;
  }
  fill_cells_kernel<<<grid_blocks((g->n_cells + 64) / 4), 256, 0, g->stream>>>(g->cells, g->dist, g->n_cells + 64);
  g->pend = false;
  g->lazy_m = false;
  DBT_CHECK_LAUNCH("fill_cells_kernel");
  DBT_CUDA(cudaMemsetAsync(g->stamped, 0, (size_t)((g->n_cert + 63) / 32) * 4, g->stream));
  DBT_CUDA(cudaStreamSynchronize(g->stream));
  g->cert_dk = 0;
  g->base_valid = false;  // replica base: the records were rewritten (dbt_replica_mark again)
  return DBT_OK;
}

int dbt_grid_info(const dbt_grid* g, int64_t dims[3], int64_t slab[2], int64_t* device_bytes) {
  if (!g) return set_error(DBT_ERR_CONFIG, "null grid handle");
  dims[0] = g->nx;
  dims[1] = g->ny;
  dims[2] = g->nz;
  slab[0] = g->x0;
  slab[1] = g->x1;
  *device_bytes = (g->n_cells + 64) * (int64_t)(sizeof(uint2) + sizeof(uint16_t)) + (g->n_cert + 63) / 32 * 4;
  return DBT_OK;
}

int dbt_grid_upload(dbt_grid* g, const uint32_t* mask, const uint8_t* sign, const uint8_t* hits) {
  int rc = check_grid(g);
  if (rc) return rc;
  const int64_t lx = g->lx, plane = g->ny * g->nz;
  int64_t xs = std::max<int64_t>(1, std::min<int64_t>(lx, kStageBytes / (plane * 6)));
  rc = ensure_stage(g, xs * plane * 6);
  if (rc) return rc;
  if (g->last_st != g->stream) {
    DBT_CUDA(cudaDeviceSynchronize());
    g->last_st = g->stream;
  }
  g->pend = false;  // every record of the slab is replaced
  uint8_t* st = (uint8_t*)g->d_stage;
  for (int64_t x = 0; x < lx; x += xs) {
    int64_t cx = std::min(xs, lx - x), n = cx * plane;
    uint32_t* dm = (uint32_t*)st;
    uint8_t* ds = st + 4 * n;
    uint8_t* dh = ds + n;
    DBT_CUDA(cudaMemcpyAsync(dm, mask + x * plane, 4 * n, cudaMemcpyHostToDevice, g->stream));
    DBT_CUDA(cudaMemcpyAsync(ds, sign + x * plane, n, cudaMemcpyHostToDevice, g->stream));
    DBT_CUDA(cudaMemcpyAsync(dh, hits + x * plane, n, cudaMemcpyHostToDevice, g->stream));
    encode_kernel<<<grid_blocks(n), 256, 0, g->stream>>>(g->cells.off(x * g->ny * g->nzp), dm, ds, dh, n,
                                                         g->nz, g->nzp);
    DBT_CHECK_LAUNCH("encode_kernel");
  }
  return finish_host_write(g);
}

// local (storage) planes [l_begin, l_end) -> host arrays of that many planes
static int download_local(dbt_grid* g, int64_t l_begin, int64_t l_end, uint32_t* mask, uint8_t* sign,
                          uint8_t* hits) {
  const int64_t lx = l_end - l_begin, plane = g->ny * g->nz;
  if (lx == 0) return DBT_OK;
  int rc = fold_pending(g, g->stream);
  if (rc) return rc;
  int64_t xs = std::max<int64_t>(1, std::min<int64_t>(lx, kStageBytes / (plane * 6)));
  rc = ensure_stage(g, xs * plane * 6);
  if (rc) return rc;
  uint8_t* st = (uint8_t*)g->d_stage;
  for (int64_t x = 0; x < lx; x += xs) {
    int64_t cx = std::min(xs, lx - x), n = cx * plane;
    uint32_t* dm = (uint32_t*)st;
    uint8_t* ds = st + 4 * n;
    uint8_t* dh = ds + n;
    decode_kernel<<<grid_blocks(n), 256, 0, g->stream>>>(g->cells.off((l_begin + x) * g->ny * g->nzp), dm, ds,
                                                         dh, n, g->nz, g->nzp);
    DBT_CHECK_LAUNCH("decode_kernel");
    DBT_CUDA(cudaMemcpyAsync(mask + x * plane, dm, 4 * n, cudaMemcpyDeviceToHost, g->stream));
    DBT_CUDA(cudaMemcpyAsync(sign + x * plane, ds, n, cudaMemcpyDeviceToHost, g->stream));
    DBT_CUDA(cudaMemcpyAsync(hits + x * plane, dh, n, cudaMemcpyDeviceToHost, g->stream));
    DBT_CUDA(cudaStreamSynchronize(g->stream));  // staging reused by the next slice
  }
  return DBT_OK;
}

int dbt_grid_download_range(dbt_grid* g, int64_t x_begin, int64_t x_end, uint32_t* mask, uint8_t* sign,
                            uint8_t* hits) {
  int rc = check_grid(g);
  if (rc) return rc;
  if (x_begin > x_end) return set_error(DBT_ERR_CONFIG, "download range outside the grid's owned planes");
  if (x_begin == x_end) return DBT_OK;
  // the global planes must be owned and stored contiguously (one slab, or
  // inside one interleave block)
  const int64_t lb = g->xm.local(x_begin), le = g->xm.local(x_end - 1);
  if (lb < 0 || le < 0 || le - lb != x_end - 1 - x_begin)
    return set_error(DBT_ERR_CONFIG, "download range outside the grid's owned planes");
  return download_local(g, lb, le + 1, mask, sign, hits);
}

int dbt_grid_download(dbt_grid* g, uint32_t* mask, uint8_t* sign, uint8_t* hits) {
  int rc = check_grid(g);
  if (rc) return rc;
  return download_local(g, 0, g->lx, mask, sign, hits);
}

static int readout(dbt_grid* g, int mode, int32_t* pop, uint8_t* obs, double* sdf) {
  int rc = check_grid(g);
  if (!rc) rc = fold_pending(g, g->stream);
  if (rc) return rc;
  const int64_t lx = g->lx, plane = g->ny * g->nz;
  const int64_t per = mode == 0 ? 4 : (mode == 1 ? 1 : 9);
  int64_t xs = std::max<int64_t>(1, std::min<int64_t>(lx, kStageBytes / (plane * per)));
  rc = ensure_stage(g, xs * plane * per);
  if (rc) return rc;
  uint8_t* st = (uint8_t*)g->d_stage;
  for (int64_t x = 0; x < lx; x += xs) {
    int64_t cx = std::min(xs, lx - x), n = cx * plane;
    int32_t* dp = (int32_t*)st;
    double* dsdf = (double*)st;
    uint8_t* dob = mode == 2 ? st + 8 * n : st;
    readout_kernel<<<grid_blocks(n), 256, 0, g->stream>>>(g->cells.off(x * g->ny * g->nzp), mode, dp, dob,
                                                          dsdf, g->vs, n, g->nz, g->nzp);
    DBT_CHECK_LAUNCH("readout_kernel");
    if (mode == 0) {
      DBT_CUDA(cudaMemcpyAsync(pop + x * plane, dp, 4 * n, cudaMemcpyDeviceToHost, g->stream));
    } else {
      DBT_CUDA(cudaMemcpyAsync(obs + x * plane, dob, n, cudaMemcpyDeviceToHost, g->stream));
      if (mode == 2)
        DBT_CUDA(cudaMemcpyAsync(sdf + x * plane, dsdf, 8 * n, cudaMemcpyDeviceToHost, g->stream));
    }
    DBT_CUDA(cudaStreamSynchronize(g->stream));
  }
  return DBT_OK;
}

int dbt_popcount(dbt_grid* g, int32_t* out) { return readout(g, 0, out, nullptr, nullptr); }
int dbt_observed(dbt_grid* g, uint8_t* out) { return readout(g, 1, nullptr, out, nullptr); }
int dbt_signed_distance_field(dbt_grid* g, double* field, uint8_t* observed) {
  return readout(g, 2, nullptr, observed, field);
}

int dbt_grid_counts(dbt_grid* g, int64_t* observed, int64_t* occupied) {
  int rc = check_grid(g);
  if (rc) return rc;
  rc = ensure_stage(g, 16);
  if (!rc) rc = fold_pending(g, g->stream);
  if (rc) return rc;
  unsigned long long* d = (unsigned long long*)g->d_stage;
  DBT_CUDA(cudaMemsetAsync(d, 0, 16, g->stream));
  const int64_t n = g->lx * g->ny * g->nz;
  count_kernel<<<grid_blocks(n), 256, 0, g->stream>>>(g->cells, n, g->nz, g->nzp, d);
  DBT_CHECK_LAUNCH("count_kernel");
  unsigned long long h[2];
  DBT_CUDA(cudaMemcpyAsync(h, d, 16, cudaMemcpyDeviceToHost, g->stream));
  DBT_CUDA(cudaStreamSynchronize(g->stream));
  *observed = (int64_t)h[0];
  *occupied = (int64_t)h[1];
  return DBT_OK;
}

int dbt_grid_gather(dbt_grid* g, const int64_t* xyz, int64_t n, uint32_t* mask, uint8_t* sign, uint8_t* hits) {
  int rc = check_grid(g);
  if (rc) return rc;
  for (int64_t i = 0; i < n; ++i) {
    const int64_t x = xyz[3 * i], y = xyz[3 * i + 1], z = xyz[3 * i + 2];
    if (g->xm.local(x) < 0 || y < 0 || y >= g->ny || z < 0 || z >= g->nz)
      return set_error(DBT_ERR_CONFIG, "voxel index outside the grid (or the owned slab)");
  }
  if (n == 0) return DBT_OK;
  rc = ensure_stage(g, n * 30);
  if (rc) return rc;
  uint8_t* st = (uint8_t*)g->d_stage;
  int64_t* didx = (int64_t*)st;
  uint32_t* dm = (uint32_t*)(st + 24 * n);
  uint8_t* ds = st + 28 * n;
  uint8_t* dh = ds + n;
  rc = fold_pending(g, g->stream);
  if (rc) return rc;
  DBT_CUDA(cudaMemcpyAsync(didx, xyz, 24 * n, cudaMemcpyHostToDevice, g->stream));
  gather_kernel<<<grid_blocks(n), 256, 0, g->stream>>>(g->cells, didx, n, g->xm, g->ny, g->nzp, dm, ds, dh);
  DBT_CHECK_LAUNCH("gather_kernel");
  if (mask) DBT_CUDA(cudaMemcpyAsync(mask, dm, 4 * n, cudaMemcpyDeviceToHost, g->stream));
  if (sign) DBT_CUDA(cudaMemcpyAsync(sign, ds, n, cudaMemcpyDeviceToHost, g->stream));
  if (hits) DBT_CUDA(cudaMemcpyAsync(hits, dh, n, cudaMemcpyDeviceToHost, g->stream));
  DBT_CUDA(cudaStreamSynchronize(g->stream));
  return DBT_OK;
}

int dbt_grid_to_records_range(dbt_grid* g, int64_t z_begin, int64_t z_end, void* out_records) {
  int rc = check_grid(g);
  if (rc) return rc;
  if (g->x0 != 0 || g->x1 != g->nx || g->xm.w != 0)
    return set_error(DBT_ERR_CONFIG, "records are defined for a whole grid, not a slab");
  if (g->ny > 65535) return set_error(DBT_ERR_CONFIG, "record transpose supports ny <= 65535");
  if (z_begin < 0 || z_end > g->nz || z_begin > z_end) return set_error(DBT_ERR_CONFIG, "z range outside the grid");
  const int64_t plane = g->nx * g->ny;
  int64_t zs = std::max<int64_t>(1, std::min<int64_t>(z_end - z_begin, kStageBytes / (plane * 8)));
  rc = ensure_stage(g, zs * plane * 8);
  if (!rc) rc = fold_pending(g, g->stream);
  if (rc) return rc;
  uint2* st = (uint2*)g->d_stage;
  for (int64_t z = z_begin; z < z_end; z += zs) {
    int64_t zc = std::min(zs, z_end - z);
    dim3 grid((unsigned)((g->nx + 31) / 32), (unsigned)g->ny, (unsigned)((zc + 31) / 32));
    to_records_kernel<<<grid, dim3(32, 8), 0, g->stream>>>(g->cells, st, g->nx, g->ny, g->nzp, z, zc);
    DBT_CHECK_LAUNCH("to_records_kernel");
    DBT_CUDA(cudaMemcpyAsync((uint64_t*)out_records + (z - z_begin) * plane, st, zc * plane * 8,
                             cudaMemcpyDeviceToHost, g->stream));
    DBT_CUDA(cudaStreamSynchronize(g->stream));
  }
  return DBT_OK;
}

int dbt_grid_to_records(dbt_grid* g, void* out_records) {
  int rc = check_grid(g);
  if (rc) return rc;
  return dbt_grid_to_records_range(g, 0, g->nz, out_records);
}

int dbt_grid_from_records_range(dbt_grid* g, int64_t z_begin, int64_t z_end, const void* records) {
  int rc = check_grid(g);
  if (rc) return rc;
  if (g->ny > 65535) return set_error(DBT_ERR_CONFIG, "record transpose supports ny <= 65535");
  if (g->x0 != 0 || g->x1 != g->nx || g->xm.w != 0)
    return set_error(DBT_ERR_CONFIG, "records are defined for a whole grid, not a slab");
  if (z_begin < 0 || z_end > g->nz || z_begin > z_end) return set_error(DBT_ERR_CONFIG, "z range outside the grid");
  const int64_t plane = g->nx * g->ny;
  int64_t zs = std::max<int64_t>(1, std::min<int64_t>(z_end - z_begin, kStageBytes / (plane * 8)));
  rc = ensure_stage(g, zs * plane * 8);
  if (!rc) rc = fold_pending(g, g->stream);  // records outside the range stay
  if (rc) return rc;
  uint2* st = (uint2*)g->d_stage;
  for (int64_t z = z_begin; z < z_end; z += zs) {
    int64_t zc = std::min(zs, z_end - z);
    DBT_CUDA(cudaMemcpyAsync(st, (const uint64_t*)records + (z - z_begin) * plane, zc * plane * 8,
                             cudaMemcpyHostToDevice, g->stream));
    dim3 grid((unsigned)((g->nx + 31) / 32), (unsigned)g->ny, (unsigned)((zc + 31) / 32));
    from_records_kernel<<<grid, dim3(32, 8), 0, g->stream>>>(g->cells, st, g->nx, g->ny, g->nzp, z, zc);
    DBT_CHECK_LAUNCH("from_records_kernel");
    DBT_CUDA(cudaStreamSynchronize(g->stream));
  }
  // distance cache of the written range; every stamp certificate dropped
  if (z_end > z_begin) {
    rebuild_dist_range_kernel<<<grid_blocks(plane * (z_end - z_begin)), 256, 0, g->stream>>>(
        g->cells.m, g->dist, plane, g->nzp, z_begin, z_end);
    DBT_CHECK_LAUNCH("rebuild_dist_range_kernel");
  }
  DBT_CUDA(cudaMemsetAsync(g->stamped, 0, (size_t)((g->n_cert + 63) / 32) * 4, g->stream));
  DBT_CUDA(cudaStreamSynchronize(g->stream));
  g->cert_dk = 0;
  g->base_valid = false;  // replica base: the records were rewritten
  return DBT_OK;
}

int dbt_grid_from_records(dbt_grid* g, const void* records) {
  int rc = check_grid(g);
  if (rc) return rc;
  return dbt_grid_from_records_range(g, 0, g->nz, records);
}

}  // extern "C"
