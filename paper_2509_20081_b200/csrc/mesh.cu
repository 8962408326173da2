// mesh.cu — marching cubes over the voxel-centre lattice, on the device
// (reference: mesher.py:43-110).
//
// The reference's output is reproduced exactly:
//   * triangles ordered by table slot k (0..4) first, then by cell in C order
//     (mesher.py:73-87), each row the indices of its three lattice edges;
//   * vertices = the referenced lattice edges sorted by key
//     ((x*ny + y)*nz + z)*3 + axis (np.unique, mesher.py:88), interpolated in
//     float64 with the reference's operation order (mesher.py:91-109).
// Sorting is replaced by ranks: the padded storage index (x*ny + y)*nzp + z
// orders lattice points exactly like the reference key, so an edge's vertex
// index is the number of referenced edges before it in a 3-bit-per-point
// bitmap (prefix per 64 points + popcount).
//
// Pipeline (all on the grid stream, whole grids only):
//   flags   1 byte per voxel: bit0 inside (field < iso | field == iso & occupied,
//           mesher.py:50, from a 66-entry host table), bit1 observed (grid.py:161-163)
//   select  active cells (all 8 corners observed, EDGE_TABLE[cube] != 0,
//           mesher.py:52-65) in C order (cub::DeviceSelect, counted first)
//   cells   cube per active cell; bits 2..4 of the flags of every lattice
//           edge its triangles use (atomicOr on the 4-byte word)
//   ranks   referenced-edge count per 64 points, exclusive scan -> vertex count
//   verts   one thread per 8 lattice points writes its vertices at their ranks
//   tris    per slot an exclusive scan of "slot present" over the active cells;
//           one thread per active cell writes its triangles
//
// The marching-cubes tables are an input (dbt_mc_tables, filled by the caller
// from the reference's _mc_tables.py), not data compiled into the engine.
#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>
#include <cub/device/device_select.cuh>
#include <thrust/iterator/counting_iterator.h>
#include <thrust/iterator/transform_iterator.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "engine.cuh"

struct dbt_mesh {
  int device = 0;
  int64_t nv = 0, nf = 0;
  double* vert = nullptr;    // (nv, 3) float64
  int64_t* tri = nullptr;    // (nf, 3) int64
  double* nrm = nullptr;     // (nv, 3) float64 once dbt_mesh_normals ran
};

using namespace dbt;

namespace {

constexpr uint64_t kEdgeBits = 0x1C1C1C1C1C1C1C1CULL;  // bits 2..4 of every byte

// derived, device-resident copy of the caller's tables
struct MeshTab {
  int8_t tri[256][16];
  uint8_t slots[256];     // bit k: slot k holds a triangle (TRI_TABLE[c][3k] >= 0)
  uint8_t active[256];    // EDGE_TABLE[c] != 0
  uint16_t used[256];     // cube edges the present slots reference
  int8_t axis[12];
  int64_t eoff[12];       // storage offset of the edge's lower lattice point
};

// one warp per (x, y) row, 4 z per lane: 16-byte mask and meta loads, 4-byte flag stores
__global__ void mesh_flags_kernel(const Cells cells, uint8_t* __restrict__ flags, int64_t rows,
                                  int64_t nz, int64_t nzp, uint64_t ins_free, uint64_t ins_occ) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
    for (int64_t z = 4 * lane; z < nzp; z += 128) {
      const uint4 qm = *reinterpret_cast<const uint4*>(cells.m + r * nzp + z);
      const uint4 qy = *reinterpret_cast<const uint4*>(cells.y + r * nzp + z);
      const uint32_t mx[4] = {qm.x, qm.y, qm.z, qm.w}, my[4] = {qy.x, qy.y, qy.z, qy.w};
      uint32_t w = 0;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const uint64_t tab = meta_sign(my[k]) == 0 ? ins_occ : ins_free;
        const uint32_t f = (uint32_t)((tab >> __popc(mx[k])) & 1u) |
                           ((uint32_t)(!(mx[k] == kFullMask && meta_hits(my[k]) == 0)) << 1);
        w |= (z + k < nz ? f : 0u) << (8 * k);
      }
      *reinterpret_cast<uint32_t*>(flags + r * nzp + z) = w;
    }
  }
}

// Active cells (all 8 corners observed, EDGE_TABLE[cube] != 0; mesher.py:
// 52-65), one warp per cell row (x, y), 4 cells per lane. kEmit = false:
// per-row counts; kEmit = true: C-order cell list + cube at the row's scanned
// offset, and bits 2..4 (referenced lattice edges) of the flags of every edge
// the cell's triangles use (atomicOr; other lanes only read bits 0..1).
struct RowGeom {
  int64_t nx, ny, nz, nzp;
  int64_t roff[4];  // the four corner rows (ox*ny + oy)*nzp, (ox, oy) in {0,1}^2
  int crow[8];      // corner -> its row
  int oz[8];        // corner z offset
};

template <bool kEmit>
__global__ void __launch_bounds__(256, 8) mesh_active_kernel(uint8_t* __restrict__ flags, const MeshTab* __restrict__ t,
                                                          RowGeom rg, unsigned long long* __restrict__ rowcnt,
                                                          int64_t* __restrict__ cell_out,
                                                          uint8_t* __restrict__ cube_out) {
  __shared__ uint8_t s_active[256];
  __shared__ uint16_t s_used[256];
  __shared__ int64_t s_eoff[12];
  __shared__ uint32_t s_ebit[12];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) {
    s_active[i] = t->active[i];
    s_used[i] = t->used[i];
  }
  if (threadIdx.x < 12) {
    s_eoff[threadIdx.x] = t->eoff[threadIdx.x];
    s_ebit[threadIdx.x] = 1u << (2 + t->axis[threadIdx.x]);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t rows = (rg.nx - 1) * rg.ny, zc = rg.nz - 1;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  for (int64_t r = blockIdx.x * (int64_t)(blockDim.x >> 5) + (threadIdx.x >> 5); r < rows; r += warps) {
    // y = ny-1 holds no cells; the emit pass also skips rows the count pass
    // found empty (scanned offsets equal)
    const bool edge_row = (r % rg.ny) == rg.ny - 1 || (kEmit && rowcnt[r + 1] == rowcnt[r]);
    const int64_t base = r * rg.nzp;
    unsigned long long run = kEmit ? rowcnt[r] : 0ull;
    for (int64_t z0 = 0; z0 < zc && !edge_row; z0 += 128) {
      const int64_t z = z0 + 4 * lane;
      uint32_t amask = 0, cubes = 0;
      if (z < zc) {
        // flag bytes z .. z+7 of the four corner rows
        uint64_t row[4];
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const uint8_t* q = flags + base + rg.roff[q4] + z;
          row[q4] = (uint64_t)*reinterpret_cast<const uint32_t*>(q) |
                    ((uint64_t)*reinterpret_cast<const uint32_t*>(q + 4) << 32);
        }
        // SWAR over the 4 cells: byte k of `cubes` collects bit c = inside
        // flag of corner c of cell z+k, byte k of `obs` = all corners observed
        uint32_t all = 0u, obs = 0x01010101u;
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const int q = rg.crow[c];  // selects, not a dynamically indexed (local-memory) array
          const uint64_t rw = q == 0 ? row[0] : q == 1 ? row[1] : q == 2 ? row[2] : row[3];
          const uint32_t vc = (uint32_t)(rw >> (8 * rg.oz[c]));
          all |= (vc & 0x01010101u) << c;
          obs &= vc >> 1;
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const uint32_t cube = (all >> (8 * k)) & 0xFFu;
          if (z + k < zc && ((obs >> (8 * k)) & 1u) && s_active[cube]) {
            amask |= 1u << k;
            cubes |= cube << (8 * k);
          }
        }
      }
      const uint32_t cnt = __popc(amask);
      uint32_t incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t u = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += u;
      }
      if (kEmit && amask) {
        unsigned long long j = run + incl - cnt;
        for (uint32_t mk = amask; mk; mk &= mk - 1, ++j) {
          const int k = __ffs(mk) - 1;
          const int64_t i = base + z + k;
          const uint32_t cube = (cubes >> (8 * k)) & 0xFFu;
          cell_out[j] = i;
          cube_out[j] = (uint8_t)cube;
          for (uint32_t u = s_used[cube]; u; u &= u - 1) {
            const int e = __ffs(u) - 1;
            const int64_t p = i + s_eoff[e];
            atomicOr(reinterpret_cast<unsigned int*>(flags + (p & ~int64_t(3))), s_ebit[e] << (8 * (int)(p & 3)));
          }
        }
      }
      run += __shfl_sync(0xffffffffu, incl, 31);
    }
    if (!kEmit && lane == 0) rowcnt[r] = run;
  }
}

// referenced edges per 64 lattice points (entry n_groups stays 0 for the scan)
__global__ void mesh_group_kernel(const uint64_t* __restrict__ fw, int64_t n_groups,
                                  unsigned long long* __restrict__ cnt) {
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g <= n_groups;
       g += (int64_t)gridDim.x * blockDim.x) {
    unsigned long long k = 0;
    if (g < n_groups) {
      const uint4* q = reinterpret_cast<const uint4*>(fw + 8 * g);
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const uint4 v = q[w];
        k += __popcll((((uint64_t)v.y << 32) | v.x) & kEdgeBits) + __popcll((((uint64_t)v.w << 32) | v.z) & kEdgeBits);
      }
    }
    cnt[g] = k;
  }
}

// vertex index of lattice edge (p, axis): referenced edges before it
__device__ __forceinline__ int64_t edge_rank(const uint64_t* __restrict__ fw,
                                             const unsigned long long* __restrict__ pre, int64_t p, int axis) {
  const int64_t w = p >> 3;
  int64_t r = (int64_t)pre[p >> 6];
  for (int64_t k = w & ~int64_t(7); k < w; ++k) r += __popcll(fw[k] & kEdgeBits);
  const int b = (int)(p & 7);
  const uint64_t below = (b ? ((1ull << (8 * b)) - 1) : 0ull) | (((1ull << axis) - 1) << (8 * b + 2));
  return r + __popcll(fw[w] & kEdgeBits & below);
}

// field value of a voxel: sigma * (popcount * voxel_size) (grid.py:170-175)
__device__ __forceinline__ double field_at(const Cells cells, int64_t i, double vs) {
  const uint2 c = cells.get(i);
  const double d = __dmul_rn((double)__popc(c.x), vs);
  return __dmul_rn(meta_sign(c.y) == 0 ? -1.0 : 1.0, d);
}

struct VertArgs {
  int64_t ny, nzp, n_words;
  double vs, iso, org[3];
};

// mesher.py:91-109, one thread per 8 lattice points
__global__ void mesh_vert_kernel(const Cells cells, const uint64_t* __restrict__ fw,
                                 const unsigned long long* __restrict__ pre, VertArgs a,
                                 double* __restrict__ vert) {
  for (int64_t w = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; w < a.n_words;
       w += (int64_t)gridDim.x * blockDim.x) {
    // groups of 64 points without a referenced edge are skipped on their
    // scanned counts (8 bytes per 8 words of flags)
    int64_t r = (int64_t)pre[w >> 3];
    if ((int64_t)pre[(w >> 3) + 1] == r) continue;
    uint64_t bits = fw[w] & kEdgeBits;
    if (!bits) continue;
    for (int64_t k = w & ~int64_t(7); k < w; ++k) r += __popcll(fw[k] & kEdgeBits);
    for (; bits; bits &= bits - 1, ++r) {
      const int pos = __ffsll((long long)bits) - 1;
      const int axis = (pos & 7) - 2;
      const int64_t p = w * 8 + (pos >> 3);
      const int64_t row = p / a.nzp, z = p - row * a.nzp;
      const int64_t x = row / a.ny, y = row - x * a.ny;
      const int64_t step = axis == 0 ? a.ny * a.nzp : (axis == 1 ? a.nzp : 1);
      const double v1 = field_at(cells, p, a.vs), v2 = field_at(cells, p + step, a.vs);
      const double den = __dsub_rn(v2, v1);
      double t = den != 0.0 ? __ddiv_rn(__dsub_rn(a.iso, v1), den) : 0.0;
      t = t < 0.0 ? 0.0 : t;  // np.clip keeps -0.0 and NaN
      t = t > 1.0 ? 1.0 : t;
      const int64_t b[3] = {x, y, z};
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const double p1 = __dadd_rn(a.org[d], __dmul_rn((double)b[d] + 0.5, a.vs));
        const double p2 = __dadd_rn(a.org[d], __dmul_rn((double)(b[d] + (d == axis)) + 0.5, a.vs));
        vert[3 * r + d] = __dadd_rn(p1, __dmul_rn(t, __dsub_rn(p2, p1)));
      }
    }
  }
}

struct SlotFlag {
  const uint8_t* cube;
  const MeshTab* t;
  int64_t n;
  int k;
  __device__ __forceinline__ unsigned long long operator()(int64_t j) const {
    return j < n ? (unsigned long long)((t->slots[cube[j]] >> k) & 1u) : 0ull;
  }
};

// mesher.py:72-89: triangle (slot k, j-th cell holding slot k) -> row
// slot_base[k] + rank_k(j); entries are vertex ranks of its three edges
__global__ void mesh_tri_kernel(const int64_t* __restrict__ cell, const uint8_t* __restrict__ cube_in,
                                int64_t n_active, const unsigned long long* __restrict__ rank, int64_t rank_pitch,
                                const MeshTab* __restrict__ t, const uint64_t* __restrict__ fw,
                                const unsigned long long* __restrict__ pre, int64_t base0, int64_t base1,
                                int64_t base2, int64_t base3, int64_t base4, int64_t* __restrict__ tri) {
  const int64_t base[5] = {base0, base1, base2, base3, base4};
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < n_active;
       j += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = cell[j];
    const int cube = cube_in[j];
    const int slots = t->slots[cube];
    for (int k = 0; k < 5; ++k) {
      if (!((slots >> k) & 1)) continue;
      const int64_t row = base[k] + (int64_t)rank[k * rank_pitch + j];
#pragma unroll
      for (int m = 0; m < 3; ++m) {
        const int e = t->tri[cube][3 * k + m];
        tri[3 * row + m] = edge_rank(fw, pre, i + t->eoff[e], t->axis[e]);
      }
    }
  }
}

// ---- vertex normals (mesher.py:113-127) ----------------------------------
// face normal = cross(v1 - v0, v2 - v0) with numpy's operation order
// (a1*b2 - a2*b1, a2*b0 - a0*b2, a0*b1 - a1*b0); one (key = vertex, value =
// j*nf + f) pair per triangle corner, in the order np.add.at visits them.
// Negative indices wrap like numpy; anything else out of range sets *bad.
__global__ void mesh_face_kernel(const double* __restrict__ v, const int64_t* __restrict__ tri, int64_t nv,
                                 int64_t nf, double* __restrict__ fn, uint32_t* __restrict__ key,
                                 int64_t* __restrict__ val, uint32_t* __restrict__ deg, int* __restrict__ bad) {
  for (int64_t f = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; f < nf;
       f += (int64_t)gridDim.x * blockDim.x) {
    int64_t id[3];
    bool ok = true;
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      int64_t k = tri[3 * f + j];
      if (k < 0) k += nv;
      ok &= k >= 0 && k < nv;
      id[j] = k;
    }
    if (!ok) {
      *bad = 1;
      continue;
    }
    double a[3], b[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      a[d] = __dsub_rn(v[3 * id[1] + d], v[3 * id[0] + d]);
      b[d] = __dsub_rn(v[3 * id[2] + d], v[3 * id[0] + d]);
    }
    fn[3 * f + 0] = __dsub_rn(__dmul_rn(a[1], b[2]), __dmul_rn(a[2], b[1]));
    fn[3 * f + 1] = __dsub_rn(__dmul_rn(a[2], b[0]), __dmul_rn(a[0], b[2]));
    fn[3 * f + 2] = __dsub_rn(__dmul_rn(a[0], b[1]), __dmul_rn(a[1], b[0]));
#pragma unroll
    for (int j = 0; j < 3; ++j) {
      key[j * nf + f] = (uint32_t)id[j];
      val[j * nf + f] = j * nf + f;
      atomicAdd(deg + id[j], 1u);
    }
  }
}

// per vertex: sequential sum of its corner normals in np.add.at order, then
// norm = sqrt((x*x + y*y) + z*z) (np.linalg.norm) and the division
__global__ void mesh_normal_kernel(const double* __restrict__ fn, const int64_t* __restrict__ val,
                                   const uint32_t* __restrict__ off, int64_t nv, int64_t nf,
                                   double* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nv;
       i += (int64_t)gridDim.x * blockDim.x) {
    double x = 0.0, y = 0.0, z = 0.0;
    for (uint32_t k = off[i]; k < off[i + 1]; ++k) {
      const int64_t e = val[k], f = e % nf;
      x = __dadd_rn(x, fn[3 * f]);
      y = __dadd_rn(y, fn[3 * f + 1]);
      z = __dadd_rn(z, fn[3 * f + 2]);
    }
    const double n = __dsqrt_rn(__dadd_rn(__dadd_rn(__dmul_rn(x, x), __dmul_rn(y, y)), __dmul_rn(z, z)));
    if (n > 0.0) {
      x = __ddiv_rn(x, n);
      y = __ddiv_rn(y, n);
      z = __ddiv_rn(z, n);
    }
    out[3 * i] = x;
    out[3 * i + 1] = y;
    out[3 * i + 2] = z;
  }
}

int blocks_for(int64_t n) {
  int64_t b = (n + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148 * 16));
}

// Mesh buffers come from the device's stream-ordered pool: repeated
// extractions reuse memory instead of paying cudaMalloc/cudaFree (which
// synchronise the device) per call. Up to kPoolKeep bytes stay reserved.
constexpr uint64_t kPoolKeep = 2ull << 30;

int pool_init(int device) {
  static bool done[256] = {};
  if (device < 0 || device >= 256 || done[device]) return DBT_OK;
  cudaMemPool_t pool;
  DBT_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
  uint64_t keep = kPoolKeep;
  DBT_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
  done[device] = true;
  return DBT_OK;
}

template <class T>
int pool_alloc(T** p, int64_t count, cudaStream_t st, const char* what) {
  *p = nullptr;
  cudaError_t e = cudaMallocAsync((void**)p, (size_t)std::max<int64_t>(1, count) * sizeof(T), st);
  return e == cudaSuccess ? DBT_OK : cuda_error(e, what);
}

// device scratch, released (stream-ordered) on every exit path
struct Scratch {
  cudaStream_t st;
  std::vector<void*> ptrs;
  explicit Scratch(cudaStream_t s) : st(s) {}
  template <class T>
  int alloc(T** p, int64_t count) {
    int rc = pool_alloc(p, count, st, "mesh scratch allocation");
    if (!rc) ptrs.push_back((void*)*p);
    return rc;
  }
  ~Scratch() {
    for (void* p : ptrs) cudaFreeAsync(p, st);
  }
};

int check_tables(const dbt_mc_tables* tb, MeshTab* h) {
  if (!tb) return set_error(DBT_ERR_CONFIG, "marching-cubes tables are required");
  std::memset(h, 0, sizeof(*h));
  for (int e = 0; e < 12; ++e) {
    const int ax = tb->edge_axis[e];
    if (ax < 0 || ax > 2) return set_error(DBT_ERR_CONFIG, "EDGE_AXIS entries must be 0, 1 or 2");
    for (int d = 0; d < 3; ++d)
      if (tb->edge_base[3 * e + d] < 0 || tb->edge_base[3 * e + d] > 1)
        return set_error(DBT_ERR_CONFIG, "EDGE_BASE entries must be 0 or 1");
    // the edge runs from its base to base + unit(axis): both inside the cube
    if (tb->edge_base[3 * e + ax] != 0) return set_error(DBT_ERR_CONFIG, "EDGE_BASE/EDGE_AXIS leave the cube");
    h->axis[e] = (int8_t)ax;
  }
  for (int c = 0; c < 8; ++c)
    for (int d = 0; d < 3; ++d)
      if (tb->corner_offsets[3 * c + d] < 0 || tb->corner_offsets[3 * c + d] > 1)
        return set_error(DBT_ERR_CONFIG, "CORNER_OFFSETS entries must be 0 or 1");
  for (int c = 0; c < 256; ++c) {
    h->active[c] = tb->edge_table[c] != 0;
    for (int m = 0; m < 16; ++m) {
      const int v = tb->tri_table[16 * c + m];
      if (v < -1 || v > 11) return set_error(DBT_ERR_CONFIG, "TRI_TABLE entries must be -1..11");
      h->tri[c][m] = (int8_t)v;
    }
    for (int k = 0; k < 5; ++k) {
      if (h->tri[c][3 * k] < 0) continue;
      h->slots[c] |= (uint8_t)(1u << k);
      for (int m = 0; m < 3; ++m) {
        const int e = h->tri[c][3 * k + m];
        if (e < 0) return set_error(DBT_ERR_CONFIG, "TRI_TABLE slot with fewer than three edges");
        h->used[c] |= (uint16_t)(1u << e);
      }
    }
  }
  return DBT_OK;
}

#define MESH_LAUNCH(name, grid_, call)          \
  do {                                          \
    int _tok;                                   \
    prof_begin(g, name, st, &_tok);             \
    call;                                       \
    prof_end(g, st, _tok);                      \
    DBT_CHECK_LAUNCH(name);                     \
  } while (0)

int extract_into(dbt_grid* g, double iso, const dbt_mc_tables* tables, MeshTab& h, dbt_mesh* m) {
  int rc;
  const int64_t nx = g->nx, ny = g->ny, nz = g->nz, nzp = g->nzp;
  if (nx < 2 || ny < 2 || nz < 2) return DBT_OK;  // empty mesh (mesher.py:45-47)
  cudaStream_t st = g->stream;
  RowGeom rg{nx, ny, nz, nzp, {}, {}, {}};
  for (int q4 = 0; q4 < 4; ++q4) rg.roff[q4] = ((q4 >> 1) * ny + (q4 & 1)) * nzp;
  for (int c = 0; c < 8; ++c) {
    const int32_t* o = tables->corner_offsets + 3 * c;
    rg.crow[c] = o[0] * 2 + o[1];
    rg.oz[c] = o[2];
  }
  for (int e = 0; e < 12; ++e)
    h.eoff[e] = (tables->edge_base[3 * e] * ny + tables->edge_base[3 * e + 1]) * nzp + tables->edge_base[3 * e + 2];
  // inside bit per (sign, popcount): field = sigma * (popcount * vs) (mesher.py:50)
  uint64_t ins_free = 0, ins_occ = 0;
  for (int k = 0; k <= 32; ++k) {
    const double d = (double)k * g->vs;
    const double fo = -1.0 * d, ff = 1.0 * d;
    if (ff < iso) ins_free |= 1ull << k;
    if (fo < iso || fo == iso) ins_occ |= 1ull << k;
  }

  const int64_t n = g->n_cells;                       // padded storage points (nzp % 8 == 0)
  const int64_t rows = nx * ny, cell_rows = (nx - 1) * ny;
  const int64_t n_groups = (n + 63) / 64, n_words = n_groups * 8;
  Scratch s(st);
  MeshTab* d_tab;
  uint8_t* flags;
  unsigned long long *pre, *rowoff;
  // flags: +64 bytes so the 8-byte corner loads of the last row stay inside
  if ((rc = s.alloc(&d_tab, 1)) || (rc = s.alloc(&flags, n_groups * 64 + 64)) || (rc = s.alloc(&pre, n_groups + 1)) ||
      (rc = s.alloc(&rowoff, cell_rows + 1)))
    return rc;
  DBT_CUDA(cudaMemcpyAsync(d_tab, &h, sizeof(h), cudaMemcpyHostToDevice, st));
  DBT_CUDA(cudaMemsetAsync(flags + n, 0, (size_t)(n_groups * 64 + 64 - n), st));
  DBT_CUDA(cudaMemsetAsync(rowoff + cell_rows, 0, 8, st));
  const int wblocks = (int)std::max<int64_t>(1, std::min<int64_t>((rows + 7) / 8, 148 * 8));
  const int cblocks = (int)std::max<int64_t>(1, std::min<int64_t>((cell_rows + 7) / 8, 148 * 8));
  MESH_LAUNCH("mesh_flags_kernel", wblocks,
              (mesh_flags_kernel<<<wblocks, 256, 0, st>>>(g->cells, flags, rows, nz, nzp, ins_free, ins_occ)));
  MESH_LAUNCH("mesh_active_count", cblocks,
              (mesh_active_kernel<false><<<cblocks, 256, 0, st>>>(flags, d_tab, rg, rowoff, nullptr, nullptr)));
  size_t tmp_rows = 0, tmp_groups = 0;
  DBT_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_rows, rowoff, cell_rows + 1, st));
  DBT_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_groups, pre, n_groups + 1, st));
  void* tmp;
  if ((rc = s.alloc((uint8_t**)&tmp, (int64_t)std::max(tmp_rows, tmp_groups)))) return rc;
  int tok;
  prof_begin(g, "cub_scan_rows", st, &tok);
  DBT_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_rows, rowoff, cell_rows + 1, st));
  prof_end(g, st, tok);
  unsigned long long n_active = 0;
  DBT_CUDA(cudaMemcpyAsync(&n_active, rowoff + cell_rows, 8, cudaMemcpyDeviceToHost, st));
  DBT_CUDA(cudaStreamSynchronize(st));
  if (n_active == 0) return DBT_OK;  // empty mesh (mesher.py:66-67)
  const int64_t A = (int64_t)n_active;
  int64_t* cell;
  uint8_t* cube;
  unsigned long long* rank;  // 5 x (A + 1)
  if ((rc = s.alloc(&cell, A)) || (rc = s.alloc(&cube, A)) || (rc = s.alloc(&rank, 5 * (A + 1)))) return rc;
  MESH_LAUNCH("mesh_active_emit", cblocks,
              (mesh_active_kernel<true><<<cblocks, 256, 0, st>>>(flags, d_tab, rg, rowoff, cell, cube)));

  const uint64_t* fw = reinterpret_cast<const uint64_t*>(flags);
  MESH_LAUNCH("mesh_group_kernel", 0,
              (mesh_group_kernel<<<blocks_for(n_groups + 1), 256, 0, st>>>(fw, n_groups, pre)));
  prof_begin(g, "cub_scan_groups", st, &tok);
  DBT_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_groups, pre, n_groups + 1, st));
  prof_end(g, st, tok);
  // per slot: rank of each active cell among those holding the slot
  thrust::counting_iterator<int64_t> idx(0);
  size_t tmp_rank = 0;
  auto it0 = thrust::make_transform_iterator(idx, SlotFlag{cube, d_tab, A, 0});
  DBT_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tmp_rank, it0, rank, A + 1, st));
  void* tmp2;
  if ((rc = s.alloc((uint8_t**)&tmp2, (int64_t)tmp_rank))) return rc;
  for (int k = 0; k < 5; ++k) {
    size_t tb = tmp_rank;
    auto it = thrust::make_transform_iterator(idx, SlotFlag{cube, d_tab, A, k});
    prof_begin(g, "cub_scan_slots", st, &tok);
    DBT_CUDA(cub::DeviceScan::ExclusiveSum(tmp2, tb, it, rank + k * (A + 1), A + 1, st));
    prof_end(g, st, tok);
  }
  unsigned long long tot[6];
  DBT_CUDA(cudaMemcpyAsync(tot, pre + n_groups, 8, cudaMemcpyDeviceToHost, st));
  DBT_CUDA(cudaMemcpy2DAsync(tot + 1, 8, rank + A, 8 * (A + 1), 8, 5, cudaMemcpyDeviceToHost, st));
  DBT_CUDA(cudaStreamSynchronize(st));
  m->nv = (int64_t)tot[0];
  int64_t base[5];
  for (int k = 0; k < 5; ++k) {
    base[k] = m->nf;
    m->nf += (int64_t)tot[1 + k];
  }
  if ((rc = pool_alloc(&m->vert, 3 * m->nv, st, "mesh output allocation")) ||
      (rc = pool_alloc(&m->tri, 3 * m->nf, st, "mesh output allocation")))
    return rc;

  VertArgs va{ny, nzp, n_words, g->vs, iso, {g->org[0], g->org[1], g->org[2]}};
  MESH_LAUNCH("mesh_vert_kernel", 0,
              (mesh_vert_kernel<<<blocks_for(n_words), 256, 0, st>>>(g->cells, fw, pre, va, m->vert)));
  MESH_LAUNCH("mesh_tri_kernel", 0,
              (mesh_tri_kernel<<<blocks_for(A), 256, 0, st>>>(cell, cube, A, rank, A + 1, d_tab, fw, pre, base[0],
                                                              base[1], base[2], base[3], base[4], m->tri)));
  DBT_CUDA(cudaStreamSynchronize(st));
  return DBT_OK;
}

}  // namespace

extern "C" {

int dbt_mesh_extract(dbt_grid* g, double iso, const dbt_mc_tables* tables, dbt_mesh** out, int64_t* n_vertices,
                     int64_t* n_triangles) {
  if (!g || !out) return set_error(DBT_ERR_CONFIG, "null grid or output handle");
  *out = nullptr;
  MeshTab h;
  int rc = check_tables(tables, &h);
  if (rc) return rc;
  if (g->xm.w != 0 || g->xm.x0 != 0 || g->xm.x1 != g->nx)
    return set_error(DBT_ERR_CONFIG, "mesh extraction needs a whole (unsharded) grid");
  rc = grid_set_device(g);
  if (!rc) rc = pool_init(g->device);
  if (!rc) rc = fold_pending(g, g->stream);
  if (rc) return rc;
  dbt_mesh* m = new dbt_mesh();
  m->device = g->device;
  rc = extract_into(g, iso, tables, h, m);
  if (rc) {
    dbt_mesh_destroy(m);
    return rc;
  }
  *out = m;
  if (n_vertices) *n_vertices = m->nv;
  if (n_triangles) *n_triangles = m->nf;
  return DBT_OK;
}

int dbt_mesh_from_host(int device, const double* vertices, int64_t n_vertices, const int64_t* triangles,
                       int64_t n_triangles, dbt_mesh** out) {
  if (!out || n_vertices < 0 || n_triangles < 0 || (n_vertices && !vertices) || (n_triangles && !triangles))
    return set_error(DBT_ERR_CONFIG, "bad mesh arrays");
  *out = nullptr;
  DBT_CUDA(cudaSetDevice(device));
  dbt_mesh* m = new dbt_mesh();
  m->device = device;
  m->nv = n_vertices;
  m->nf = n_triangles;
  int rc = pool_init(device);
  if (!rc) rc = pool_alloc(&m->vert, 3 * n_vertices, nullptr, "mesh upload");
  if (!rc) rc = pool_alloc(&m->tri, 3 * n_triangles, nullptr, "mesh upload");
  if (rc) {
    dbt_mesh_destroy(m);
    return rc;
  }
  cudaError_t e = cudaSuccess;
  if (n_vertices) e = cudaMemcpy(m->vert, vertices, (size_t)n_vertices * 24, cudaMemcpyHostToDevice);
  if (e == cudaSuccess && n_triangles)
    e = cudaMemcpy(m->tri, triangles, (size_t)n_triangles * 24, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    dbt_mesh_destroy(m);
    return cuda_error(e, "mesh upload");
  }
  *out = m;
  return DBT_OK;
}

int dbt_mesh_normals(dbt_mesh* m) {
  if (!m) return set_error(DBT_ERR_CONFIG, "null mesh handle");
  DBT_CUDA(cudaSetDevice(m->device));
  if (m->nv >= (int64_t)UINT32_MAX || 3 * m->nf >= (int64_t)UINT32_MAX)
    return set_error(DBT_ERR_RESOURCE, "mesh too large for vertex normals (2^32 corners)");
  cudaStream_t st = nullptr;
  int rc;
  if (!m->nrm && (rc = pool_alloc(&m->nrm, 3 * m->nv, st, "mesh normals allocation"))) return rc;
  if (m->nv == 0) return DBT_OK;
  const int64_t nv = m->nv, nf = m->nf, nc = 3 * nf;
  Scratch s(st);
  double* fn;
  uint32_t *key, *key2, *deg;
  int64_t *val, *val2;
  int* bad;
  if ((rc = s.alloc(&fn, 3 * nf)) || (rc = s.alloc(&key, nc)) || (rc = s.alloc(&key2, nc)) ||
      (rc = s.alloc(&val, nc)) || (rc = s.alloc(&val2, nc)) || (rc = s.alloc(&deg, nv + 1)) || (rc = s.alloc(&bad, 1)))
    return rc;
  DBT_CUDA(cudaMemsetAsync(deg, 0, (size_t)(nv + 1) * 4, st));
  DBT_CUDA(cudaMemsetAsync(bad, 0, 4, st));
  if (nf) {
    mesh_face_kernel<<<blocks_for(nf), 256, 0, st>>>(m->vert, m->tri, nv, nf, fn, key, val, deg, bad);
    DBT_CHECK_LAUNCH("mesh_face_kernel");
  }
  int end_bit = 1;
  while (end_bit < 32 && ((int64_t)1 << end_bit) < nv) ++end_bit;
  size_t t_sort = 0, t_scan = 0;
  DBT_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, t_sort, key, key2, val, val2, nc, 0, end_bit, st));
  DBT_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, t_scan, deg, nv + 1, st));
  uint8_t* tmp;
  if ((rc = s.alloc(&tmp, (int64_t)std::max(t_sort, t_scan)))) return rc;
  if (nc) DBT_CUDA(cub::DeviceRadixSort::SortPairs(tmp, t_sort, key, key2, val, val2, nc, 0, end_bit, st));
  DBT_CUDA(cub::DeviceScan::ExclusiveSum(tmp, t_scan, deg, nv + 1, st));
  mesh_normal_kernel<<<blocks_for(nv), 256, 0, st>>>(fn, val2, deg, nv, nf, m->nrm);
  DBT_CHECK_LAUNCH("mesh_normal_kernel");
  int h_bad = 0;
  DBT_CUDA(cudaMemcpyAsync(&h_bad, bad, 4, cudaMemcpyDeviceToHost, st));
  DBT_CUDA(cudaStreamSynchronize(st));
  if (h_bad) {
    cudaFreeAsync(m->nrm, st);
    m->nrm = nullptr;
    return set_error(DBT_ERR_CONFIG, "triangle index out of range");
  }
  return DBT_OK;
}

int dbt_mesh_download_normals(const dbt_mesh* m, double* normals) {
  if (!m || !m->nrm) return set_error(DBT_ERR_CONFIG, "mesh normals not computed (dbt_mesh_normals)");
  DBT_CUDA(cudaSetDevice(m->device));
  if (m->nv) DBT_CUDA(cudaMemcpy(normals, m->nrm, (size_t)m->nv * 24, cudaMemcpyDeviceToHost));
  return DBT_OK;
}

int dbt_mesh_info(const dbt_mesh* m, int64_t* n_vertices, int64_t* n_triangles) {
  if (!m) return set_error(DBT_ERR_CONFIG, "null mesh handle");
  if (n_vertices) *n_vertices = m->nv;
  if (n_triangles) *n_triangles = m->nf;
  return DBT_OK;
}

int dbt_mesh_download(const dbt_mesh* m, double* vertices, int64_t* triangles) {
  if (!m) return set_error(DBT_ERR_CONFIG, "null mesh handle");
  DBT_CUDA(cudaSetDevice(m->device));
  if (m->nv && vertices) DBT_CUDA(cudaMemcpy(vertices, m->vert, (size_t)m->nv * 24, cudaMemcpyDeviceToHost));
  if (m->nf && triangles) DBT_CUDA(cudaMemcpy(triangles, m->tri, (size_t)m->nf * 24, cudaMemcpyDeviceToHost));
  return DBT_OK;
}

int dbt_mesh_device_buffers(const dbt_mesh* m, const double** vertices, const int64_t** triangles) {
  if (!m) return set_error(DBT_ERR_CONFIG, "null mesh handle");
  if (vertices) *vertices = m->vert;
  if (triangles) *triangles = m->tri;
  return DBT_OK;
}

int dbt_mesh_destroy(dbt_mesh* m) {
  if (!m) return DBT_OK;
  cudaSetDevice(m->device);
  // the legacy stream orders the release after any work on blocking streams;
  // extract/normals synchronise before returning
  if (m->vert) cudaFreeAsync(m->vert, nullptr);
  if (m->tri) cudaFreeAsync(m->tri, nullptr);
  if (m->nrm) cudaFreeAsync(m->nrm, nullptr);
  delete m;
  return DBT_OK;
}

}  // extern "C"
