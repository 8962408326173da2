// bank.cu — device copy of the KernelBank (reference kernels.py:122-193).
//
// The bank is built on the host exactly as the reference builds it (one
// shared K^3 distance kernel + one shadow offset list per azimuth-elevation
// bin) and staged here once. Two device tables are derived:
//  * the sweep table: for each of the 8 possible z-alignments of a centre,
//    each DISTINCT kernel z-row (identical rows are shared; 66 of the 441
//    rows of the standard 21^3 kernel are distinct) and each 8-voxel chunk of
//    that row, the 8 run lengths + 1 packed into a uint2 (64 marks a voxel
//    outside the kernel, which can never lower a distance <= 32), plus the
//    row -> distinct-row map;
//  * whether the kernel is isotropic (run length a non-decreasing function
//    of |o|^2), which licenses the culling sweep;
//  * the shadow table in CSR form, offsets as int8 (|o| <= R <= 15).
#include <algorithm>
#include <cstring>
#include <vector>

#include "engine.cuh"

using namespace dbt;

static uint64_t g_bank_serial = 0;

extern "C" {

int dbt_bank_create(int32_t size, int32_t b_az, int32_t b_el, const uint32_t* distance_kernel,
                    const int32_t* shadow_xyz, const int32_t* shadow_counts, int device,
                    dbt_bank** out) {
  *out = nullptr;
  if (size < 1 || size % 2 == 0)
    return set_error(DBT_ERR_CONFIG, "kernel size must be odd and positive (kernels.py:160-161)");
  if (size > kMaxK) return set_error(DBT_ERR_CONFIG, "kernel size above 31 is not supported on device");
  if (b_az < 1 || b_el < 1) return set_error(DBT_ERR_CONFIG, "bin counts must be at least 1");
  if ((int64_t)b_az * b_el > 65535) return set_error(DBT_ERR_CONFIG, "more than 65535 direction bins");
  const int K = size, R = size / 2, K3 = K * K * K, rows = K * K;
  const int CH = (K + 7 + 7) / 8;
  std::vector<uint8_t> len(K3);
  int max_d = 0;
  for (int i = 0; i < K3; ++i) {
    uint32_t m = distance_kernel[i];
    int pc = __builtin_popcount(m);
    int clz = m ? __builtin_clz(m) : 32;
    if (pc + clz != 32)
      return set_error(DBT_ERR_CORRUPTION, "distance kernel entry is not a low-bit run mask");
    len[i] = (uint8_t)pc;
    max_d = std::max(max_d, pc);
  }
  // distinct kernel rows (the standard kernel depends on (|dx|,|dy|) and is
  // symmetric in dx<->dy: 66 distinct rows of 441)
  std::vector<int> rowid(rows);
  std::vector<int> distinct;  // representative row of each distinct id
  for (int r = 0; r < rows; ++r) {
    int id = -1;
    for (size_t q = 0; q < distinct.size() && id < 0; ++q)
      if (std::memcmp(&len[(size_t)distinct[q] * K], &len[(size_t)r * K], K) == 0) id = (int)q;
    if (id < 0) {
      id = (int)distinct.size();
      distinct.push_back(r);
    }
    rowid[r] = id;
  }
  const int nd = (int)distinct.size();
  std::vector<uint2> dtab((size_t)8 * nd * CH);
  for (int s = 0; s < 8; ++s)
    for (int q = 0; q < nd; ++q)
      for (int c = 0; c < CH; ++c) {
        uint32_t v[2] = {0, 0};
        for (int i = 0; i < 8; ++i) {
          int zk = 8 * c + i - s;
          // d + 1, 64 outside the kernel (see the sweep's byte test)
          uint32_t d = (zk >= 0 && zk < K) ? len[(size_t)distinct[q] * K + zk] + 1u : 64u;
          v[i >> 2] |= d << (8 * (i & 3));
        }
        dtab[((size_t)s * nd + q) * CH + c] = make_uint2(v[0], v[1]);
      }
  // isotropic kernel: run length = h(|o|^2) with h non-decreasing (the
  // culling sweep's premise; every bank build_kernel_bank makes)
  bool iso = CH <= 4;
  {
    std::vector<int> h(3 * R * R + 1, -1);
    for (int dx = -R; dx <= R && iso; ++dx)
      for (int dy = -R; dy <= R && iso; ++dy)
        for (int dz = -R; dz <= R && iso; ++dz) {
          const int q = dx * dx + dy * dy + dz * dz;
          const int l = len[((size_t)(dx + R) * K + (dy + R)) * K + (dz + R)];
          if (h[q] < 0) h[q] = l;
          else if (h[q] != l) iso = false;
        }
    int prev = -1;
    for (size_t q = 0; q < h.size() && iso; ++q)
      if (h[q] >= 0) {
        if (h[q] < prev) iso = false;
        prev = h[q];
      }
  }
  std::vector<uint16_t> rowd(rows);
  for (int r = 0; r < rows; ++r) rowd[r] = (uint16_t)(rowid[r] * CH);
  const int nb = b_az * b_el;
  std::vector<int32_t> start(nb + 1, 0);
  int max_s = 0;
  for (int b = 0; b < nb; ++b) {
    if (shadow_counts[b] < 0) return set_error(DBT_ERR_CONFIG, "negative shadow count");
    start[b + 1] = start[b] + shadow_counts[b];
    max_s = std::max(max_s, (int)shadow_counts[b]);
  }
  const int64_t total = start[nb];
  std::vector<int8_t> sx((size_t)std::max<int64_t>(total, 1) * 4, 0);
  for (int64_t i = 0; i < total; ++i)
    for (int k = 0; k < 3; ++k) {
      int32_t v = shadow_xyz[3 * i + k];
      if (v < -R || v > R) return set_error(DBT_ERR_CONFIG, "shadow offset outside the kernel cube");
      sx[4 * i + k] = (int8_t)v;
    }

  dbt_bank* b = new dbt_bank();
  b->device = device;
  b->K = K;
  b->R = R;
  b->b_az = b_az;
  b->b_el = b_el;
  b->n_bins = nb;
  b->max_shadow = max_s;
  b->total_shadow = total;
  b->chunks_per_row = CH;
  b->max_d = max_d;
  b->n_distinct = nd;
  b->iso = iso ? 1 : 0;
  uint64_t hsh = 1469598103934665603ull ^ (uint64_t)K;
  for (int i = 0; i < K3; ++i) hsh = (hsh ^ len[i]) * 1099511628211ull;
  b->dk_hash = hsh | 1;
  b->serial = ++g_bank_serial;
  cudaError_t e = cudaSetDevice(device);
  if (e == cudaSuccess) e = cudaMalloc(&b->d_len, K3);
  if (e == cudaSuccess) e = cudaMalloc(&b->d_dtab, dtab.size() * sizeof(uint2));
  if (e == cudaSuccess) e = cudaMalloc(&b->d_rowd, rows * sizeof(uint16_t));
  if (e == cudaSuccess) e = cudaMemcpy(b->d_rowd, rowd.data(), rows * sizeof(uint16_t), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMalloc(&b->d_shadow_xyz, sx.size());
  if (e == cudaSuccess) e = cudaMalloc(&b->d_shadow_start, (nb + 1) * 4);
  if (e == cudaSuccess) e = cudaMemcpy(b->d_len, len.data(), K3, cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(b->d_dtab, dtab.data(), dtab.size() * sizeof(uint2), cudaMemcpyHostToDevice);
  if (e == cudaSuccess) e = cudaMemcpy(b->d_shadow_xyz, sx.data(), sx.size(), cudaMemcpyHostToDevice);
  if (e == cudaSuccess)
    e = cudaMemcpy(b->d_shadow_start, start.data(), (nb + 1) * 4, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) {
    int code = cuda_error(e, "kernel bank staging");
    dbt_bank_destroy(b);
    return code;
  }
  *out = b;
  return DBT_OK;
}

int dbt_bank_destroy(dbt_bank* b) {
  if (!b) return DBT_OK;
  cudaSetDevice(b->device);
  if (b->d_len) cudaFree(b->d_len);
  if (b->d_dtab) cudaFree(b->d_dtab);
  if (b->d_rowd) cudaFree(b->d_rowd);
  if (b->d_shadow_xyz) cudaFree(b->d_shadow_xyz);
  if (b->d_shadow_start) cudaFree(b->d_shadow_start);
  delete b;
  return DBT_OK;
}

}  // extern "C"
