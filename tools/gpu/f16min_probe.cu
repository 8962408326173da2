// Probe: red.global.min.noftz.v4.f16x2 on 16-bit integers 0..64 stored as raw
// f16 bit patterns (subnormals): does the hardware min equal the integer min?
#include <cstdio>
#include <cstdint>
#include <vector>
__global__ void k(uint16_t* p, const uint16_t* v, int n8) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n8) return;
  const uint4 w = reinterpret_cast<const uint4*>(v)[i];
  asm volatile("red.global.min.noftz.v4.f16x2 [%0], {%1,%2,%3,%4};" ::"l"(p + 8 * i), "r"(w.x), "r"(w.y), "r"(w.z),
               "r"(w.w) : "memory");
}
int main() {
  const int n = 65 * 65 * 8;
  std::vector<uint16_t> a(n), b(n), r(n);
  for (int i = 0; i < n; ++i) { a[i] = (i / 8) / 65; b[i] = (i / 8) % 65; }
  uint16_t *da, *db;
  cudaMalloc(&da, n * 2); cudaMalloc(&db, n * 2);
  cudaMemcpy(da, a.data(), n * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), n * 2, cudaMemcpyHostToDevice);
  k<<<(n / 8 + 255) / 256, 256>>>(da, db, n / 8);
  cudaMemcpy(r.data(), da, n * 2, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < n; ++i) bad += r[i] != (a[i] < b[i] ? a[i] : b[i]);
  printf("f16x8 min on raw ints 0..64: %d mismatches of %d (%s)\n", bad, n, cudaGetErrorString(cudaGetLastError()));
  return bad != 0;
}
