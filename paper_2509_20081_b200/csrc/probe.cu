// probe.cu — microbenchmarks for the roofline denominators SURVEY.md §8(d)
// asks for besides the HBM copy peak: the L2 atomic (RED.AND) throughput on
// 4-byte words of an L2-resident buffer -- the roof of an L2-resident
// integration launch -- and the L2-resident 8-byte load bandwidth (the
// distance-cache sweep reads). Timed with CUDA events, best of several runs.
#include "engine.cuh"

using namespace dbt;

namespace {

// every warp ANDs 32 consecutive words (one 128-byte line) per step; the
// grid walks the buffer so every word is hit `rounds` times
__global__ void l2_red_kernel(uint32_t* __restrict__ buf, int64_t nwords, int rounds) {
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  for (int r = 0; r < rounds; ++r)
    for (int64_t i = t; i < nwords; i += nthr) atomicAnd(buf + i, ~(1u << ((r + (int)i) & 31)));
}

__global__ void l2_load_kernel(const uint2* __restrict__ buf, int64_t n, int rounds, uint32_t* __restrict__ sink) {
  const int64_t nthr = (int64_t)gridDim.x * blockDim.x;
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  uint32_t acc = 0;
  for (int r = 0; r < rounds; ++r)
    for (int64_t i = t; i < n; i += nthr) {
      const uint2 v = __ldcg(buf + i);
      acc ^= v.x + v.y;
    }
  if (acc == 0x9E3779B9u) *sink = acc;  // keeps the loads
}

}  // namespace

extern "C" {

int dbt_probe_l2(int device, int64_t bytes, double* out) {
  // out[0] = RED.AND Gop/s, out[1] = RED.AND GB/s (4 B per op),
  // out[2] = ld.cg 8-byte GB/s, all on an L2-resident buffer of `bytes`
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) return cuda_error(e, "cudaSetDevice");
  if (bytes < (1 << 20)) return set_error(DBT_ERR_CONFIG, "probe buffer below 1 MiB");
  void* buf = nullptr;
  uint32_t* sink = nullptr;
  DBT_CUDA(cudaMalloc(&buf, bytes));
  DBT_CUDA(cudaMalloc(&sink, 4));
  DBT_CUDA(cudaMemset(buf, 0xFF, bytes));
  int sms = 0;
  DBT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device));
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int rounds = 8;
  const int64_t nw = bytes / 4, n8 = bytes / 8;
  float best_red = 1e30f, best_ld = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    cudaEventRecord(a);
    l2_red_kernel<<<sms * 8, 256>>>((uint32_t*)buf, nw, rounds);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    if (rep) best_red = std::min(best_red, ms);  // first run warms L2
    cudaEventRecord(a);
    l2_load_kernel<<<sms * 8, 256>>>((const uint2*)buf, n8, rounds, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (rep) best_ld = std::min(best_ld, ms);
  }
  cudaError_t le = cudaGetLastError();
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(buf);
  cudaFree(sink);
  if (le != cudaSuccess) return cuda_error(le, "l2 probe kernels");
  const double ops = (double)nw * rounds;
  out[0] = ops / (best_red * 1e-3) / 1e9;
  out[1] = out[0] * 4.0;
  out[2] = (double)n8 * 8.0 * rounds / (best_ld * 1e-3) / 1e9;
  return DBT_OK;
}

}  // extern "C"
