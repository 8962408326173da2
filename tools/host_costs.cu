// Host-side cost of the CUDA runtime calls on the synchronous integrate path
// (B200 box): average CPU time per call over 2000 calls, idle device.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 tools/host_costs.cu -o gpurun_out/host_costs
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_empty(int* p, int n) {
  if (threadIdx.x == 0 && blockIdx.x == 0 && n < 0) p[0] = 1;
}

static double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
  cudaSetDevice(0);
  cudaStream_t st, aux;
  cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&aux, cudaStreamNonBlocking);
  cudaEvent_t ea, eb, ef;
  cudaEventCreate(&ea);
  cudaEventCreate(&eb);
  cudaEventCreateWithFlags(&ef, cudaEventDisableTiming);
  int* d;
  cudaMalloc(&d, 1 << 20);
  void* h;
  cudaHostAlloc(&h, 1 << 20, cudaHostAllocMapped | cudaHostAllocPortable);
  void* hp = malloc(1 << 20);
  const int N = 2000;
  double t;
  cudaPointerAttributes at;
#define TIME(label, ...)                                    \
  cudaDeviceSynchronize();                                   \
  t = now_us();                                              \
  for (int i = 0; i < N; ++i) { __VA_ARGS__; }                    \
  printf("%-44s %.2f us\n", label, (now_us() - t) / N);      \
  cudaDeviceSynchronize();
  TIME("cudaPointerGetAttributes (pinned)", cudaPointerGetAttributes(&at, h));
  TIME("cudaPointerGetAttributes (pageable)", { cudaPointerGetAttributes(&at, hp); cudaGetLastError(); });
  TIME("cudaSetDevice", cudaSetDevice(0));
  TIME("cudaEventRecord", cudaEventRecord(ea, st));
  TIME("cudaMemsetAsync 64 B", cudaMemsetAsync(d, 0, 64, st));
  TIME("kernel launch <<<256,256>>>", k_empty<<<256, 256, 0, st>>>(d, 1));
  TIME("cudaStreamWaitEvent", cudaStreamWaitEvent(aux, ef, 0));
  TIME("cudaMemcpyAsync D2H 64 B (pinned dst)", cudaMemcpyAsync(h, d, 64, cudaMemcpyDeviceToHost, st));
  TIME("cudaGetLastError", cudaGetLastError());
  // a whole synchronous sequence like dbt_integrate_frame's, empty kernels
  TIME("sequence: rec,memset,k,rec,wait,k(aux),rec,k,wait,d2h,rec,spin", {
    cudaEventRecord(ea, st);
    cudaMemsetAsync(d, 0, 64, st);
    k_empty<<<256, 256, 0, st>>>(d, 1);
    cudaEventRecord(ef, st);
    cudaStreamWaitEvent(aux, ef, 0);
    k_empty<<<1024, 256, 0, aux>>>(d, 1);
    cudaEventRecord(ef, aux);
    k_empty<<<1036, 128, 0, st>>>(d, 1);
    cudaStreamWaitEvent(st, ef, 0);
    cudaMemcpyAsync(h, d, 64, cudaMemcpyDeviceToHost, st);
    cudaEventRecord(eb, st);
    while (cudaEventQuery(eb) == cudaErrorNotReady) {
    }
  });
  float ms;
  TIME("cudaEventElapsedTime", cudaEventElapsedTime(&ms, ea, eb));
  // graph of the same sequence
  cudaGraph_t gr;
  cudaGraphExec_t ge;
  cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal);
  cudaMemsetAsync(d, 0, 64, st);
  k_empty<<<256, 256, 0, st>>>(d, 1);
  cudaEventRecord(ef, st);
  cudaStreamWaitEvent(aux, ef, 0);
  k_empty<<<1024, 256, 0, aux>>>(d, 1);
  cudaEventRecord(ef, aux);
  k_empty<<<1036, 128, 0, st>>>(d, 1);
  cudaStreamWaitEvent(st, ef, 0);
  cudaMemcpyAsync(h, d, 64, cudaMemcpyDeviceToHost, st);
  cudaStreamEndCapture(st, &gr);
  cudaGraphInstantiate(&ge, gr, 0);
  TIME("graph launch + rec + spin", {
    cudaGraphLaunch(ge, st);
    cudaEventRecord(eb, st);
    while (cudaEventQuery(eb) == cudaErrorNotReady) {
    }
  });
  TIME("graph launch only", cudaGraphLaunch(ge, st));
  return 0;
}
