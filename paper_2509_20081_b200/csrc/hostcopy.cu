// hostcopy.cu — multi-threaded host copy of pageable scans into the grid's
// pinned staging buffer.
//
// A stock caller (cli.run_fuse, the reference's own tests) passes pageable
// numpy arrays. cudaMemcpyAsync from pageable memory goes through the
// driver's single-threaded bounce buffer (~11 GB/s measured on the B200 box);
// copying into pinned, device-mapped staging with several host threads and
// letting the prep kernel read it over the host link (as for pinned scans)
// moves the same bytes in a fraction of that time. A small persistent pool:
// workers sleep on a condition variable between calls; one job at a time.
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstring>
#include <mutex>
#include <thread>
#include <vector>

#include "engine.cuh"

namespace dbt {
namespace {

class CopyPool {
 public:
  explicit CopyPool(int n) {
    for (int i = 0; i < n; ++i) workers_.emplace_back([this, i] { run(i + 1); });
  }
  ~CopyPool() {
    {
      std::lock_guard<std::mutex> l(mu_);
      stop_ = true;
      ++gen_;
    }
    cv_.notify_all();
    for (auto& t : workers_) t.join();
  }
  int size() const { return (int)workers_.size() + 1; }

  void copy(char* dst, const char* src, size_t bytes, int parts) {
    std::lock_guard<std::mutex> job(job_mu_);  // one job at a time
    parts = std::max(1, std::min(parts, size()));
    {
      std::lock_guard<std::mutex> l(mu_);
      dst_ = dst;
      src_ = src;
      bytes_ = bytes;
      parts_ = parts;
      done_.store(0, std::memory_order_relaxed);
      ++gen_;
    }
    cv_.notify_all();
    chunk(0);  // the caller copies part 0
    while (done_.load(std::memory_order_acquire) < parts - 1) std::this_thread::yield();
  }

 private:
  void chunk(int k) {
    const size_t per = (bytes_ / parts_ + 63) & ~size_t(63);
    const size_t a = std::min(bytes_, per * (size_t)k), b = std::min(bytes_, a + per);
    if (b > a) std::memcpy(dst_ + a, src_ + a, b - a);
  }
  void run(int id) {
    uint64_t seen = 0;
    while (true) {
      std::unique_lock<std::mutex> l(mu_);
      cv_.wait(l, [&] { return gen_ != seen; });
      seen = gen_;
      if (stop_) return;
      const bool mine = id < parts_;
      l.unlock();
      if (mine) {
        chunk(id);
        done_.fetch_add(1, std::memory_order_release);
      }
    }
  }

  std::vector<std::thread> workers_;
  std::mutex mu_, job_mu_;
  std::condition_variable cv_;
  uint64_t gen_ = 0;
  bool stop_ = false;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t bytes_ = 0;
  int parts_ = 1;
  std::atomic<int> done_{0};
};

CopyPool& pool() {
  static CopyPool p([] {
    const char* e = getenv("DBT_COPY_THREADS");
    int n = e ? atoi(e) : (int)std::min(8u, std::max(1u, std::thread::hardware_concurrency() / 2));
    return std::max(0, n - 1);
  }());
  return p;
}

}  // namespace

// Copy n pageable host buffers (srcs[i], bytes[i]) back to back into the
// grid's pinned, mapped staging (grown on demand); out[i] = device pointer of
// buffer i. Returns false (nothing staged) when staging is unavailable or
// the scans are small, and the caller falls back to cudaMemcpyAsync.
bool stage_pageable(dbt_grid* g, const void* const* srcs, const int64_t* bytes, int n, const void** out) {
  int64_t total = 0;
  for (int i = 0; i < n; ++i) total += (bytes[i] + 63) & ~int64_t(63);
  if (total < (64 << 10) || getenv("DBT_NO_HOST_STAGE")) return false;
  if (total > g->cap_hstage) {
    const int64_t cap = std::max<int64_t>(total, g->cap_hstage + g->cap_hstage / 2);
    if (g->h_stage) cudaFreeHost(g->h_stage);
    g->h_stage = nullptr;
    g->cap_hstage = 0;
    if (cudaHostAlloc(&g->h_stage, (size_t)cap, cudaHostAllocMapped | cudaHostAllocPortable) != cudaSuccess) {
      cudaGetLastError();
      g->h_stage = nullptr;
      return false;
    }
    g->cap_hstage = cap;
  }
  char* d = nullptr;
  if (cudaHostGetDevicePointer((void**)&d, g->h_stage, 0) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  // the previous synchronous call has completed (it waited for its
  // stream), so nothing on the device still reads the staging buffer
  int64_t off = 0;
  for (int i = 0; i < n; ++i) {
    const int parts = (int)std::min<int64_t>(pool().size(), std::max<int64_t>(1, bytes[i] / (128 << 10)));
    if (bytes[i]) pool().copy((char*)g->h_stage + off, (const char*)srcs[i], (size_t)bytes[i], parts);
    out[i] = d + off;
    off += (bytes[i] + 63) & ~int64_t(63);
  }
  return true;
}

// The same pooled copy into any host buffer (the asynchronous call's per-slot
// pinned staging).
void pooled_host_copy(void* dst, const void* src, size_t bytes) {
  const int parts = (int)std::min<int64_t>(pool().size(), std::max<int64_t>(1, (int64_t)bytes / (128 << 10)));
  if (bytes) pool().copy((char*)dst, (const char*)src, bytes, parts);
}

}  // namespace dbt
