// abi.cu — error plumbing, measurement hooks and small C-ABI utilities.
//
// Error codes follow the reference's exception -> exit-code mapping
// (cli.py:34-40; errors.py:7-29).
#include <atomic>
#include <cstring>
#include <string>

#include "engine.cuh"

namespace dbt {

static thread_local std::string g_last_error;
static std::atomic<int64_t> g_launches{0};

int set_error(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

int cuda_error(cudaError_t e, const char* what) {
  std::string msg = std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")";
  // an allocation failure is the device analogue of the reference's memory cap
  // (grid.py:77-81 -> ResourceError)
  int code = (e == cudaErrorMemoryAllocation) ? DBT_ERR_RESOURCE : DBT_ERR_GENERIC;
  return set_error(code, msg);
}

void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
void add_launches(int64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

static int prof_index(dbt_grid* g, const char* name) {
  for (size_t i = 0; i < g->prof_names.size(); ++i)
    if (g->prof_names[i] == name) return (int)i;
  g->prof_names.emplace_back(name);
  g->prof_ms.push_back(0.0);
  g->prof_launches.push_back(0);
  return (int)g->prof_names.size() - 1;
}

static cudaEvent_t pool_get(dbt_grid* g) {
  if (!g->event_pool.empty()) {
    cudaEvent_t e = g->event_pool.back();
    g->event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}

void prof_begin(dbt_grid* g, const char* name, cudaStream_t s, int* token) {
  *token = -1;
  if (!g->profiling) return;
  if (g->pending.size() > 65536) prof_flush(g);
  ProfEvent pe;
  pe.a = pool_get(g);
  pe.b = pool_get(g);
  pe.kernel = prof_index(g, name);
  cudaEventRecord(pe.a, s);
  g->pending.push_back(pe);
  *token = (int)g->pending.size() - 1;
}

void prof_end(dbt_grid* g, cudaStream_t s, int token) {
  if (token < 0) return;
  cudaEventRecord(g->pending[token].b, s);
}

int prof_flush(dbt_grid* g) {
  for (auto& pe : g->pending) {
    cudaEventSynchronize(pe.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, pe.a, pe.b);
    g->prof_ms[pe.kernel] += ms;
    g->prof_launches[pe.kernel] += 1;
    g->event_pool.push_back(pe.a);
    g->event_pool.push_back(pe.b);
  }
  g->pending.clear();
  return DBT_OK;
}

}  // namespace dbt

extern "C" {

const char* dbt_last_error(void) { return dbt::g_last_error.c_str(); }

const char* dbt_version(void) { return "dbtsdf-b200 0.1.0 (sm_100a)"; }

int dbt_device_count(int* out) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    *out = 0;
    return dbt::cuda_error(e, "cudaGetDeviceCount");
  }
  *out = n;
  return DBT_OK;
}

int64_t dbt_launch_count(void) { return dbt::g_launches.load(); }

int dbt_profile_enable(dbt_grid* g, int on) {
  if (!g) return dbt::set_error(DBT_ERR_CONFIG, "null grid");
  g->profiling = on != 0;
  return DBT_OK;
}

int dbt_profile_reset(dbt_grid* g) {
  if (!g) return dbt::set_error(DBT_ERR_CONFIG, "null grid");
  dbt::prof_flush(g);
  for (auto& v : g->prof_ms) v = 0.0;
  for (auto& v : g->prof_launches) v = 0;
  return DBT_OK;
}

int dbt_profile_read(dbt_grid* g, char* names, double* ms, int64_t* launches, int32_t cap,
                     int32_t* n) {
  if (!g) return dbt::set_error(DBT_ERR_CONFIG, "null grid");
  dbt::prof_flush(g);
  int32_t k = (int32_t)g->prof_names.size();
  *n = k;
  for (int32_t i = 0; i < k && i < cap; ++i) {
    std::strncpy(names + 32 * i, g->prof_names[i].c_str(), 31);
    names[32 * i + 31] = 0;
    ms[i] = g->prof_ms[i];
    launches[i] = g->prof_launches[i];
  }
  return DBT_OK;
}

int dbt_host_alloc(int64_t bytes, void** out) {
  DBT_CUDA(cudaHostAlloc(out, (size_t)bytes, cudaHostAllocDefault));
  return DBT_OK;
}

int dbt_host_free(void* p) {
  DBT_CUDA(cudaFreeHost(p));
  return DBT_OK;
}

}  // extern "C"
