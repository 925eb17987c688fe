// runtime.cpp — device memory caching allocator and per-kernel event profiler.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <unordered_map>
#include <vector>

#include "common.cuh"

namespace groot {

// ---------------------------------------------------------------------------
// Caching allocator. All library work is ordered on one stream, so a block
// freed by the host can be handed to the next allocation immediately: any
// kernel still reading it precedes, in stream order, every kernel that will
// write it.
// ---------------------------------------------------------------------------
namespace {
std::mutex g_mem_mu;
std::multimap<size_t, void*> g_free;             // size -> block
std::unordered_map<void*, size_t> g_live;         // block -> size
size_t g_cached_bytes = 0;

size_t round_size(size_t b) {
  if (b <= (1u << 20)) return (b + 511) & ~size_t(511);
  return (b + (2u << 20) - 1) & ~size_t((2u << 20) - 1);
}

void release_all_free() {
  for (auto& kv : g_free) cudaFree(kv.second);
  g_free.clear();
  g_cached_bytes = 0;
}
}  // namespace

void* dev_alloc(size_t bytes) {
  const size_t sz = round_size(bytes);
  std::lock_guard<std::mutex> lk(g_mem_mu);
  // best fit among cached blocks no more than 25% (+2 MB) larger than needed
  auto it = g_free.lower_bound(sz);
  if (it != g_free.end() && it->first <= sz + sz / 4 + (2u << 20)) {
    void* p = it->second;
    const size_t have = it->first;
    g_free.erase(it);
    g_cached_bytes -= have;
    g_live[p] = have;
    return p;
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, sz);
  if (e != cudaSuccess) {
    cudaGetLastError();
    cudaDeviceSynchronize();
    release_all_free();
    e = cudaMalloc(&p, sz);
    if (e != cudaSuccess) {
      cudaGetLastError();
      fail(GROOT_ECUDA, "device allocation of " + std::to_string(sz) + " bytes failed: " + cudaGetErrorString(e));
    }
  }
  g_live[p] = sz;
  return p;
}

void dev_free(void* p) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_mem_mu);
  auto it = g_live.find(p);
  if (it == g_live.end()) return;
  g_free.emplace(it->second, p);
  g_cached_bytes += it->second;
  g_live.erase(it);
}

void dev_empty_cache() {
  std::lock_guard<std::mutex> lk(g_mem_mu);
  cudaDeviceSynchronize();
  release_all_free();
}

// ---------------------------------------------------------------------------
// Profiler: CUDA events recorded on the library stream around named launches.
// ---------------------------------------------------------------------------
namespace {
struct Rec {
  const char* name;
  cudaEvent_t a, b;
};
std::mutex g_prof_mu;
bool g_prof_on = false;
std::vector<Rec> g_recs;
std::vector<cudaEvent_t> g_pool;
struct Agg {
  double ms = 0;
  uint64_t n = 0;
};
std::map<std::string, Agg> g_agg;

cudaEvent_t take_event() {
  if (!g_pool.empty()) {
    cudaEvent_t e = g_pool.back();
    g_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  GROOT_CUDA(cudaEventCreate(&e));
  return e;
}

void drain() {  // caller holds g_prof_mu
  if (g_recs.empty()) return;
  GROOT_CUDA(cudaStreamSynchronize(stream()));
  for (Rec& r : g_recs) {
    float ms = 0.f;
    GROOT_CUDA(cudaEventElapsedTime(&ms, r.a, r.b));
    Agg& a = g_agg[r.name];
    a.ms += ms;
    a.n += 1;
    g_pool.push_back(r.a);
    g_pool.push_back(r.b);
  }
  g_recs.clear();
}
}  // namespace

ProfScope::ProfScope(const char* name) {
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (!g_prof_on) return;
  if (g_recs.size() > 4096) drain();
  Rec r{name, take_event(), take_event()};
  GROOT_CUDA(cudaEventRecord(r.a, stream()));
  g_recs.push_back(r);
  slot = static_cast<int>(g_recs.size()) - 1;
}

ProfScope::~ProfScope() {
  if (slot < 0) return;
  std::lock_guard<std::mutex> lk(g_prof_mu);
  if (slot < static_cast<int>(g_recs.size())) cudaEventRecord(g_recs[slot].b, stream());
}

}  // namespace groot

using namespace groot;

extern "C" {

int groot_profile_enable(int on) {
  return guarded([&] {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    drain();
    g_agg.clear();
    g_prof_on = on != 0;
  });
}

// Per-kernel totals since enable: names (max entries x 48 chars, NUL padded),
// total milliseconds and launch counts. *count receives the number of kernels.
int groot_profile_read(uint32_t max, char* names, double* total_ms, uint64_t* launches, uint32_t* count) {
  return guarded([&] {
    std::lock_guard<std::mutex> lk(g_prof_mu);
    drain();
    uint32_t i = 0;
    for (auto& kv : g_agg) {
      if (i < max) {
        if (names) {
          std::memset(names + 48 * i, 0, 48);
          std::strncpy(names + 48 * i, kv.first.c_str(), 47);
        }
        if (total_ms) total_ms[i] = kv.second.ms;
        if (launches) launches[i] = kv.second.n;
      }
      ++i;
    }
    if (count) *count = i;
  });
}

int groot_empty_cache(void) {
  return guarded([] { dev_empty_cache(); });
}

}  // extern "C"
