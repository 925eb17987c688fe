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
// Caching allocator, one pool per device. All library work on a device is
// ordered on that device's library stream, so a block freed by the host can
// be handed to the next allocation immediately: any kernel still reading it
// precedes, in stream order, every kernel that will write it.
// ---------------------------------------------------------------------------
namespace {
std::mutex g_mem_mu;
// Per device: cached blocks by size, and the size of every live block.
struct DevPool {
  std::multimap<size_t, void*> free_blocks;
  std::unordered_map<void*, size_t> live;
  size_t cached_bytes = 0;
};
DevPool g_pools[kMaxDevices];

size_t round_size(size_t b) {
  if (b <= (1u << 20)) return (b + 511) & ~size_t(511);
  return (b + (2u << 20) - 1) & ~size_t((2u << 20) - 1);
}

void release_all_free(DevPool& pool) {  // the pool's device is current
  for (auto& kv : pool.free_blocks) cudaFree(kv.second);
  pool.free_blocks.clear();
  pool.cached_bytes = 0;
}
}  // namespace

void* dev_alloc(size_t bytes) {
  const size_t sz = round_size(bytes);
  DevPool& pool = g_pools[current_device()];
  std::lock_guard<std::mutex> lk(g_mem_mu);
  // best fit among cached blocks no more than 25% (+2 MB) larger than needed
  auto it = pool.free_blocks.lower_bound(sz);
  if (it != pool.free_blocks.end() && it->first <= sz + sz / 4 + (2u << 20)) {
    void* p = it->second;
    const size_t have = it->first;
    pool.free_blocks.erase(it);
    pool.cached_bytes -= have;
    pool.live[p] = have;
    return p;
  }
  void* p = nullptr;
  cudaError_t e = cudaMalloc(&p, sz);
  if (e != cudaSuccess) {
    cudaGetLastError();
    cudaDeviceSynchronize();
    release_all_free(pool);
    e = cudaMalloc(&p, sz);
    if (e != cudaSuccess) {
      cudaGetLastError();
      fail(GROOT_ECUDA, "device allocation of " + std::to_string(sz) + " bytes failed: " + cudaGetErrorString(e));
    }
  }
  pool.live[p] = sz;
  return p;
}

void dev_free(void* p) {
  if (!p) return;
  std::lock_guard<std::mutex> lk(g_mem_mu);
  for (DevPool& pool : g_pools) {  // the block's owner (free may run with another device current)
    auto it = pool.live.find(p);
    if (it == pool.live.end()) continue;
    pool.free_blocks.emplace(it->second, p);
    pool.cached_bytes += it->second;
    pool.live.erase(it);
    return;
  }
}

void dev_empty_cache() {
  std::lock_guard<std::mutex> lk(g_mem_mu);
  int cur = 0;
  cudaGetDevice(&cur);
  for (int d = 0; d < kMaxDevices; ++d) {
    if (g_pools[d].free_blocks.empty()) continue;
    cudaSetDevice(d);
    cudaDeviceSynchronize();
    release_all_free(g_pools[d]);
  }
  cudaSetDevice(cur);
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
