// common.cuh — shared host/device plumbing for libgroot_b200 (sm_100a only).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <atomic>
#include <stdexcept>
#include <string>
#include <vector>

#include "groot.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ != 1000)
#error "libgroot_b200 is built for sm_100a only (-gencode arch=compute_100a,code=sm_100a)"
#endif

namespace groot {

// Error carried to the C ABI: code is one of GROOT_E*.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }
inline void require(bool ok, const char* msg) {
  if (!ok) fail(GROOT_EINVAL, msg);
}

#define GROOT_CUDA(expr)                                                                       \
  do {                                                                                         \
    cudaError_t _e = (expr);                                                                   \
    if (_e != cudaSuccess)                                                                     \
      ::groot::fail(GROOT_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e));          \
  } while (0)

extern std::atomic<uint64_t> g_launches;
constexpr int kMaxDevices = 64;
int current_device();
// The library stream of the calling thread's current device (groot_set_stream).
cudaStream_t stream();
// A second (copy) stream of the current device (forward.cu).
cudaStream_t side_stream();
// Timing-free CUDA event owned by a scope.
struct Event {
  cudaEvent_t e = nullptr;
  Event() { GROOT_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming)); }
  ~Event() {
    if (e) cudaEventDestroy(e);
  }
  Event(const Event&) = delete;
  Event& operator=(const Event&) = delete;
};

// Makes `dev` the current device for a scope (restored on exit): entry points
// taking a handle run on the device that owns it.
struct DeviceScope {
  int prev = -1;
  explicit DeviceScope(int dev) {
    int cur = 0;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != dev && cudaSetDevice(dev) == cudaSuccess) prev = cur;
  }
  ~DeviceScope() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceScope(const DeviceScope&) = delete;
  DeviceScope& operator=(const DeviceScope&) = delete;
};

// Launch helper: counts launches (bench evidence) and checks the launch.
#define GROOT_LAUNCH(kernel, grid, block, smem, ...)                                           \
  do {                                                                                         \
    kernel<<<(grid), (block), (smem), ::groot::stream()>>>(__VA_ARGS__);                      \
    ::groot::g_launches.fetch_add(1, std::memory_order_relaxed);                               \
    GROOT_CUDA(cudaGetLastError());                                                            \
  } while (0)

inline void stream_sync() { GROOT_CUDA(cudaStreamSynchronize(stream())); }

// Thread-local message returned by groot_last_error().
void set_last_error(const std::string& msg);

// Runs f, mapping exceptions to GROOT_* status codes for the C ABI.
template <class F>
int guarded(F&& f) {
  try {
    f();
    return GROOT_OK;
  } catch (const Error& e) {
    set_last_error(e.what());
    return e.code;
  } catch (const std::bad_alloc&) {
    set_last_error("out of host memory");
    return GROOT_ERUNTIME;
  } catch (const std::exception& e) {
    set_last_error(e.what());
    return GROOT_ERUNTIME;
  }
}
int num_sms();

// Caching device allocator (like torch's): blocks are rounded to size
// classes and recycled, so per-call temporaries (CUB scratch, CSR counters,
// activations of a re-encoded graph) cost no cudaMalloc/cudaFree after warm-up.
void* dev_alloc(size_t bytes);
void dev_free(void* p);
void dev_empty_cache();

// Per-kernel CUDA-event timing on the library stream (groot_profile_*).
struct ProfScope {
  int slot = -1;
  explicit ProfScope(const char* name);
  ~ProfScope();
};

// Owning device buffer.
template <class T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  explicit DevBuf(size_t count) { alloc(count); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), n(o.n) { o.p = nullptr; o.n = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; n = o.n; o.p = nullptr; o.n = 0; }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(size_t count) {
    release();
    n = count;
    if (count) p = static_cast<T*>(dev_alloc(count * sizeof(T) + 16));
  }
  void release() {
    if (p) dev_free(p);
    p = nullptr;
    n = 0;
  }
  void zero() {
    if (p) GROOT_CUDA(cudaMemsetAsync(p, 0, n * sizeof(T), stream()));
  }
  void upload(const T* h, size_t count) {
    if (count) GROOT_CUDA(cudaMemcpyAsync(p, h, count * sizeof(T), cudaMemcpyHostToDevice, stream()));
  }
  void download(T* h, size_t count) const {
    if (count) GROOT_CUDA(cudaMemcpyAsync(h, p, count * sizeof(T), cudaMemcpyDeviceToHost, stream()));
  }
};

inline unsigned blocks_for(uint64_t items, unsigned threads, unsigned cap = 148u * 16u) {
  uint64_t b = (items + threads - 1) / threads;
  if (b == 0) b = 1;
  return static_cast<unsigned>(b < cap ? b : cap);
}

// ---- graph-building primitives (graph_build.cu) -----------------------------
// Symmetric CSR from a forward edge list (build_symmetric_csr, src/encode.cpp:14-31):
// rows ascending, duplicates kept. rp: u32[n+1], col: u32[2*ne].
void build_csr(uint32_t n, uint64_t ne, const uint32_t* d_edges, uint32_t* d_rp, uint32_t* d_col);
// Exclusive prefix sum of u32 counts into u32 offsets (count+1 outputs).
void exclusive_scan_u32(const uint32_t* d_in, uint32_t* d_out, uint64_t count);
void exclusive_scan_u64(const uint64_t* d_in, uint64_t* d_out, uint64_t count);
// dst[k*len + i] = src[i] + k*offset (graph_build.cu)
__global__ void replicate_offset_kernel(uint64_t len, uint32_t copies, uint32_t offset, const uint32_t* src,
                                        uint32_t* dst);

}  // namespace groot

// ---- opaque handle bodies --------------------------------------------------------
struct groot_graph {
  int device = 0;
  uint32_t n = 0;
  uint64_t nnz = 0, ne = 0;
  groot::DevBuf<uint32_t> rp;      // n+1 (u32: nnz < 2^32 enforced)
  groot::DevBuf<uint32_t> col;     // nnz
  groot::DevBuf<uint8_t> feat;     // 4n, byte j of node v = feature j (== u32 per node)
  groot::DevBuf<uint8_t> labels;   // n
  groot::DevBuf<uint32_t> edges;   // 2*ne (fwd_edges pairs)
  // every feature byte is 0 or 1 (encode's features always are; host uploads are
  // scanned): packed byte counters in the layer-0 gathers are exact
  bool binary_feat = true;
  // Forward-path cache: row classifier output and activation buffers.
  uint32_t hd_threshold = 0;
  uint32_t num_hd = 0;
  groot::DevBuf<uint32_t> hd_rows;  // rows with degree >= hd_threshold, ascending
  groot::DevBuf<float> hd_mean;     // num_hd x 32 neighbour means (scratch per layer)
  groot::DevBuf<float> act[2];      // n x 32 ping-pong activations
  // Per-tile gather plan of the fused layer / SpMM (tile_plan.cuh), built lazily.
  uint32_t tp_threshold = 0, tp_halo_cap = 0, tp_slow = 0;
  uint32_t tp_period = 0, tp_period_rows = 0;  // > 0: periodic plan of one batch copy (see forward.cu)
  groot::DevBuf<uint32_t> tile_ctr;            // dynamic tile scheduler counter of the tile kernels
  // HD plan (forward.cu, hd_chunk_kernel): chunk units sorted by first neighbour
  bool hdp_valid = false;
  uint32_t hdp_nunits = 0;
  groot::DevBuf<uint32_t> hdp_base, hdp_slot, hdp_k, hdp_units;
  groot::DevBuf<float> hdp_partial;
  groot::DevBuf<uint32_t> tp_meta;  // TileMeta per tile (4 x u32)
  groot::DevBuf<uint16_t> tp_lrp;   // kTpLrp u16 per tile
  groot::DevBuf<uint16_t> tp_lcol;  // local neighbour slots
  groot::DevBuf<unsigned long long> tp_rec;  // row records (tile_plan.cuh), tiles x 128
  groot::DevBuf<uint32_t> tp_halo;  // halo rows per tile
  // Keyed layer 0 (forward.cu, l0_key_kernel): per-row records and entry ids,
  // the record dictionary and the entry rows; l0_mode 0 unknown, 1 keyable, 2 not
  int l0_mode = 0;
  groot::DevBuf<unsigned long long> l0_key, l0_dict, l0_ctab;  // l0_key: HD rows' records
  groot::DevBuf<uint16_t> l0_slot;                             // LD rows: slot in their CTA's table
  groot::DevBuf<uint8_t> l0_id, l0_idmap, l0_hid, l0_xlat;
  groot::DevBuf<float> l0_table;
  groot::DevBuf<float> l0_xtab;  // keyed layer 1, transform first: Tn | Ts (entry rows . W_neigh / W_self)
  groot::DevBuf<uint32_t> l0_flags;
};

struct groot_assignment {
  int device = 0;
  uint32_t n = 0, k = 0;
  groot::DevBuf<uint32_t> part_of;
};

struct groot_parts {
  int device = 0;
  uint32_t k = 0;
  int with_boundary = 1;
  std::vector<uint64_t> core_off, bnd_off, edge_off;  // host copies, k+1 each
  groot::DevBuf<uint32_t> core;    // concatenated core_nodes
  groot::DevBuf<uint32_t> bnd;     // concatenated boundary_nodes
  groot::DevBuf<uint32_t> edges;   // concatenated local edge pairs
};

struct groot_model {
  int device = 0;                   // weights live on this device
  uint32_t depth = 0, in_dim = 0, hidden = 0, classes = 0;
  std::vector<double> params;       // fp64, ASG1 order (host copy)
  groot::DevBuf<float> l0;          // layer 0: Ws[4x32], Wn[4x32], b[32]
  float l0w[4 * 32 * 2 + 32];       // same, passed by value as kernel parameters
  groot::DevBuf<uint32_t> bimg;     // layers >= 1: 16 KB smem image each (B hi/lo, swizzled)
  groot::DevBuf<float> bias;        // layers >= 1: 32 each
  groot::DevBuf<float> naive_w;     // fp32 row-major weights for the naive debug path
  groot::DevBuf<float> head;        // W_out[32 x classes] then b_out[classes]
  groot::DevBuf<uint32_t> hbimg;    // last layer's tensor-core head: 4 KB W_out smem image (hi/lo)
  float headw[32 * 8 + 8 + 32];     // same, classes padded to 8, + layer bias; kernel parameters
  std::vector<float> bias_h;        // layers >= 1 biases (host copy for the parameter block)
};
