// tile_plan.cu — builds the per-tile gather plan (tile_plan.cuh) on the device.
//
// One CTA per 128-row tile, two passes (count, fill) around two prefix sums:
//   * LD degree of each row (degree < threshold; HD rows get 0 and a flag),
//     block scan -> the tile's local row offsets (lrp) and LD nonzero count L;
//   * out-of-tile columns of the LD rows collected in shared memory, bitonic
//     sort, unique -> the halo list (ascending global row ids);
//   * each LD nonzero re-indexed to its local slot: c - row0 inside the tile,
//     128 + rank of c in the halo list otherwise.
// Deterministic (sorted halo, nonzero order kept). Built once per graph and
// row-classifier threshold and cached on the graph, like the reference's
// make_context builds its plans once per graph (src/gnn.cpp:140-170).
#include <cub/cub.cuh>

#include <cstdlib>

#include "common.cuh"
#include "tile_plan.cuh"

namespace groot {

namespace {

constexpr int kTpThreads = 128;

struct TpShared {
  uint32_t keys[kTpColCap];
  uint32_t uniq[kTpColCap];
  typename cub::BlockScan<uint32_t, kTpThreads>::TempStorage scan;
  uint32_t cnt;
};

__device__ __forceinline__ uint32_t lower_bound_u32(const uint32_t* a, uint32_t len, uint32_t x) {
  uint32_t lo = 0, hi = len;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// kFill = false: lcnt[t] / hcnt[t] = staged lcol / halo-list entries (padded).
// kFill = true : writes meta, lrp, lcol, halo at the scanned offsets.
template <bool kFill>
__global__ void __launch_bounds__(kTpThreads) tile_plan_kernel(uint32_t n, const uint32_t* __restrict__ rp,
                                                               const uint32_t* __restrict__ col, uint32_t thr,
                                                               uint32_t halo_cap, uint32_t* lcnt, uint32_t* hcnt,
                                                               TileMeta* meta, uint16_t* lrp, uint16_t* lcol,
                                                               uint32_t* halo, uint32_t* slow_count) {
  __shared__ TpShared sh;
  const uint32_t tid = threadIdx.x;
  const uint32_t ntiles = (n + kTpRows - 1) / kTpRows;
  using Scan = cub::BlockScan<uint32_t, kTpThreads>;
  for (uint32_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const uint32_t row0 = t * kTpRows, r = row0 + tid;
    uint32_t b = 0, d = 0;
    if (r < n) {
      b = rp[r];
      d = rp[r + 1] - b;
    }
    const bool hd = d >= thr;
    const uint32_t dl = hd ? 0u : d;
    uint32_t off, L;
    Scan(sh.scan).ExclusiveSum(dl, off, L);
    bool slow = L > kTpColCap;
    uint32_t H = 0;
    if (!slow) {
      if (tid == 0) sh.cnt = 0;
      __syncthreads();
      for (uint32_t k = 0; k < dl; ++k) {
        const uint32_t c = col[b + k];
        if (c - row0 >= kTpRows) sh.keys[atomicAdd(&sh.cnt, 1u)] = c;
      }
      __syncthreads();
      const uint32_t O = sh.cnt;
      uint32_t P = 1;
      while (P < O) P <<= 1;
      for (uint32_t i = O + tid; i < P; i += kTpThreads) sh.keys[i] = 0xFFFFFFFFu;
      __syncthreads();
      for (uint32_t k = 2; k <= P; k <<= 1)
        for (uint32_t j = k >> 1; j > 0; j >>= 1) {
          for (uint32_t i = tid; i < P; i += kTpThreads) {
            const uint32_t ixj = i ^ j;
            if (ixj > i) {
              const uint32_t a = sh.keys[i], c = sh.keys[ixj];
              if ((a > c) == ((i & k) == 0)) {
                sh.keys[i] = c;
                sh.keys[ixj] = a;
              }
            }
          }
          __syncthreads();
        }
      // unique: thread tid owns keys [tid*per, tid*per + per)
      const uint32_t per = (O + kTpThreads - 1) / kTpThreads;
      const uint32_t i0 = min(tid * per, O), i1 = min(i0 + per, O);
      uint32_t u = 0;
      for (uint32_t i = i0; i < i1; ++i) u += (i == 0 || sh.keys[i] != sh.keys[i - 1]);
      uint32_t uo;
      Scan(sh.scan).ExclusiveSum(u, uo, H);
      for (uint32_t i = i0; i < i1; ++i)
        if (i == 0 || sh.keys[i] != sh.keys[i - 1]) sh.uniq[uo++] = sh.keys[i];
      __syncthreads();
      slow = H > halo_cap;
    }
    const uint32_t lpad = slow ? 0u : (L + 7u) & ~7u;
    const uint32_t hpad = slow ? 0u : (H + 3u) & ~3u;
    if (!kFill) {
      if (tid == 0) {
        lcnt[t] = lpad;
        hcnt[t] = hpad;
      }
    } else {
      const uint32_t lo = lcnt[t], ho = hcnt[t];  // scanned offsets
      if (tid == 0) {
        meta[t] = TileMeta{lo, ho, lpad, slow ? kTpSlow : H};
        if (slow) atomicAdd(slow_count, 1u);
      }
      uint16_t* lr = lrp + static_cast<size_t>(t) * kTpLrp;
      lr[tid] = static_cast<uint16_t>(slow ? 0u : (off | (hd ? kTpHdBit : 0u)));
      if (tid < kTpLrp - kTpRows) lr[kTpRows + tid] = static_cast<uint16_t>(slow ? 0u : L);
      if (!slow) {
        for (uint32_t i = tid; i < hpad; i += kTpThreads) halo[ho + i] = sh.uniq[min(i, H - 1)];
        for (uint32_t k = 0; k < dl; ++k) {
          const uint32_t c = col[b + k];
          const uint32_t loc = (c - row0 < kTpRows) ? c - row0 : kTpRows + lower_bound_u32(sh.uniq, H, c);
          lcol[lo + off + k] = static_cast<uint16_t>(loc);
        }
        for (uint32_t i = L + tid; i < lpad; i += kTpThreads) lcol[lo + i] = 0;
      }
    }
    __syncthreads();
  }
}

}  // namespace

uint32_t tile_halo_cap() {
  static uint32_t cap = [] {
    const char* e = std::getenv("GROOT_TP_HALO_CAP");  // test knob: force slow tiles
    const uint32_t v = e ? static_cast<uint32_t>(std::strtoul(e, nullptr, 10)) : kTpHaloCap;
    return v > kTpHaloCap ? kTpHaloCap : v;
  }();
  return cap;
}

void build_tile_plan(groot_graph* g, uint32_t thr) {
  const uint32_t cap = tile_halo_cap();
  if (g->tp_threshold == thr && g->tp_halo_cap == cap && g->tp_meta.p) return;
  const uint32_t n = g->n;
  const uint32_t ntiles = (n + kTpRows - 1) / kTpRows;
  if (ntiles == 0) return;
  const unsigned grid = std::min<uint32_t>(ntiles, static_cast<uint32_t>(num_sms()) * 16u);
  DevBuf<uint32_t> lc(ntiles + 1ull), hc(ntiles + 1ull), loff(ntiles + 1ull), hoff(ntiles + 1ull), slow(1);
  GROOT_LAUNCH(tile_plan_kernel<false>, grid, kTpThreads, 0, n, g->rp.p, g->col.p, thr, cap, lc.p, hc.p, nullptr,
               nullptr, nullptr, nullptr, nullptr);
  exclusive_scan_u32(lc.p, loff.p, ntiles);
  exclusive_scan_u32(hc.p, hoff.p, ntiles);
  uint32_t tot[2];
  GROOT_CUDA(cudaMemcpyAsync(&tot[0], loff.p + ntiles, 4, cudaMemcpyDeviceToHost, stream()));
  GROOT_CUDA(cudaMemcpyAsync(&tot[1], hoff.p + ntiles, 4, cudaMemcpyDeviceToHost, stream()));
  stream_sync();
  g->tp_meta.alloc(4ull * ntiles);
  g->tp_lrp.alloc(static_cast<size_t>(ntiles) * kTpLrp);
  g->tp_lcol.alloc(tot[0] + 8ull);
  g->tp_halo.alloc(tot[1] + 4ull);
  slow.zero();
  GROOT_LAUNCH(tile_plan_kernel<true>, grid, kTpThreads, 0, n, g->rp.p, g->col.p, thr, cap, loff.p, hoff.p,
               reinterpret_cast<TileMeta*>(g->tp_meta.p), g->tp_lrp.p, g->tp_lcol.p, g->tp_halo.p, slow.p);
  slow.download(&g->tp_slow, 1);
  stream_sync();
  g->tp_threshold = thr;
  g->tp_halo_cap = cap;
}

}  // namespace groot
