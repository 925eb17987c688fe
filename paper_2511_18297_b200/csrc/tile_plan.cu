// tile_plan.cu — builds the per-tile gather plan (tile_plan.cuh) on the device.
//
// One warp per 128-row tile, one pass, no global scans:
//   * LD degree of each row (degree < threshold; HD rows are flagged and
//     skipped) -> row offsets into the tile's lcol segment (lrp);
//   * out-of-tile columns of the LD rows gathered into shared memory (warp
//     ballots), bitonic sort, unique -> the halo list (ascending global ids),
//     written to the tile's fixed kTpHaloCap-entry slot;
//   * each LD nonzero re-indexed to its local slot, stored at its own CSR
//     position (lcol is aligned with col_idx): c - row0 inside the tile,
//     128 + rank of c in the halo list otherwise.
// Deterministic (sorted halo, nonzero order kept). Built once per graph and
// row-classifier threshold and cached on the graph, like the reference's
// make_context builds its plans once per graph (src/gnn.cpp:140-170).
#include <cstdlib>

#include "common.cuh"
#include "tile_plan.cuh"

namespace groot {

namespace {

constexpr int kTpWarps = 4;  // tiles per CTA

__device__ __forceinline__ uint32_t lower_bound_u32(const uint32_t* a, uint32_t len, uint32_t x) {
  uint32_t lo = 0, hi = len;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ uint32_t warp_excl_scan(uint32_t v, uint32_t lane, uint32_t& total) {
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= static_cast<uint32_t>(o)) x += y;
  }
  total = __shfl_sync(0xffffffffu, x, 31);
  return x - v;
}

__global__ void __launch_bounds__(kTpWarps * 32) tile_plan_kernel(uint32_t n, const uint32_t* __restrict__ rp,
                                                                  const uint32_t* __restrict__ col, uint32_t thr,
                                                                  uint32_t halo_cap, TileMeta* meta, uint16_t* lrp,
                                                                  uint16_t* lcol, uint32_t* halo,
                                                                  uint32_t* slow_count) {
  __shared__ uint32_t keys_all[kTpWarps][kTpColCap];
  __shared__ uint32_t uniq_all[kTpWarps][kTpHaloCap + 1];
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint32_t* keys = keys_all[wib];
  uint32_t* uniq = uniq_all[wib];
  const uint32_t ntiles = (n + kTpRows - 1) / kTpRows;
  for (uint32_t t = blockIdx.x * kTpWarps + wib; t < ntiles; t += gridDim.x * kTpWarps) {
    const uint32_t row0 = t * kTpRows;
    uint32_t b[4], d[4];
    bool hd[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {  // rows row0 + 32i + lane: prefix order is i-major
      const uint32_t r = min(row0 + 32u * i + lane, n);
      b[i] = rp[r];
      d[i] = r < n ? rp[r + 1] - b[i] : 0u;
      hd[i] = d[i] >= thr;
    }
    const uint32_t base = __shfl_sync(0xffffffffu, b[0], 0);
    const uint32_t end = rp[min(row0 + kTpRows, n)];
    const uint32_t loff = base & ~7u;
    const uint32_t lcnt = (end - loff + 7u) & ~7u;
    bool slow = lcnt > kTpColCap;
    uint32_t H = 0;
    if (!slow) {
      // out-of-tile columns of the LD rows
      uint32_t cnt = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const uint32_t dl = hd[i] ? 0u : d[i];
        const uint32_t dmax = __reduce_max_sync(0xffffffffu, dl);
        for (uint32_t k = 0; k < dmax; ++k) {
          const uint32_t c = k < dl ? col[b[i] + k] : row0;
          const bool out = k < dl && c - row0 >= kTpRows;
          const uint32_t m = __ballot_sync(0xffffffffu, out);
          if (out) keys[cnt + __popc(m & ((1u << lane) - 1u))] = c;
          cnt += __popc(m);
        }
      }
      uint32_t P = 32;
      while (P < cnt) P <<= 1;
      for (uint32_t i = cnt + lane; i < P; i += 32) keys[i] = 0xFFFFFFFFu;
      __syncwarp();
      for (uint32_t k = 2; k <= P; k <<= 1)
        for (uint32_t jj = k >> 1; jj > 0; jj >>= 1) {
          for (uint32_t x = lane; x < P / 2; x += 32) {
            const uint32_t i = 2 * jj * (x / jj) + (x % jj), p = i + jj;
            const uint32_t u = keys[i], v = keys[p];
            if ((u > v) == ((i & k) == 0)) {
              keys[i] = v;
              keys[p] = u;
            }
          }
          __syncwarp();
        }
      // unique: lane owns keys [lane*per, lane*per + per)
      const uint32_t per = (cnt + 31) / 32;
      const uint32_t i0 = min(lane * per, cnt), i1 = min(i0 + per, cnt);
      uint32_t u = 0;
      for (uint32_t i = i0; i < i1; ++i) u += (i == 0 || keys[i] != keys[i - 1]);
      uint32_t pos = warp_excl_scan(u, lane, H);
      slow = H > halo_cap;
      if (!slow)
        for (uint32_t i = i0; i < i1; ++i)
          if (i == 0 || keys[i] != keys[i - 1]) uniq[pos++] = keys[i];
      __syncwarp();
    }
    if (lane == 0) {
      meta[t] = TileMeta{loff, t * kTpHaloCap, slow ? 0u : lcnt, slow ? kTpSlow : H};
      if (slow) atomicAdd(slow_count, 1u);
    }
    if (slow) continue;
    uint16_t* lr = lrp + static_cast<size_t>(t) * kTpLrp;
#pragma unroll
    for (int i = 0; i < 4; ++i) lr[32 * i + lane] = static_cast<uint16_t>((b[i] - loff) | (hd[i] ? kTpHdBit : 0u));
    if (lane < kTpLrp - kTpRows) lr[kTpRows + lane] = static_cast<uint16_t>(end - loff);
    for (uint32_t i = lane; i < ((H + 3u) & ~3u); i += 32) halo[t * kTpHaloCap + i] = uniq[min(i, H - 1)];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      if (hd[i]) continue;
      for (uint32_t k = 0; k < d[i]; ++k) {
        const uint32_t c = col[b[i] + k];
        const uint32_t loc = (c - row0 < kTpRows) ? c - row0 : kTpRows + lower_bound_u32(uniq, H, c);
        lcol[b[i] + k] = static_cast<uint16_t>(loc);
      }
    }
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
  ProfScope ps("tile_plan");
  g->tp_meta.alloc(4ull * ntiles);
  g->tp_lrp.alloc(static_cast<size_t>(ntiles) * kTpLrp);
  g->tp_lcol.alloc(g->nnz + 16ull);
  g->tp_halo.alloc(static_cast<size_t>(ntiles) * kTpHaloCap);
  DevBuf<uint32_t> slow(1);
  slow.zero();
  const unsigned grid = std::min<uint32_t>((ntiles + kTpWarps - 1) / kTpWarps, static_cast<uint32_t>(num_sms()) * 8u);
  GROOT_LAUNCH(tile_plan_kernel, grid, kTpWarps * 32, 0, n, g->rp.p, g->col.p, thr, cap,
               reinterpret_cast<TileMeta*>(g->tp_meta.p), g->tp_lrp.p, g->tp_lcol.p, g->tp_halo.p, slow.p);
  slow.download(&g->tp_slow, 1);
  stream_sync();
  g->tp_threshold = thr;
  g->tp_halo_cap = cap;
}

}  // namespace groot
