// tile_plan.cu — builds the per-tile gather plan (tile_plan.cuh) on the device.
//
// One warp per 128-row tile, no global scans (tile_plan_kernel below has the
// details: the tile's slot segment staged in shared memory, nonzero-parallel):
//   * LD degree of each row (degree < threshold; HD rows are flagged and
//     skipped) -> row offsets into the tile's lcol segment (lrp);
//   * each LD nonzero re-indexed to its local slot, stored at its own CSR
//     position (lcol is aligned with col_idx): c - row0 inside the tile;
//   * out-of-tile columns collected in a shared-memory hash set (dedup),
//     compacted and bitonic-sorted -> the halo list (ascending global ids, the
//     tile's fixed kTpHaloCap-entry slot); each out-of-tile nonzero gets 128 +
//     the rank of its column (looked up through the set).
// Deterministic (sorted halo, nonzero order kept). Built once per graph and
// row-classifier threshold and cached on the graph, like the reference's
// make_context builds its plans once per graph (src/gnn.cpp:140-170).
#include <cstdlib>

#include "common.cuh"
#include "tile_plan.cuh"

static_assert(groot::kTpHaloCap <= 256, "halo list sort buffer");

namespace groot {

namespace {

constexpr int kTpWarps = 4;      // tiles per CTA

constexpr uint32_t kHashSlots = 512;  // per-tile open-addressing set of out-of-tile columns
constexpr uint32_t kEmpty = 0xFFFFFFFFu;

__device__ __forceinline__ uint32_t hslot(uint32_t c) { return (c * 2654435761u) >> (32 - 9); }

// Insert c (warp-divergent callers allowed); returns its slot.
__device__ __forceinline__ uint32_t hash_insert(uint32_t* hk, uint32_t c) {
  uint32_t h = hslot(c);
  while (true) {
    const uint32_t old = atomicCAS(&hk[h], kEmpty, c);
    if (old == kEmpty || old == c) return h;
    h = (h + 1) & (kHashSlots - 1);
  }
}
__device__ __forceinline__ uint32_t hash_find(const uint32_t* hk, uint32_t c) {
  uint32_t h = hslot(c);
  while (hk[h] != c) h = (h + 1) & (kHashSlots - 1);
  return h;
}

// Warp-wide bitonic sort of 32*PER keys held PER per lane (index lane*PER + k),
// ascending: in-register compare-exchanges below distance PER, shuffles above.
template <uint32_t PER>
__device__ __forceinline__ void warp_sort(uint32_t (&v)[PER], uint32_t lane) {
#pragma unroll
  for (uint32_t s = 2; s <= 32 * PER; s <<= 1) {
#pragma unroll
    for (uint32_t d = s >> 1; d > 0; d >>= 1) {
      if (d >= PER) {
        const uint32_t lb = d / PER;
        const bool lower = (lane & lb) == 0;
#pragma unroll
        for (uint32_t k = 0; k < PER; ++k) {
          const uint32_t p = __shfl_xor_sync(0xffffffffu, v[k], lb);
          const bool up = ((lane * PER + k) & s) == 0;
          v[k] = (lower == up) ? min(v[k], p) : max(v[k], p);
        }
      } else {
#pragma unroll
        for (uint32_t k = 0; k < PER; ++k) {
          if (k & d) continue;
          const uint32_t x = v[k], y = v[k ^ d];
          const bool up = ((lane * PER + k) & s) == 0;
          if ((x > y) == up) {
            v[k] = y;
            v[k ^ d] = x;
          }
        }
      }
    }
  }
}

// One warp per tile, nonzero-parallel over the tile's staged slot segment:
// the segment [loff, loff + lcnt) of col_idx is copied to shared memory once
// (coalesced); each lane takes nonzeros lane, lane + 32, ...: in-tile columns
// get their slot, out-of-tile columns go into a shared-memory hash set; the
// set is compacted and sorted in registers (the halo list); a second pass over
// the staged segment gives out-of-tile nonzeros their rank. HD rows' nonzeros
// are masked out (a bitmap over the segment). Row records from the staged slots.
__global__ void __launch_bounds__(kTpWarps * 32) tile_plan_kernel(uint32_t n, const uint32_t* __restrict__ rp,
                                                                  const uint32_t* __restrict__ col, uint32_t thr,
                                                                  uint32_t halo_cap, TileMeta* meta, uint16_t* lrp,
                                                                  uint16_t* lcol, uint32_t* halo,
                                                                  unsigned long long* rec, uint32_t* slow_count) {
  __shared__ uint32_t hk_all[kTpWarps][kHashSlots];      // set of out-of-tile columns
  __shared__ uint16_t hv_all[kTpWarps][kHashSlots];      // their rank in the sorted halo list
  __shared__ __align__(16) uint32_t seg_all[kTpWarps][kTpColCap];  // the tile's slot segment of col_idx
  __shared__ uint16_t sl_all[kTpWarps][kTpColCap];       // local slot of every staged nonzero
  __shared__ uint32_t hdm_all[kTpWarps][kTpColCap / 32];  // staged nonzeros of HD rows (bitmap)
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint32_t* hk = hk_all[wib];
  uint16_t* hv = hv_all[wib];
  uint32_t* seg = seg_all[wib];
  uint16_t* sl = sl_all[wib];
  uint32_t* hdm = hdm_all[wib];
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
    const uint32_t k0 = base - loff, k1 = end - loff;  // this tile's nonzeros in the segment
    bool slow = lcnt > kTpColCap;
    uint32_t H = 0;
    uint32_t hsorted[8];
    if (!slow) {
      // stage the segment (16-B loads: loff is a multiple of 8 entries) and the HD mask
      for (uint32_t i = lane; i < lcnt / 4; i += 32)
        reinterpret_cast<uint4*>(seg)[i] = __ldg(reinterpret_cast<const uint4*>(col + loff) + i);
      for (uint32_t i = lane; i < kTpColCap / 32; i += 32) hdm[i] = 0u;
#pragma unroll
      for (uint32_t i = lane; i < kHashSlots; i += 32) hk[i] = kEmpty;
      __syncwarp();
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (hd[i] && d[i])
          for (uint32_t k = b[i] - loff; k < b[i] - loff + d[i] && k < kTpColCap; ++k) atomicOr(&hdm[k >> 5], 1u << (k & 31));
      __syncwarp();
      // pass 1: in-tile slots; out-of-tile columns into the set (more than half
      // the set's slots of out-of-tile references -> slow tile)
      uint32_t outs = 0;
      for (uint32_t k = k0 + lane; k < k1; k += 32) {
        if ((hdm[k >> 5] >> (k & 31)) & 1u) continue;
        const uint32_t c = seg[k];
        if (c - row0 < kTpRows) sl[k] = static_cast<uint16_t>(c - row0);
        else ++outs;
      }
      slow = __reduce_add_sync(0xffffffffu, outs) > kHashSlots / 2;
      if (!slow) {
        for (uint32_t k = k0 + lane; k < k1; k += 32) {
          if ((hdm[k >> 5] >> (k & 31)) & 1u) continue;
          const uint32_t c = seg[k];
          if (c - row0 >= kTpRows) hash_insert(hk, c);
        }
        __syncwarp();
        // compact the set into registers (lane*8 + k), then sort: the halo list
        uint32_t* uq = reinterpret_cast<uint32_t*>(hv);  // (hv is rewritten below) 512 u16 = 256 u32 scratch
#pragma unroll
        for (uint32_t i0 = 0; i0 < kHashSlots; i0 += 32) {
          const uint32_t c = hk[i0 + lane];
          const uint32_t m = __ballot_sync(0xffffffffu, c != kEmpty);
          const uint32_t at = H + __popc(m & ((1u << lane) - 1u));
          if (c != kEmpty && at < 256) uq[at] = c;
          H += __popc(m);
        }
        slow = H > halo_cap;
        if (!slow) {
          __syncwarp();
          if (H <= 128) {  // the usual halo (~120 rows on CSA tiles): a 128-key sort, 4 per lane
            uint32_t h4[4];
#pragma unroll
            for (uint32_t k = 0; k < 4; ++k) h4[k] = lane * 4 + k < H ? uq[lane * 4 + k] : kEmpty;
            __syncwarp();
            warp_sort<4>(h4, lane);
#pragma unroll
            for (uint32_t k = 0; k < 8; ++k) {  // to the 8-per-lane layout: element lane*8+k
              const uint32_t x = __shfl_sync(0xffffffffu, h4[k & 3], (2 * lane + (k >> 2)) & 31);
              hsorted[k] = lane < 16 ? x : kEmpty;
            }
          } else {
#pragma unroll
            for (uint32_t k = 0; k < 8; ++k) hsorted[k] = lane * 8 + k < H ? uq[lane * 8 + k] : kEmpty;
            __syncwarp();
            warp_sort<8>(hsorted, lane);
          }
#pragma unroll
          for (uint32_t k = 0; k < 8; ++k)
            if (lane * 8 + k < H) hv[hash_find(hk, hsorted[k])] = static_cast<uint16_t>(lane * 8 + k);
          __syncwarp();
          // pass 2: out-of-tile nonzeros get 128 + their rank; every slot to lcol
          for (uint32_t k = k0 + lane; k < k1; k += 32) {
            if ((hdm[k >> 5] >> (k & 31)) & 1u) continue;
            const uint32_t c = seg[k];
            uint32_t v;
            if (c - row0 < kTpRows) v = c - row0;
            else {
              v = kTpRows + hv[hash_find(hk, c)];
              sl[k] = static_cast<uint16_t>(v);
            }
            lcol[loff + k] = static_cast<uint16_t>(v);
          }
          __syncwarp();
        }
      }
    }
    // the slot list is staged only for tiles with a row of degree > kTpRecSlots
    // (the records hold every other row's slots)
    bool lng = false;
#pragma unroll
    for (int i = 0; i < 4; ++i) lng |= !hd[i] && d[i] > kTpRecSlots;
    lng = __any_sync(0xffffffffu, lng);
    if (lane == 0) {
      meta[t] = TileMeta{loff, t * kTpHaloCap, (slow || !lng) ? 0u : lcnt, slow ? kTpSlow : H};
      if (slow) atomicAdd(slow_count, 1u);
    }
    if (!slow) {
      uint16_t* lr = lrp + static_cast<size_t>(t) * kTpLrp;
#pragma unroll
      for (int i = 0; i < 4; ++i) lr[32 * i + lane] = static_cast<uint16_t>((b[i] - loff) | (hd[i] ? kTpHdBit : 0u));
      if (lane < kTpLrp - kTpRows) lr[kTpRows + lane] = static_cast<uint16_t>(end - loff);
      // halo list: sorted element i lives in lane i / 8, register i % 8 (padded to a multiple of 4)
      const uint32_t hp = (H + 3u) & ~3u;
#pragma unroll
      for (uint32_t k = 0; k < 8; ++k) {
        const uint32_t i = lane * 8 + k;
        if (i < H) halo[t * kTpHaloCap + i] = hsorted[k];
      }
      if (H & 3u) {  // padding entries repeat the last row (read, never used)
        const uint32_t last = __shfl_sync(0xffffffffu, hsorted[(H - 1) & 7], (H - 1) >> 3);
        for (uint32_t i = H + lane; i < hp; i += 32) halo[t * kTpHaloCap + i] = last;
      }
      // row records: the first kTpRecSlots slots of each row, unused fields -> the zero slot
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        uint32_t f[kTpRecSlots];
#pragma unroll
        for (uint32_t k = 0; k < kTpRecSlots; ++k)
          f[k] = (!hd[i] && k < d[i] ? static_cast<uint32_t>(sl[b[i] - loff + k]) : kTpZeroSlot) << 7;
        const uint32_t dl = hd[i] ? 0u : d[i];  // LD degree < thr <= 256
        f[0] |= dl & 0x7Fu;
        f[1] |= (hd[i] ? 1u : 0u) | (dl > kTpRecSlots ? 2u : 0u) | ((dl >> 7) << 2);
        rec[static_cast<size_t>(t) * kTpRows + 32 * i + lane] =
            static_cast<unsigned long long>(f[0] | (f[1] << 16)) | (static_cast<unsigned long long>(f[2] | (f[3] << 16)) << 32);
      }
    }
    __syncwarp();
  }
}

}  // namespace

uint32_t tile_halo_cap() {
  static uint32_t cap = [] {
    const char* e = std::getenv("GROOT_TP_HALO_CAP");  // test knob: force slow tiles
    // (the last halo slot is the zero row of the row records: kTpZeroSlot)
    const uint32_t v = e ? static_cast<uint32_t>(std::strtoul(e, nullptr, 10)) : kTpHaloCap - 1;
    return v > kTpHaloCap - 1 ? kTpHaloCap - 1 : v;
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
  g->tp_rec.alloc(static_cast<size_t>(ntiles) * kTpRows);
  DevBuf<uint32_t> slow(1);
  slow.zero();
  const unsigned grid = std::min<uint32_t>((ntiles + kTpWarps - 1) / kTpWarps, static_cast<uint32_t>(num_sms()) * 16u);
  GROOT_LAUNCH(tile_plan_kernel, grid, kTpWarps * 32, 0, n, g->rp.p, g->col.p, thr, cap,
               reinterpret_cast<TileMeta*>(g->tp_meta.p), g->tp_lrp.p, g->tp_lcol.p, g->tp_halo.p, g->tp_rec.p, slow.p);
  g->tp_threshold = thr;  // (the slow-tile count stays on the device: no host synchronisation)
  g->tp_halo_cap = cap;
}

}  // namespace groot

namespace groot {
void classify_rows(groot_graph* g, uint32_t thr);
uint32_t hd_threshold();
void replicate_hd_plan(groot_graph* src, groot_graph* dst, uint32_t copies);

// Give the tile-aligned batch `dst` (batch_padded(src, copies, P)) the row
// classifier output of `src` replicated and the tile plan of `src` as a
// periodic plan: tile k*T + t of the batch reads plan tile t of copy 0 (same
// row offsets and local slots, lcol segments inside copy 0's nonzeros) and
// shifts its halo rows by k*P. False if the layout does not allow it (the
// forward then builds its own plan).
bool replicate_forward_plan(groot_graph* src, groot_graph* dst, uint32_t copies, uint32_t P) {
  const uint32_t T = (src->n + kTpRows - 1) / kTpRows;
  if (src->n == 0 || P != T * kTpRows) return false;
  const uint32_t thr = hd_threshold();
  classify_rows(src, thr);
  build_tile_plan(src, thr);
  // (slow tiles need nothing per copy: they gather from the batch's own CSR)
  // row classifier: HD rows of copy 0, shifted per copy (stays ascending)
  dst->num_hd = src->num_hd * copies;
  dst->hd_rows.alloc(dst->num_hd);
  if (dst->num_hd)
    GROOT_LAUNCH(replicate_offset_kernel, blocks_for(dst->num_hd / 4 + 1, 256), 256, 0,
                 static_cast<uint64_t>(src->num_hd), copies, P, src->hd_rows.p, dst->hd_rows.p);
  dst->hd_mean.alloc(static_cast<size_t>(dst->num_hd) * 32);
  dst->hd_threshold = thr;
  replicate_hd_plan(src, dst, copies);
  dst->tp_meta = std::move(src->tp_meta);
  dst->tp_lrp = std::move(src->tp_lrp);
  dst->tp_lcol = std::move(src->tp_lcol);
  dst->tp_halo = std::move(src->tp_halo);
  dst->tp_rec = std::move(src->tp_rec);
  dst->tp_threshold = src->tp_threshold;
  dst->tp_halo_cap = src->tp_halo_cap;
  dst->tp_slow = src->tp_slow * copies;
  dst->tp_period = T;
  dst->tp_period_rows = P;
  src->tp_threshold = 0;  // src no longer owns a plan
  return true;
}
}  // namespace groot
