// tile_plan.cuh — the per-tile gather plan of the fused SAGE layer and the
// standalone SpMM (the device-side counterpart of the reference's SpmmPlan,
// src/spmm.cpp:37-127, inc/spmm.hpp:51-100).
//
// The reference plans work units over degree-sorted rows and stages LD rows
// contiguously ("coalesce dumping", inc/spmm.hpp:129-135). On B200 the unit is
// a 128-row tile in natural (topological) row order, and what is planned is
// where each neighbour row comes from:
//   * rows inside the tile   -> the tile's own feature rows, one TMA box load;
//   * rows outside the tile  -> the tile's halo: the sorted, unique
//                               out-of-tile neighbours of its LD rows, copied
//                               into shared memory right after the tile rows.
// Every LD nonzero is re-indexed to a u16 local slot (< 128: tile row, >= 128:
// halo row 128 + k), so a neighbour read is one shared-memory access instead
// of a 128-byte L2 gather; nonzero order is kept, so sums are in the
// reference's order. In a 1024-bit CSA graph 61% of nonzeros are in-tile and
// the halo averages 117 rows per tile (1.4 references per halo row), which
// cuts the per-layer L2->SM gather volume from 68.7 GB to ~16 GB.
//
// Tiles whose LD nonzeros or halo exceed the staging capacity are flagged
// slow: the kernels gather them straight from the global CSR (rare: 40 of
// 65,481 tiles of a 1024-bit copy, all next to the primary inputs).
#pragma once
#include <stdint.h>

namespace groot {

constexpr uint32_t kTpRows = 128;      // rows per tile (= UMMA M)
constexpr uint32_t kTpHaloCap = 160;   // halo rows staged per tile
constexpr uint32_t kTpColCap = 1024;   // LD nonzeros staged per tile
constexpr uint32_t kTpLrp = 136;       // u16 row offsets per tile (129 used; 272 B, 16-B multiple)
constexpr uint32_t kTpSlow = 1u << 31; // meta.w flag: gather from the global CSR
constexpr uint32_t kTpHdBit = 0x8000u; // lrp entry flag: row is HD (mean computed by the HD kernel)
// The last halo slot is never a halo row (at most kTpHaloCap - 1 are staged):
// the kernels keep it zero, and row records point their unused neighbour
// slots at it, so the gather of a row is branch-free (adding +0 to a sum that
// starts at +0 changes nothing).
constexpr uint32_t kTpZeroSlot = kTpRows + kTpHaloCap - 1;
// Row record (u64 per tile row, 8 B): the row's first four local neighbour
// slots inline, so the producers need one shared-memory load per row before
// its neighbour rows instead of the chain row offsets -> slot list -> rows.
// u16 field k (k = 0..3) = slot_k * 128 (the row's byte offset in the staged
// rows; kTpZeroSlot past the degree) | low 7 bits:
//   field 0: LD degree bits 0..6 (0 for HD rows)
//   field 1: bit 0 HD row (mean from the HD kernel), bit 1 degree > 4 (slots
//            4.. come from the lcol segment at the lrp offset), bit 2 degree
//            bit 7 (LD degree < threshold <= 256)
constexpr uint32_t kTpRecSlots = 4;
constexpr uint32_t kTpRecOffMask = 0xFF80u;
constexpr uint32_t kTpRecHd = 1u << 16, kTpRecLong = 1u << 17;  // in the low u32 of the record
constexpr uint32_t tp_rec_degree(uint32_t lo32) { return (lo32 & 0x7Fu) | ((lo32 >> 11) & 0x80u); }
static_assert((kTpZeroSlot << 7) <= 0xFFFFu, "slot byte offsets fit a u16 field");

// Layout: rec holds one record per tile row (tiles x kTpRows); lcol is aligned with col_idx (entry e = local slot of nonzero e;
// entries of HD rows are not written), each tile's halo list sits in a fixed
// kTpHaloCap-entry slot, lrp holds the rows' offsets into the tile's staged
// lcol segment [lcol_off, lcol_off + lcol_cnt) | kTpHdBit.
// Per-tile record (16 B): lcol segment start (entries, multiple of 8), halo
// list offset (= tile * kTpHaloCap), staged lcol entries (multiple of 8; 0 if
// slow or if no row of the tile has more than kTpRecSlots neighbours: the row
// records then hold every slot), halo row count | kTpSlow.
struct TileMeta {
  uint32_t lcol_off, halo_off, lcol_cnt, halo;
};

}  // namespace groot
