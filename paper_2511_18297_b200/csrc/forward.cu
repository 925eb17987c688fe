// forward.cu — GraphSAGE mean-aggregator forward + classify on sm_100a.
//
// Reference: run_forward / predict_full (src/gnn.cpp:37-52, 259-300) over the
// degree-polarised SpMM (src/spmm.cpp:37-127, inc/spmm.hpp:106-181).
//
// Per layer l >= 1 (32 -> 32) one persistent, warp-specialised kernel per SM
// (sage_tile_kernel) walks 128-row tiles with the tile plan of tile_plan.cuh:
//   loader warp   plan records (row records, halo list; row offsets and slot
//                 list for tiles with rows of degree > 4) by bulk copy, the
//                 tile's 128 feature rows by one TMA box
//   copier warps  the tile's halo rows (out-of-tile neighbours) by cp.async,
//                 into the stage right behind the tile rows
//   8 producers   per row: one row record (its first four neighbour slots,
//                 tile_plan.cuh), the neighbour rows from shared memory, sum in
//                 nonzero order, x 1/deg, TF32 hi/lo split of [h | mean(h_N)]
//                 written straight into tensor memory (tcgen05.st)
//   MMA warp      tcgen05.mma kind::tf32, A from TMEM, W from smem, 3 products
//                 (hi*hi + hi*lo + lo*hi) into a double-buffered accumulator
//   4 epilogue    tcgen05.ld, + bias, ReLU, 256-bit stores of whole rows (or, in
//                 the last layer, the 32 -> classes head on the tensor core +
//                 first-max argmax; classes-only calls certify each row's class
//                 from a single-operand head with a margin bound, GROOT_HEAD_CERT)
// The same kernel without the MMA is the standalone LD SpMM. High-degree rows
// (the row classifier's HD band; the PIs of a multiplier) are aggregated first
// in L2-ordered chunks with a fixed-order reduction (hd_chunk_kernel).
// Layer 0 (4 -> 32, inputs in {0,1}^4) is keyed by default: per row an exact
// integer record, a dictionary of the distinct records, their 4 -> 32 rows and
// a u8 entry id per row (l0_key_tile_kernel ...); layer 1 then reads entry ids
// instead of layer-0 rows and, when more layers follow, runs transform-first
// (kModeXform). Graphs that are not keyable use sage_layer0_kernel.
#include <cub/cub.cuh>
#include <cuda.h>

#include <atomic>
#include <chrono>
#include <cstdlib>
#include <mutex>
#include <cstdio>
#include <cstring>

#include "common.cuh"
#include "ptx.cuh"
#include "tile_plan.cuh"

namespace groot {

constexpr int kF = 32;                       // hidden width (tensor-core layers)
constexpr int kTileM = 128;                  // rows per MMA tile (UMMA M)
static_assert(kTileM == static_cast<int>(kTpRows), "plan tiles are MMA tiles");
constexpr int kEpiWarps = 4;                 // warps 0..3: accumulator drain (TMEM lane quadrant = warp)
constexpr int kProdWarps = 8;                // warps 4..11: gather producers, 16 rows each
constexpr int kMmaWarp = kEpiWarps + kProdWarps;  // warp 12: TMEM alloc + tcgen05.mma issue
constexpr int kLoadWarp = kMmaWarp + 1;           // warp 13: plan records + tile rows
constexpr int kThreads = 16 * 32;  // 512; warps 14, 15 copy halo rows
constexpr int kStages = 3;
// Tensor memory (512 columns x 128 lanes x 32 bit): the A operand lives there,
// so the gather never goes through a shared-memory operand tile. Stage s owns
// columns [128s, 128s+128): h_hi | m_hi | h_lo | m_lo (32 columns each, K
// order permuted, see kcol_feature); the two accumulators follow.
constexpr uint32_t kStageCols = 128;
constexpr uint32_t kAccCols = 32;
constexpr uint32_t kAccCol0 = kStages * kStageCols;  // 384
constexpr uint32_t kTmemCols = 512;
static_assert(kAccCol0 + 2 * kAccCols <= kTmemCols, "tensor memory budget");
constexpr uint32_t kBBytes = 4 * 4096;            // W_self hi/lo, W_neigh hi/lo (32 x 32 each)
constexpr int kMaxClasses = 8;
// Last layer: the 32 -> classes head runs on the tensor core too: the epilogue
// writes its A operand into TMEM (kHeadHiCol), one MMA group of N = 16
// (classes zero-padded) leaves the logits in kHeadDCol. Without the certified
// head (GROOT_HEAD_CERT=0) the A operand is relu(acc + b) split into TF32 hi
// and lo (kHeadLoCol), and the last layer keeps ONE accumulator (freed right
// after the epilogue loads it) to make room.
constexpr uint32_t kHeadN = 16;
// Last layer, classes only (no logits requested): certified single-operand head.
// The epilogue stores relu(acc + b) once (no TF32 hi/lo split); the head MMA
// forms x.W (W hi + lo) and, in columns 8.., S_c = x.|W_c|, with x taken at
// TF32 by the tensor core (|x - tf32(x)| <= 2^-10 tf32(x)), so every logit is
// within 2^-10 S_c of x.W. A row whose top-2 margin exceeds the two bounds has
// the class of the exact logits; any other row (and every row when logits are
// requested) recomputes its head in fp32 FFMA from x in registers.
#ifndef GROOT_HEAD_CERT
#define GROOT_HEAD_CERT 1
#endif
#ifndef GROOT_LAST_PIPE
#define GROOT_LAST_PIPE (!GROOT_HEAD_CERT)  // last layer: head of tile i drained behind the split of tile i + 1
#endif
// GROOT_LAST_ACC2 (certified head only): its A operand needs 32 columns, not
// 64, so the last layer can keep both accumulators (head A at 448, logits at
// 480) with the MMA warp issuing tile i's head after tile i + 1's layer MMAs.
// Measured +1.5 % against one accumulator (two A/B pairs), so off.
#ifndef GROOT_LAST_ACC2
#define GROOT_LAST_ACC2 0
#endif
static_assert(!(GROOT_HEAD_CERT && GROOT_LAST_PIPE), "the certified head keeps its row's x in registers");
static_assert(!GROOT_LAST_ACC2 || GROOT_HEAD_CERT, "two accumulators leave room for the certified head only");
// the MMA warp issues tile i's head after tile i + 1's layer MMAs
#ifndef GROOT_HEAD_AFTER_MMA
#define GROOT_HEAD_AFTER_MMA (GROOT_LAST_PIPE || GROOT_LAST_ACC2)
#endif
constexpr uint32_t kHeadHiCol = kAccCol0 + (GROOT_LAST_ACC2 ? 2 : 1) * kAccCols;  // 448 (ACC2) / 416 (the unused second accumulator)
constexpr uint32_t kHeadLoCol = kAccCol0 + 2 * kAccCols;  // 448 (not with the certified head)
constexpr uint32_t kHeadDCol = kAccCol0 + 3 * kAccCols;   // 480
static_assert(kHeadDCol + kHeadN <= kTmemCols, "tensor memory budget (head)");
constexpr uint32_t kHeadBBytes = 2 * kHeadN * 128;        // W_out hi/lo, K-major SW128, N = 16 rows
// Column c (0..31) of an A block in tensor memory holds input feature
// kcol_feature(c): lane j of a row's 4-lane group loads features 8j..8j+7
// (one 32-byte load) and 16x256b stores put its values in columns 8i+2j+e.
// The weight image permutes B's K rows the same way, so A.B is unchanged.
__host__ __device__ constexpr uint32_t kcol_feature(uint32_t c) {
  return ((c >> 1) & 3u) * 8u + (c >> 3) * 2u + (c & 1u);
}
// Column holding feature f (inverse of kcol_feature): f = 8j + 2i + e -> 8i + 2j + e.
__host__ __device__ constexpr uint32_t kcol_inverse(uint32_t f) {
  return ((f >> 1) & 3u) * 8u + (f >> 3) * 2u + (f & 1u);
}
static_assert(kcol_inverse(kcol_feature(13)) == 13 && kcol_feature(kcol_inverse(22)) == 22, "permutation");

static uint32_t env_u32(const char* name, uint32_t dflt) {
  const char* e = std::getenv(name);
  return e ? static_cast<uint32_t>(std::strtoul(e, nullptr, 10)) : dflt;
}

uint32_t hd_threshold() {
  static uint32_t t = [] {
    const char* e = std::getenv("GROOT_HD_THRESHOLD");
    // LD rows (degree < threshold) index a 256-entry reciprocal table in the fused layer.
    const uint32_t v = e ? static_cast<uint32_t>(std::strtoul(e, nullptr, 10)) : 128u;
    return v < 1 ? 1u : (v > 256 ? 256u : v);
  }();
  return t;
}

struct HdInfo {
  const uint32_t* rows;  // ascending
  uint32_t count;
  uint32_t threshold;
  const float* mean;  // count x width
};

__device__ __forceinline__ uint32_t hd_slot(const HdInfo& hd, uint32_t row) {
  uint32_t lo = 0, hi = hd.count;
  while (lo < hi) {
    const uint32_t mid = (lo + hi) >> 1;
    if (hd.rows[mid] < row) lo = mid + 1; else hi = mid;
  }
  return lo;
}

__device__ __forceinline__ float4 f4add(float4 a, float4 b) {
  return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
}

__device__ __forceinline__ float4 f4scale(float4 a, float s) {
  return make_float4(a.x * s, a.y * s, a.z * s, a.w * s);
}

// Head weights by value: kernel parameters live in the constant bank, so the
// 32 x classes FFMAs of the last epilogue read them as free operands.
struct HeadW {
  float w[32][8];  // W_out[k][c], classes padded to 8
  float b[8];
  float bias[32];  // this layer's bias (constant-bank operand in the epilogue)
};

// TF32 split by truncation of one 16-row slice (rows r, r+8 of the lane's
// group; lane j holds features 8j..8j+7 of each) into tensor memory: hi = x with
// the low 13 mantissa bits cleared (an exact TF32 value), lo = x - hi (exact,
// Sterbenz). Register 4i+2h+e of the 16x256b store is feature 2i+e of row h.
__device__ __forceinline__ void split_regs(const float4 (&x)[2][2], uint32_t (&hi)[16], uint32_t (&lo)[16]) {
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const float f[4] = {x[h][c].x, x[h][c].y, x[h][c].z, x[h][c].w};
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const int idx = 4 * (2 * c + p) + 2 * h;  // features 4c+2p, 4c+2p+1
        const float h0 = __uint_as_float(__float_as_uint(f[2 * p]) & 0xFFFFE000u);
        const float h1 = __uint_as_float(__float_as_uint(f[2 * p + 1]) & 0xFFFFE000u);
        const float2 l = ptx::fsub2(make_float2(f[2 * p], f[2 * p + 1]), make_float2(h0, h1));
        hi[idx] = __float_as_uint(h0);
        hi[idx + 1] = __float_as_uint(h1);
        lo[idx] = __float_as_uint(l.x);
        lo[idx + 1] = __float_as_uint(l.y);
      }
    }
}
// Both operand halves of a row pair at once: [h | m] hi into columns 0..63, lo
// into 64..127, two 64-column stores.
__device__ __forceinline__ void tmem_store_split2(uint32_t taddr, const float4 (&hs)[2][2], const float4 (&mm)[2][2]) {
  uint32_t hi[32], lo[32];
  split_regs(hs, reinterpret_cast<uint32_t(&)[16]>(hi[0]), reinterpret_cast<uint32_t(&)[16]>(lo[0]));
  split_regs(mm, reinterpret_cast<uint32_t(&)[16]>(hi[16]), reinterpret_cast<uint32_t(&)[16]>(lo[16]));
  ptx::tmem_st_16x256b_x8(taddr, hi);
  ptx::tmem_st_16x256b_x8(taddr + 64, lo);
}
__device__ __forceinline__ void tmem_store_split(uint32_t taddr, const float4 (&x)[2][2]) {
  uint32_t hi[16], lo[16];
#pragma unroll
  for (int h = 0; h < 2; ++h)
#pragma unroll
    for (int c = 0; c < 2; ++c) {
      const float f[4] = {x[h][c].x, x[h][c].y, x[h][c].z, x[h][c].w};
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const int idx = 4 * (2 * c + p) + 2 * h;  // features 4c+2p, 4c+2p+1
        const float h0 = __uint_as_float(__float_as_uint(f[2 * p]) & 0xFFFFE000u);
        const float h1 = __uint_as_float(__float_as_uint(f[2 * p + 1]) & 0xFFFFE000u);
        const float2 l = ptx::fsub2(make_float2(f[2 * p], f[2 * p + 1]), make_float2(h0, h1));
        hi[idx] = __float_as_uint(h0);
        hi[idx + 1] = __float_as_uint(h1);
        lo[idx] = __float_as_uint(l.x);
        lo[idx + 1] = __float_as_uint(l.y);
      }
    }
  ptx::tmem_st_16x256b_x4(taddr, hi);
  ptx::tmem_st_16x256b_x4(taddr + 64, lo);
}

struct LayerArgs {
  uint32_t n;
  const uint32_t* rp;
  const uint32_t* col;
  const float* hin;      // n x 32
  float* hout;           // n x 32 (layer mode)
  const uint32_t* bimg;  // 16 KB swizzled W image (hi/lo), K and N permuted by kcol_feature
  HdInfo hd;
  uint32_t classes;
  uint8_t* cls;          // last layer: n classes
  float* logits;         // last layer: n x classes (optional)
  // tile plan (tile_plan.cuh)
  const TileMeta* tmeta;
  const uint16_t* lrp;
  const uint16_t* lcol;
  const uint32_t* halo;
  const unsigned long long* rec;  // row records (tiles x 128), tile_plan.cuh
  float* spmm_out;       // SpMM mode: n x 32 neighbour means (LD rows)
  unsigned long long* trace;  // diagnostic timeline of CTA 0 (GROOT_TRACE): [64 tiles][16 clock64 stamps]
  uint32_t plan_period;       // > 0: the plan is one copy's (tiles 0..period-1), tile t uses t % period
  uint32_t period_rows;       //      and its halo rows shift by (t / period) * period_rows
  uint32_t* tile_counter;     // dynamic tile scheduler (zeroed before the launch); null: static b + i*G
  uint32_t tile_begin, tile_end;  // tiles [tile_begin, tile_end) of this launch
  const float* ktable_self;   // kModeXform: Ts (entry rows . W_self + b)
  const uint32_t* hbimg;      // kModeLast: 4 KB W_out image (hi/lo), K permuted by kcol_feature, N padded to 16
  float head_cert;            // kModeLast, GROOT_HEAD_CERT: scale of the margin bound (1; huge = every row exact)
  const uint8_t* keys;        // keyed layer 1: u8 entry id per row (hin unused; tiles x 128), see l0_key_kernel
  const uint8_t* hids;        //                entry ids of the halo rows (tiles x kTpHaloCap, as the halo list)
  const float* ktable;        //                kTkTableRows x 32 rows of the entries
};

// Timeline stamp of CTA 0 for tile iteration it (< 64), event slot k (< 16).
// Compiled in only with -DGROOT_TRACE_BUILD (the stamps cost registers).
#ifdef GROOT_TRACE_BUILD
constexpr bool kTraceOn = true;
#else
constexpr bool kTraceOn = false;
#endif
__device__ __forceinline__ void tstamp(unsigned long long* tr, uint32_t it, int k) {
  if (kTraceOn && tr && blockIdx.x == 0 && it < 60) tr[it * 16 + k] = clock64();
}

// ---------------------------------------------------------------------------
// Tile-planned fused layer / SpMM. Shared memory holds two rings:
//   plan ring  (kTkMetaStages x ~3 KB): a tile's row offsets, local slots and
//              halo list; issued kTkMetaLead tiles ahead of the rows, so the
//              halo list is there when the tile's rows are fetched;
//   row ring   (kTkRowStages x 36 KB): rows 0..127 = the tile (TMA box),
//              rows 128.. = its halo (cp.async by the copier warps).
// Rows are stored unswizzled. Lane j of a row's 4-lane group reads the 32 B
// of features 8j..8j+7 as two 16-B loads; groups of odd parity issue the two
// halves in the opposite order, so the two rows served in one 8-lane phase
// always touch disjoint banks (even vs odd 16-B chunks) whatever the rows
// are. Their accumulators are swapped back once per row.
// ---------------------------------------------------------------------------
// kModeXform (keyed layer 1 of a model with more layers): transform first.
// mean(H1[N(v)]) . Wn = mean over u of (table[id_u] . Wn), so with the entry
// table transformed once (Tn = table . Wn, Ts = table . Ws; <= 255 rows) the
// layer is a gather-sum of 32-wide rows: relu(Ts[id_v] + mean Tn[id_u] + b),
// stored by the producers as in SpMM mode -- no tensor-core pass.
enum TileMode { kModeLayer = 0, kModeLast = 1, kModeSpmm = 2, kModeXform = 3 };
constexpr int kTkMetaStages = 8;
constexpr uint32_t kCopiersMma = 2;   // warps 14, 15
constexpr uint32_t kCopiersSpmm = 2;  // warps 14, 15 (7 copiers measured no faster)
constexpr uint32_t kTkRowBytes = (kTpRows + kTpHaloCap) * 128u;
constexpr uint32_t kTkLrpOff = 0;
constexpr uint32_t kTkLcolOff = kTpLrp * 2u + 16u;
constexpr uint32_t kTkHaloOff = kTkLcolOff + kTpColCap * 2u;
constexpr uint32_t kTkKidOff = kTkHaloOff + kTpHaloCap * 4u;  // keyed: entry ids of the tile rows
constexpr uint32_t kTkHidOff = kTkKidOff + kTpRows;             //        and of the halo rows
constexpr uint32_t kTkRecOff = kTkHidOff + kTpHaloCap;           // row records (8 B per tile row)
constexpr uint32_t kTkMetaBytes = ((kTkRecOff + kTpRows * 8u + 127u) / 128u) * 128u;
#ifndef GROOT_GRAB
#define GROOT_GRAB 8
#endif
// Poll intervals (ns) of the waits off the critical path (ptx::mbar_wait_poll);
// 0 = the previous forms (spinning loader, suspend-hint epilogue).
#ifndef GROOT_EPI_POLL_NS
#define GROOT_EPI_POLL_NS 0
#endif
#ifndef GROOT_LOAD_POLL_NS
#define GROOT_LOAD_POLL_NS 0
#endif
constexpr uint32_t kTileRing = 32;     // tile ids of the CTA's iterations (dynamic scheduler)
constexpr uint32_t kEndTile = 0xFFFFFFFFu;
constexpr uint32_t kTkTableRows = 256;  // keyed layer 1: entry rows (ids are u8)
#ifndef GROOT_ST_X8
#define GROOT_ST_X8 1  // producers store [h | m] hi and lo with two 64-column tcgen05.st (x8) instead of four x4
#endif
#ifndef GROOT_XFORM_SELF_PARITY
#define GROOT_XFORM_SELF_PARITY 1  // transform-first layer: self (Ts) rows in lane-group parity order (-1 %)
#endif
#ifndef GROOT_ROW_STAGES
#define GROOT_ROW_STAGES 4
#endif

// Shared-memory plan per variant: staged-row kernels spend it on the row ring,
// keyed kernels stage no rows (no row ring: the copier warps translate the
// plan's row records into entry-row offsets) and hold the entry tables. (5 row
// stages fit only with the plan lead cut to 3 tiles: measured 2 % slower.)
#ifndef GROOT_KEYED_META
#define GROOT_KEYED_META 8
#endif
#ifndef GROOT_KEYED_ROWS
#define GROOT_KEYED_ROWS 4
#endif
template <bool kKeyed>
struct TkCfg {
  static constexpr int kRowStages = kKeyed ? GROOT_KEYED_ROWS : GROOT_ROW_STAGES;
  static constexpr int kMetaStages = kKeyed ? GROOT_KEYED_META : kTkMetaStages;  // keyed: deeper plan ring
  static constexpr int kMetaLead = kMetaStages - kRowStages;
  static constexpr uint32_t kRowMem = kKeyed ? 0u : kRowStages * kTkRowBytes;
  static constexpr uint32_t kTableMem = kKeyed ? 2u * kTkTableRows * 128u : 0u;  // entry rows (Tn) | Ts
  static constexpr uint32_t kSmem = kRowMem + kMetaStages * kTkMetaBytes + kTableMem + kBBytes + kHeadBBytes +
                                    (256 + 32 + kTileRing) * 4 + 16 * kMetaStages +
                                    8 * (2 * kStages + 6 + 2 * kRowStages + 3 * kMetaStages) + 16 + 1024;
  static_assert(kMetaLead + kRowStages + kStages + 4 < static_cast<int>(kTileRing), "tile ring covers every role's lag");
  static_assert(kSmem <= 232448, "tile kernel exceeds the 227 KB shared-memory limit");
  static_assert(kMetaLead >= 2, "plan records lead the rows");
};
static_assert(kTkRowBytes % 1024 == 0, "row stages keep 1024-B alignment");
static_assert(kTkLcolOff % 16 == 0 && kTkHaloOff % 16 == 0 && kTkKidOff % 16 == 0 && kTkHidOff % 16 == 0 &&
                  kTkRecOff % 16 == 0 &&
                  kTpHaloCap % 16 == 0,
              "bulk-copy destinations and keyed halo-id sources must be 16-B aligned");

__device__ __forceinline__ void acc_row(float2 (&m)[4], const float4& x0, const float4& x1) {
  m[0] = ptx::fadd2(m[0], make_float2(x0.x, x0.y));
  m[1] = ptx::fadd2(m[1], make_float2(x0.z, x0.w));
  m[2] = ptx::fadd2(m[2], make_float2(x1.x, x1.y));
  m[3] = ptx::fadd2(m[3], make_float2(x1.z, x1.w));
}
__device__ __forceinline__ void swap_halves(float2 (&m)[4], bool sw) {
  if (sw) {
    const float2 t0 = m[0], t1 = m[1];
    m[0] = m[2];
    m[1] = m[3];
    m[2] = t0;
    m[3] = t1;
  }
}

template <int kMode, bool kKeyed = false>
__global__ void __launch_bounds__(kThreads, 1) sage_tile_kernel(const LayerArgs a, const HeadW hw,
                                                                const __grid_constant__ CUtensorMap tmap_in) {
  constexpr bool kMma = kMode == kModeLayer || kMode == kModeLast;
  constexpr uint32_t kAccBufs = kMode == kModeLast && !GROOT_LAST_ACC2 ? 1u : 2u;  // last layer: see kHeadHiCol
  constexpr bool kXform = kMode == kModeXform;
  static_assert(!kXform || kKeyed, "transform-first mode reads the entry tables");
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (ptx::smem_addr(smem_raw) & 1023u)) & 1023u);
  using Cfg = TkCfg<kKeyed>;
  constexpr int kTkMetaStages = Cfg::kMetaStages;
  constexpr int kTkRowStages = Cfg::kRowStages;
  constexpr int kTkMetaLead = Cfg::kMetaLead;
  uint8_t* sRows = smem;                                 // [kTkRowStages] tile + halo rows (none when keyed)
  uint8_t* sPlan = sRows + Cfg::kRowMem;                 // [kTkMetaStages] lrp | lcol | halo list
  uint8_t* sTable = sPlan + kTkMetaStages * kTkMetaBytes;  // keyed layer 1: entry rows
  uint8_t* sB = sTable + Cfg::kTableMem;
  uint8_t* sHB = sB + kBBytes;                            // head W_out image (last layer)
  float* sInv = reinterpret_cast<float*>(sHB + kHeadBBytes);  // 1/d, d < 256
  float* sBias = sInv + 256;                              // layer bias by output feature
  uint32_t* sTile = reinterpret_cast<uint32_t*>(sBias + 32);  // [kTileRing] tile of iteration i (kEndTile: done)
  uint4* sMeta = reinterpret_cast<uint4*>(sTile + kTileRing);  // [kTkMetaStages] TileMeta of the staged plan
  uint64_t* bars = reinterpret_cast<uint64_t*>(sMeta + kTkMetaStages);
  uint64_t* full = bars;                     // [kStages] producers -> MMA (A operand in TMEM)
  uint64_t* empty = full + kStages;          // [kStages] MMA done reading the A stage
  uint64_t* tfull = empty + kStages;         // [2] accumulator ready
  uint64_t* tempty = tfull + 2;              // [2] accumulator drained
  uint64_t* m_full = tempty + 2;             // [kTkMetaStages] plan records landed
  uint64_t* m_empty = m_full + kTkMetaStages;
  uint64_t* r_full = m_empty + kTkMetaStages;  // [kTkRowStages] tile + halo rows landed
  uint64_t* r_empty = r_full + kTkRowStages;
  uint64_t* m_ready = r_empty + kTkRowStages;  // [kTkMetaStages] keyed: the plan's row records translated to entry rows
  uint64_t* hdone = m_ready + kTkMetaStages;  // last layer: head MMA of the current tile complete
  uint64_t* hready = hdone + 1;              // last layer: the head's A operand is in TMEM (epilogue -> MMA warp)
  uint32_t* sTmem = reinterpret_cast<uint32_t*>(hready + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t n = a.n;
  const uint32_t ntiles = (n + kTileM - 1) / kTileM;
  const uint32_t G = gridDim.x;
  constexpr uint32_t kCopiers = kMma ? kCopiersMma : kCopiersSpmm;

  if (kMma)
    for (uint32_t i = threadIdx.x; i < kBBytes / 16; i += kThreads)
      reinterpret_cast<uint4*>(sB)[i] = __ldg(reinterpret_cast<const uint4*>(a.bimg) + i);
  if (kMode == kModeLast)
    for (uint32_t i = threadIdx.x; i < kHeadBBytes / 16; i += kThreads)
      reinterpret_cast<uint4*>(sHB)[i] = __ldg(reinterpret_cast<const uint4*>(a.hbimg) + i);
  // the zero row of the row records: entry 255 of the keyed table (entry ids
  // are < kDictCap = 255), the last halo slot of every row stage otherwise
  if (kKeyed)
    for (uint32_t i = threadIdx.x; i < kTkTableRows * 8; i += kThreads)
      reinterpret_cast<uint4*>(sTable)[i] =
          i >= (kTkTableRows - 1) * 8 ? make_uint4(0, 0, 0, 0) : __ldg(reinterpret_cast<const uint4*>(a.ktable) + i);
  else
    for (uint32_t i = threadIdx.x; i < kTkRowStages * 8; i += kThreads)
      reinterpret_cast<uint4*>(sRows + (i >> 3) * kTkRowBytes + kTpZeroSlot * 128u)[i & 7] = make_uint4(0, 0, 0, 0);
  if (kXform)
    for (uint32_t i = threadIdx.x; i < kTkTableRows * 8; i += kThreads)
      reinterpret_cast<uint4*>(sTable + kTkTableRows * 128)[i] = __ldg(reinterpret_cast<const uint4*>(a.ktable_self) + i);
  for (uint32_t d = threadIdx.x; d < 256; d += kThreads) sInv[d] = d ? 1.0f / static_cast<float>(d) : 0.0f;
  if (kMma || kXform) {
    for (uint32_t i = threadIdx.x; i < 32; i += kThreads) sBias[i] = hw.bias[i];
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&full[s], kProdWarps * 32);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      ptx::mbar_init(&tfull[s], 1);
      ptx::mbar_init(&tempty[s], kEpiWarps * 32);
    }
    for (int s = 0; s < kTkMetaStages; ++s) {
      ptx::mbar_init(&m_full[s], 1);
      ptx::mbar_init(&m_ready[s], 32 * kCopiers);
      ptx::mbar_init(&m_empty[s], kProdWarps * 32);
    }
    for (int s = 0; s < kTkRowStages; ++s) {
      ptx::mbar_init(&r_full[s], 1 + 32 * kCopiers);  // TMA box (expect_tx) + each copier lane's cp.async arrival
      ptx::mbar_init(&r_empty[s], kProdWarps * 32);
    }
    ptx::mbar_init(hdone, 1);
    ptx::mbar_init(hready, kEpiWarps * 32);
    ptx::mbar_fence_init();
  }
  if (kMma && warp == kMmaWarp) ptx::tmem_alloc<kTmemCols>(sTmem);
  ptx::fence_proxy_async_smem();
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  const uint32_t tmem_base = kMma ? *sTmem : 0u;

  // halo copier warps: the two spare warps 14, 15
  static_assert(kCopiersMma == 2 && kCopiersSpmm == 2, "copier warps are 14 and 15");
  const int copier = warp > kLoadWarp ? warp - (kLoadWarp + 1) : -1;
  if (warp == kLoadWarp) {
    // ===== loader: plan records and tile rows (one lane) =====
    if (lane == 0) {
      // Tiles are handed out by a global counter (all CTAs work on one
      // contiguous window of tiles, which keeps the halo rows of neighbouring
      // tiles L2-resident), kTkMetaLead + kQ iterations ahead of the rows. The
      // tile of iteration i is published in sTile[i % kTileRing] before the
      // plan of iteration i completes m_full; the first tile past the end is
      // published as kEndTile and ends every role's loop.
      constexpr int kQ = 4;  // TileMeta records prefetched into registers beyond the plan ring
      // one atomic per kGrab consecutive tiles (measured: 1 -> SpMM +20 %, 8 best)
      constexpr uint32_t kGrab = GROOT_GRAB;
      uint32_t grabbed = 0, chunk = 0;
      auto grab = [&]() -> uint32_t {
        uint32_t t;
        if (a.tile_counter) {
          if (grabbed % kGrab == 0) chunk = atomicAdd(a.tile_counter, kGrab);
          t = a.tile_begin + chunk + grabbed % kGrab;
        } else {
          t = a.tile_begin + blockIdx.x + grabbed * G;
        }
        ++grabbed;
        return t < a.tile_end ? t : kEndTile;
      };
      auto meta_of = [&](uint32_t tt) -> uint4 {
        if (tt == kEndTile) return make_uint4(0, 0, 0, 0);
        const uint32_t pt = a.plan_period ? tt % a.plan_period : tt;
        return __ldg(reinterpret_cast<const uint4*>(a.tmeta) + pt);
      };
      bool end_published = false;
      auto issue_plan = [&](uint32_t i, uint32_t t, const uint4& m) {
        if (end_published) return;
        const uint32_t ms = i % kTkMetaStages;
        if (GROOT_LOAD_POLL_NS) ptx::mbar_wait_poll(&m_empty[ms], ((i / kTkMetaStages) & 1) ^ 1, GROOT_LOAD_POLL_NS);
        else ptx::mbar_wait(&m_empty[ms], ((i / kTkMetaStages) & 1) ^ 1);
        sTile[i % kTileRing] = t;
        if (t == kEndTile) {
          end_published = true;
          sMeta[ms] = make_uint4(0, 0, 0, 0);
          ptx::mbar_arrive(&m_full[ms]);
          return;
        }
        uint8_t* sp = sPlan + ms * kTkMetaBytes;
        sMeta[ms] = m;
        const bool slow = (m.w & kTpSlow) != 0;
        const uint32_t hpad = (slow || kKeyed) ? 0u : (m.w + 3u) & ~3u;  // keyed: halo ids instead of rows
        const uint32_t kpad = kKeyed ? (slow ? 0u : (m.w + 15u) & ~15u) : 0u;
        // row offsets and slot list only for tiles with rows of degree > 4 (m.z > 0)
        ptx::mbar_arrive_expect_tx(&m_full[ms], (m.z ? kTpLrp * 2u + m.z * 2u : 0u) + hpad * 4u + (kKeyed ? kTpRows + kpad : 0u) +
                                                    (slow ? 0u : kTpRows * 8u));
        if (kKeyed) {
          ptx::bulk_load(sp + kTkKidOff, a.keys + static_cast<size_t>(t) * kTpRows, kTpRows, &m_full[ms]);
          if (kpad) ptx::bulk_load(sp + kTkHidOff, a.hids + static_cast<size_t>(t) * kTpHaloCap, kpad, &m_full[ms]);
        }
        const uint32_t pt = a.plan_period ? t % a.plan_period : t;
        if (m.z) {
          ptx::bulk_load(sp + kTkLrpOff, a.lrp + static_cast<size_t>(pt) * kTpLrp, kTpLrp * 2u, &m_full[ms]);
          ptx::bulk_load(sp + kTkLcolOff, a.lcol + m.x, m.z * 2u, &m_full[ms]);
        }
        if (hpad) ptx::bulk_load(sp + kTkHaloOff, a.halo + m.y, hpad * 4u, &m_full[ms]);
        if (!slow)  // (keyed: translated to entry rows by the copier warps)
          ptx::bulk_load(sp + kTkRecOff, a.rec + static_cast<size_t>(pt) * kTpRows, kTpRows * 8u, &m_full[ms]);
      };
      uint32_t rows_tile[kTkMetaLead];  // tiles of iterations it .. it + kTkMetaLead - 1
      for (int i = 0; i < kTkMetaLead; ++i) {
        rows_tile[i] = grab();
        issue_plan(i, rows_tile[i], meta_of(rows_tile[i]));
      }
      uint32_t qid[kQ];
      uint4 q[kQ];
#pragma unroll
      for (int k = 0; k < kQ; ++k) {
        qid[k] = grab();
        q[k] = meta_of(qid[k]);
      }
      for (uint32_t it = 0;; ++it) {
        const uint32_t t = rows_tile[0];
        // plan records of iteration it + kTkMetaLead
        const uint32_t tl = qid[0];
        const uint4 mq = q[0];
#pragma unroll
        for (int k = 0; k + 1 < kQ; ++k) {
          qid[k] = qid[k + 1];
          q[k] = q[k + 1];
        }
        qid[kQ - 1] = grab();
        q[kQ - 1] = meta_of(qid[kQ - 1]);
        issue_plan(it + kTkMetaLead, tl, mq);
#pragma unroll
        for (int k = 0; k + 1 < kTkMetaLead; ++k) rows_tile[k] = rows_tile[k + 1];
        rows_tile[kTkMetaLead - 1] = tl;
        if (t == kEndTile) break;
        // rows of iteration it
        if (kKeyed) continue;  // keyed: no rows (the producers read the entry table)
        const uint32_t rs = it % kTkRowStages;
        if (GROOT_LOAD_POLL_NS) ptx::mbar_wait_poll(&r_empty[rs], ((it / kTkRowStages) & 1) ^ 1, GROOT_LOAD_POLL_NS);
        else ptx::mbar_wait(&r_empty[rs], ((it / kTkRowStages) & 1) ^ 1);
        tstamp(a.trace, it, 0);
        ptx::mbar_arrive_expect_tx(&r_full[rs], kTpRows * 128u);
        ptx::tma_load_2d(&tmap_in, sRows + rs * kTkRowBytes, &r_full[rs], 0, static_cast<int32_t>(t * kTileM));
      }
    }
    __syncwarp();
  } else if (copier >= 0 && kKeyed) {
    // ===== keyed layers (no rows to stage): the copier warps translate each
    // plan stage's row records in place, local slot byte offsets -> entry-row
    // byte offsets (the zero slot -> entry kTkTableRows - 1, kept zero), a few
    // tiles ahead of the producers =====
    const uint32_t gl = static_cast<uint32_t>(copier) * 32u + lane;
    for (uint32_t it = 0;; ++it) {
      const uint32_t ms = it % kTkMetaStages;
      ptx::mbar_wait_sleep(&m_full[ms], (it / kTkMetaStages) & 1, 100);
      if (sTile[it % kTileRing] == kEndTile) {
        ptx::mbar_arrive(&m_ready[ms]);  // the producers see the end through m_ready
        break;
      }
      if (!(sMeta[ms].w & kTpSlow)) {
        uint8_t* sp = sPlan + ms * kTkMetaBytes;
        uint32_t* rw = reinterpret_cast<uint32_t*>(sp + kTkRecOff);
        const uint8_t* kid = sp + kTkKidOff;  // entry ids of the tile rows, then of the halo rows
        auto map = [&](uint32_t f) -> uint32_t {
          const uint32_t sl = f >> 7;
          return ((sl == kTpZeroSlot ? kTkTableRows - 1u : static_cast<uint32_t>(kid[sl])) << 7) | (f & 0x7Fu);
        };
#pragma unroll 4
        for (uint32_t k = gl; k < 2 * kTpRows; k += 32 * kCopiers) {
          const uint32_t w = rw[k];
          rw[k] = map(w & 0xFFFFu) | (map(w >> 16) << 16);
        }
        // the stage is refilled by bulk copies (async proxy) once the producers
        // release it: order these generic-proxy writes before that
        ptx::fence_proxy_async_smem();
      }
      ptx::mbar_arrive(&m_ready[ms]);
    }
  } else if (copier >= 0) {
    // ===== halo copiers: 16-B cp.async per lane, 8 lanes per row =====
    const uint32_t sRows_s = ptx::smem_addr(sRows);
    const uint32_t gl = static_cast<uint32_t>(copier) * 32u + lane;
    const uint32_t c = gl & 7, s0 = gl >> 3;
    constexpr uint32_t kStride = kCopiers * 4u;  // rows per pass of all copier lanes
    for (uint32_t it = 0;; ++it) {
      const uint32_t rs = it % kTkRowStages, ms = it % kTkMetaStages;
      ptx::mbar_wait_sleep(&m_full[ms], (it / kTkMetaStages) & 1, 100);
      const uint32_t t = sTile[it % kTileRing];
      if (t == kEndTile) break;
      ptx::mbar_wait_sleep(&r_empty[rs], ((it / kTkRowStages) & 1) ^ 1, 100);
      const uint32_t hc = sMeta[ms].w;
      if (gl == 0) tstamp(a.trace, it, 1);
      if (!(hc & kTpSlow)) {
        const uint32_t shift = a.plan_period ? (t / a.plan_period) * a.period_rows : 0u;
        const float* hin_c = a.hin + static_cast<size_t>(shift) * kF + 4 * c;
        const uint32_t* hl = reinterpret_cast<const uint32_t*>(sPlan + ms * kTkMetaBytes + kTkHaloOff);
        const uint32_t sbase = sRows_s + rs * kTkRowBytes + kTpRows * 128u + c * 16u;
        // 4 halo ids per batch read before the copies are issued (the asm
        // memory clobber would otherwise serialise each LDS behind a copy)
        for (uint32_t b0 = s0; b0 < hc; b0 += 4 * kStride) {
          uint32_t row[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) row[u] = b0 + u * kStride < hc ? hl[b0 + u * kStride] : 0u;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const uint32_t slot = b0 + u * kStride;
            if (slot < hc) ptx::cp_async16(sbase + slot * 128u, hin_c + static_cast<size_t>(row[u]) * kF);
          }
        }
      }
      if (gl == 0) tstamp(a.trace, it, 2);
      ptx::cp_async_mbar_arrive(ptx::smem_addr(&r_full[rs]));
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  } else if (kMma && warp == kMmaWarp) {
    // ===== MMA issuer: the whole warp runs the loop (warp-uniform operands
    // stay in uniform registers), one elected lane issues =====
    constexpr uint32_t idesc = ptx::idesc_tf32<kTileM, kF>();
    const uint32_t b0s = ptx::smem_addr(sB);
    // the previous tile's 32 -> classes head, once the epilogue has put its A
    // operand (relu(acc + b) split into TF32 hi / lo) into TMEM
    auto issue_head = [&](uint32_t it) {
        ptx::mbar_wait(hready, (it - 1) & 1);
        ptx::tc_fence_after();
        if (ptx::elect_one()) {
          constexpr uint32_t hdesc = ptx::idesc_tf32<kTileM, kHeadN>();
          const uint32_t ahi = tmem_base + kHeadHiCol, alo = tmem_base + kHeadLoCol;
          const uint32_t hb = ptx::smem_addr(sHB);
#pragma unroll
          for (uint32_t kk = 0; kk < 4; ++kk) {
            const uint64_t bhi = ptx::umma_desc_sw128(hb + kk * 32), blo = ptx::umma_desc_sw128(hb + kHeadN * 128 + kk * 32);
            ptx::mma_tf32_ts(tmem_base + kHeadDCol, ahi + kk * 8, bhi, hdesc, kk != 0);
            ptx::mma_tf32_ts(tmem_base + kHeadDCol, ahi + kk * 8, blo, hdesc, 1);
            if (!GROOT_HEAD_CERT) ptx::mma_tf32_ts(tmem_base + kHeadDCol, alo + kk * 8, bhi, hdesc, 1);
          }
          ptx::mma_commit(hdone);
        }
        __syncwarp();
    };
    for (uint32_t it = 0;; ++it) {
      const uint32_t s = it % kStages, ph = (it / kStages) & 1;
      const uint32_t acc = kAccBufs == 2 ? (it & 1) : 0u, aph = kAccBufs == 2 ? ((it >> 1) & 1) : (it & 1);
      // GROOT_LAST_PIPE: tile it's layer MMAs go first (the accumulator is free
      // once the epilogue has loaded tile it-1), the head of it-1 after them,
      // while the epilogue works on the split
      if (kMode == kModeLast && !GROOT_HEAD_AFTER_MMA && it > 0) issue_head(it);
      ptx::mbar_wait(&full[s], ph);
      if (lane == 0) tstamp(a.trace, it, 8);
      ptx::mbar_wait(&tempty[acc], aph ^ 1);
      if (sTile[it % kTileRing] == kEndTile) {  // producers' end hand-over: wake the epilogue and stop
        if (kMode == kModeLast && GROOT_HEAD_AFTER_MMA && it > 0) issue_head(it);
        if (lane == 0) ptx::mbar_arrive(&tfull[acc]);
        break;
      }
      if (lane == 0) tstamp(a.trace, it, 9);
      ptx::tc_fence_after();
      if (ptx::elect_one()) {
        const uint32_t d = tmem_base + kAccCol0 + acc * kAccCols;
        const uint32_t as = tmem_base + s * kStageCols;
#pragma unroll
        for (uint32_t kb = 0; kb < 2; ++kb)
#pragma unroll
          for (uint32_t kk = 0; kk < 4; ++kk) {
            const uint32_t ahi = as + kb * 32 + kk * 8;  // h (kb 0) or m (kb 1), K = 8 columns
            const uint32_t bo = b0s + kb * 8192 + kk * 32;
            const uint64_t bhi = ptx::umma_desc_sw128(bo), blo = ptx::umma_desc_sw128(bo + 4096);
            const uint32_t first = (kb | kk) != 0;
            ptx::mma_tf32_ts(d, ahi, bhi, idesc, first);
            ptx::mma_tf32_ts(d, ahi, blo, idesc, 1);
            ptx::mma_tf32_ts(d, ahi + 64, bhi, idesc, 1);
          }
        ptx::mma_commit(&empty[s]);
        ptx::mma_commit(&tfull[acc]);
      }
      __syncwarp();
      if (kMode == kModeLast && GROOT_HEAD_AFTER_MMA && it > 0) issue_head(it);
      if (lane == 0) tstamp(a.trace, it, 10);
    }
  } else if (warp >= kEpiWarps && warp < kMmaWarp) {
    // ===== producers: 8 warps x 16 rows. Warp w may only reach its TMEM
    // lane quadrant (w % 4): it owns tile rows 32(w%4) + 16h' .. +15 with
    // h' = (w-4)/4; lane group r = lane/4 owns rows r and r+8 of that slice,
    // lane j = lane%4 features 8j..8j+7 — the registers a 16x256b tcgen05.st
    // takes (A's K order permuted to match, kcol_feature) =====
    const uint32_t lbase = (warp & 3) * 32 + ((warp - kEpiWarps) >> 2) * 16;
    const uint32_t j = lane & 3;
    const uint32_t gp = (lane >> 2) & 1;                   // lane group parity: which half is read first
    // (natural half order instead, i.e. 2-way conflicts on the neighbour reads: +21 %)
    const uint32_t off0 = (2u * j + gp) * 16u, off1 = (2u * j + 1u - gp) * 16u;
    const uint32_t li = lbase + (lane >> 2);  // tile rows li and li + 8
    const uint32_t thr = a.hd.threshold;
    const float* hin_j = a.hin + 8 * j;
    unsigned long long wt0 = 0, wt1 = 0, wt2 = 0, wt3 = 0;
    unsigned long long acc_rows = 0, acc_gather = 0, acc_wait = 0, acc_store = 0;
    // The A stage of tile i is handed to the MMA (tcgen05.wait::st, fence,
    // arrive) after the gather of tile i + 1: the TMEM stores complete behind
    // the next tile's shared-memory reads instead of stalling the warp.
    uint32_t pend = kStages;  // stage with stores in flight (kStages: none)
    auto hand_over = [&]() {
      if (kMma && pend < kStages) {
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        ptx::mbar_arrive(&full[pend]);
        pend = kStages;
      }
    };
    for (uint32_t it = 0;; ++it) {
      const uint32_t rs = it % kTkRowStages, ms = it % kTkMetaStages;
      unsigned long long* tr = (warp == kEpiWarps && lane == 0) ? a.trace : nullptr;
      unsigned long long* tr7 = (warp == kEpiWarps + 3 && lane == 0) ? a.trace : nullptr;
      tstamp(tr, it, 3);
      tstamp(tr7, it, 13);
      if (kTraceOn) wt0 = clock64();
      ptx::mbar_wait(kKeyed ? &m_ready[ms] : &m_full[ms], (it / kTkMetaStages) & 1);
      const uint32_t t = sTile[it % kTileRing];
      if (t == kEndTile) {  // hand the MMA an empty stage so it sees the end too
        hand_over();
        if (kMma) {
          const uint32_t s = it % kStages;
          ptx::mbar_wait(&empty[s], ((it / kStages) & 1) ^ 1);
          ptx::mbar_arrive(&full[s]);
        }
        if (kTraceOn && a.trace && blockIdx.x == 0 && lane == 0) {  // per-warp totals: trace rows 60..61
          unsigned long long* tw = a.trace + 60 * 16 + (warp - kEpiWarps) * 4;
          tw[0] = acc_rows;
          tw[1] = acc_gather;
          tw[2] = acc_wait;
          tw[3] = acc_store;
        }
        break;
      }
      const uint32_t row0 = t * kTileM;
      if (!kKeyed) ptx::mbar_wait(&r_full[rs], (it / kTkRowStages) & 1);
      tstamp(tr, it, 4);
      if (kTraceOn) wt1 = clock64();
      const uint8_t* st = sRows + rs * kTkRowBytes;
      const uint8_t* sp = sPlan + ms * kTkMetaBytes;
      // neighbour rows: staged rows, or (keyed) entry rows: the keyed row
      // records hold entry-row offsets (l0_halo_ids_kernel)
      const uint8_t* rbase = kKeyed ? sTable : st;
      const bool slow = (sMeta[ms].w & kTpSlow) != 0;
      float2 m[2][4];
      uint32_t d[2];
      bool hd[2];
      float inv[2];
      float4 hs[2][2], mm[2][2];
#pragma unroll
      for (int h = 0; h < 2; ++h)
#pragma unroll
        for (int q = 0; q < 4; ++q) m[h][q] = make_float2(0.f, 0.f);
      if (!slow) {
        const uint16_t* lr = reinterpret_cast<const uint16_t*>(sp + kTkLrpOff);
        const uint16_t* lc = reinterpret_cast<const uint16_t*>(sp + kTkLcolOff);
        // one record per row: its first four neighbour slots as byte offsets
        // (unused ones -> the zero row), so every row's neighbour reads are
        // issued together, branch-free, right after one shared-memory load
        uint2 rr[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          rr[h] = *reinterpret_cast<const uint2*>(sp + kTkRecOff + (li + 8 * h) * 8u);
          hd[h] = (rr[h].x & kTpRecHd) != 0;
          d[h] = tp_rec_degree(rr[h].x);
          inv[h] = sInv[d[h]];
        }
        if (kMma || kXform) {
          const uint8_t* sself = kXform ? sTable + kTkTableRows * 128 : sTable;  // Ts, or the entry rows
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const uint8_t* rowp = kKeyed ? sself + sp[kTkKidOff + li + 8 * h] * 128u : st + (li + 8 * h) * 128u;
            if (kXform && GROOT_XFORM_SELF_PARITY) {
              // lane-group parity order (conflict-free like the neighbour reads), swapped back
              const float4 f0 = ptx::lds_f4(ptx::smem_addr(rowp) + off0);
              const float4 f1 = ptx::lds_f4(ptx::smem_addr(rowp) + off1);
              hs[h][0] = gp ? f1 : f0;
              hs[h][1] = gp ? f0 : f1;
            } else {  // natural half order (rows li, li + 1 share banks: 2-way)
              hs[h][0] = ptx::lds_f4(ptx::smem_addr(rowp) + 32u * j);
              hs[h][1] = ptx::lds_f4(ptx::smem_addr(rowp) + 32u * j + 16u);
            }
          }
        }
        {
          // 16-B shared loads (ld.shared.v4: a float4 dereference of these
          // computed addresses compiles to pairs of 8-B loads)
          const uint32_t rb0 = ptx::smem_addr(rbase) + off0, rb1 = ptx::smem_addr(rbase) + off1;
          float4 x[2][kTpRecSlots][2];
#pragma unroll
          for (int h = 0; h < 2; ++h)
#pragma unroll
            for (uint32_t u = 0; u < kTpRecSlots; ++u) {
              const uint32_t w = u < 2 ? rr[h].x : rr[h].y;
              const uint32_t o = ((u & 1) ? (w >> 16) : w) & kTpRecOffMask;
              x[h][u][0] = ptx::lds_f4(rb0 + o);
              x[h][u][1] = ptx::lds_f4(rb1 + o);
            }
          // the sum starts at the first neighbour (0 + x is x, up to the sign of a zero)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            m[h][0] = make_float2(x[h][0][0].x, x[h][0][0].y);
            m[h][1] = make_float2(x[h][0][0].z, x[h][0][0].w);
            m[h][2] = make_float2(x[h][0][1].x, x[h][0][1].y);
            m[h][3] = make_float2(x[h][0][1].z, x[h][0][1].w);
#pragma unroll
            for (uint32_t u = 1; u < kTpRecSlots; ++u) acc_row(m[h], x[h][u][0], x[h][u][1]);
          }
        }
#pragma unroll
        for (int h = 0; h < 2; ++h)
          if (rr[h].x & kTpRecLong) {  // degree > 4 (rare in an AIG): the rest from the slot list
            const uint32_t lo = lr[li + 8 * h] & 0x7FFFu;
            const uint32_t rb = ptx::smem_addr(rbase);
            for (uint32_t k = kTpRecSlots; k < d[h]; ++k) {
              // (keyed: the slot's entry id, staged with the plan)
              const uint32_t o = rb + (kKeyed ? static_cast<uint32_t>(sp[kTkKidOff + lc[lo + k]]) : lc[lo + k]) * 128u;
              acc_row(m[h], ptx::lds_f4(o + off0), ptx::lds_f4(o + off1));
            }
          }
#pragma unroll
        for (int h = 0; h < 2; ++h) swap_halves(m[h], gp != 0);
      } else {
        uint32_t b[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint32_t r = row0 + li + 8 * h;
          b[h] = r < n ? __ldg(a.rp + r) : 0u;
          const uint32_t dd = r < n ? __ldg(a.rp + r + 1) - b[h] : 0u;
          hd[h] = dd >= thr;
          d[h] = hd[h] ? 0u : dd;
          inv[h] = sInv[d[h]];
        }
#pragma unroll
        for (int h = 0; h < 2; ++h)
          for (uint32_t k = 0; k < d[h]; ++k) {
            float4 x0, x1;
            const uint32_t cc = __ldg(a.col + b[h] + k);
            ptx::ldg_f8(kKeyed ? a.ktable + static_cast<size_t>(__ldg(a.keys + cc)) * kF + 8 * j
                               : hin_j + static_cast<size_t>(cc) * kF,
                        x0, x1);
            acc_row(m[h], x0, x1);
          }
      }
      if ((kMma || kXform) && slow) {
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const uint8_t* sself = kXform ? sTable + kTkTableRows * 128 : sTable;  // Ts, or the entry rows
          const uint8_t* rowp = kKeyed ? sself + sp[kTkKidOff + li + 8 * h] * 128u : st + (li + 8 * h) * 128u;
          hs[h][0] = ptx::lds_f4(ptx::smem_addr(rowp) + 32u * j);
          hs[h][1] = ptx::lds_f4(ptx::smem_addr(rowp) + 32u * j + 16u);
        }
      }
      tstamp(tr, it, 5);
      tstamp(tr7, it, 14);
      if (kTraceOn) wt2 = clock64();
      if (!kKeyed) ptx::mbar_arrive(&r_empty[rs]);
      ptx::mbar_arrive(&m_empty[ms]);
      hand_over();  // the previous tile's A stage
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const uint32_t r = row0 + li + 8 * h;
        if (hd[h]) {
          if (kMma || kXform) {
            const float* src = a.hd.mean + static_cast<size_t>(hd_slot(a.hd, r)) * kF + 8 * j;
            mm[h][0] = ptx::ldg_f4(src);
            mm[h][1] = ptx::ldg_f4(src + 4);
          }
        } else {
          const float2 iv = make_float2(inv[h], inv[h]);
#pragma unroll
          for (int q = 0; q < 4; ++q) m[h][q] = ptx::fmul2(m[h][q], iv);
          mm[h][0] = make_float4(m[h][0].x, m[h][0].y, m[h][1].x, m[h][1].y);
          mm[h][1] = make_float4(m[h][2].x, m[h][2].y, m[h][3].x, m[h][3].y);
        }
        if (kMode == kModeSpmm) {
          if (r < n && !hd[h]) ptx::stg_f8(a.spmm_out + static_cast<size_t>(r) * kF + 8 * j, mm[h][0], mm[h][1]);
        } else if (kXform) {
          if (r < n) {  // relu(Ts[id] + b + mean Tn): the bias is in the self table (l1_xform_kernel)
            const float2 s0 = ptx::fadd2(make_float2(hs[h][0].x, hs[h][0].y), make_float2(mm[h][0].x, mm[h][0].y));
            const float2 s1 = ptx::fadd2(make_float2(hs[h][0].z, hs[h][0].w), make_float2(mm[h][0].z, mm[h][0].w));
            const float2 s2 = ptx::fadd2(make_float2(hs[h][1].x, hs[h][1].y), make_float2(mm[h][1].x, mm[h][1].y));
            const float2 s3 = ptx::fadd2(make_float2(hs[h][1].z, hs[h][1].w), make_float2(mm[h][1].z, mm[h][1].w));
            const float4 o0 = make_float4(fmaxf(s0.x, 0.f), fmaxf(s0.y, 0.f), fmaxf(s1.x, 0.f), fmaxf(s1.y, 0.f));
            const float4 o1 = make_float4(fmaxf(s2.x, 0.f), fmaxf(s2.y, 0.f), fmaxf(s3.x, 0.f), fmaxf(s3.y, 0.f));
            ptx::stg_f8(a.hout + static_cast<size_t>(r) * kF + 8 * j, o0, o1);
          }
        } else if (r >= n) {
          hs[h][0] = hs[h][1] = mm[h][0] = mm[h][1] = make_float4(0.f, 0.f, 0.f, 0.f);
        }
      }
      if (kMma) {
        const uint32_t s = it % kStages, ph = (it / kStages) & 1;
        ptx::mbar_wait(&empty[s], ph ^ 1);
        tstamp(tr, it, 6);
        if (kTraceOn) wt3 = clock64();
        ptx::tc_fence_after();
        const uint32_t ta = tmem_base + (lbase << 16) + s * kStageCols;
#if GROOT_ST_X8
        tmem_store_split2(ta, hs, mm);  // columns 0..31 / 32..63 (hi: self, mean), 64..95 / 96..127 (lo)
#else
        tmem_store_split(ta, hs);       // columns 0..31 (hi), 64..95 (lo): self features
        tmem_store_split(ta + 32, mm);  // columns 32..63 (hi), 96..127 (lo): neighbour mean
#endif
        pend = s;                       // handed over after the next tile's gather
        tstamp(tr, it, 7);
        if (kTraceOn) {
          const unsigned long long wt4 = clock64();
          acc_rows += wt1 - wt0;
          acc_gather += wt2 - wt1;
          acc_wait += wt3 - wt2;
          acc_store += wt4 - wt3;
        }
        tstamp(tr7, it, 15);
      }
    }
  } else if (kMma && warp < kEpiWarps) {
    // ===== epilogue (4 warps, TMEM lane quadrant = warp). The weight image
    // permutes the output columns by kcol_feature, so a 16x256b load gives
    // lane j of a 4-lane group features 8j..8j+7 of two rows: whole 128-B
    // rows leave as 256-bit stores, no staging =====
    const uint32_t q = warp;
    const uint32_t j = lane & 3, r4 = lane >> 2;
    float b8[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) b8[k] = sBias[8 * j + k];
    // last layer: each lane's row's logits -> first maximum (and the logits)
    auto head_out = [&](uint32_t row, const float (&lg)[8]) {
      float best = 0.f;
      uint32_t arg = 0;
#pragma unroll
      for (int cl = 0; cl < kMaxClasses; ++cl) {
        if (cl < static_cast<int>(a.classes)) {
          const float sc = lg[cl] + hw.b[cl];
          if (cl == 0 || sc > best) { best = sc; arg = cl; }
          if (a.logits && row < n) a.logits[static_cast<size_t>(row) * a.classes + cl] = sc;
        }
      }
      if (row < n) a.cls[row] = static_cast<uint8_t>(arg);
    };
    uint32_t prev_row = 0;  // GROOT_LAST_PIPE: this lane's row of the tile whose head is in flight
    for (uint32_t e = 0;; ++e) {
      const uint32_t acc = kAccBufs == 2 ? (e & 1) : 0u, ph = kAccBufs == 2 ? ((e >> 1) & 1) : (e & 1);
      if (GROOT_EPI_POLL_NS) ptx::mbar_wait_poll(&tfull[acc], ph, GROOT_EPI_POLL_NS);
      else ptx::mbar_wait_sleep(&tfull[acc], ph, 200);
      const uint32_t t = sTile[e % kTileRing];
      if (t == kEndTile) {
        if (kMode == kModeLast && GROOT_LAST_PIPE && e > 0) {  // the last tile's head
          ptx::mbar_wait(hdone, (e - 1) & 1);
          ptx::tc_fence_after();
          float lg[8];
          ptx::tmem_ld_32x32b_x8(tmem_base + kHeadDCol + ((q * 32u) << 16), lg);
          head_out(prev_row, lg);
        }
        break;
      }
      if (warp == 0 && lane == 0) tstamp(a.trace, e, 11);
      ptx::tc_fence_after();
      const uint32_t tq = tmem_base + kAccCol0 + acc * kAccCols + ((q * 32u) << 16);
      const uint32_t row0 = t * kTileM + q * 32;
      if (kMode == kModeLayer) {
        float v[2][16];
        ptx::tmem_ld_16x256b_x4(tq, v[0]);
        ptx::tmem_ld_16x256b_x4(tq + (16u << 16), v[1]);
        ptx::tmem_wait_ld();
        ptx::tmem_regs_ready(v[0]);
        ptx::tmem_regs_ready(v[1]);
        ptx::tc_fence_before();
        ptx::mbar_arrive(&tempty[acc]);
#pragma unroll
        for (int hh = 0; hh < 2; ++hh)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            // register 4i+2h+e = column 8i+2j+e = feature 8j+2i+e of row r4 + 8h
            float o[8];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
              for (int e2 = 0; e2 < 2; ++e2) o[2 * i + e2] = fmaxf(v[hh][4 * i + 2 * h + e2] + b8[2 * i + e2], 0.0f);
            const uint32_t row = row0 + 16 * hh + r4 + 8 * h;
            if (row < n)
              ptx::stg_f8(a.hout + static_cast<size_t>(row) * kF + 8 * j, make_float4(o[0], o[1], o[2], o[3]),
                          make_float4(o[4], o[5], o[6], o[7]));
          }
      } else {
        // last layer: the accumulator is freed as soon as it is loaded; relu(acc + b)
        // split into TF32 hi / lo goes to the head's TMEM columns, then the 32 ->
        // classes head runs as one tensor-core MMA group, issued by the MMA warp
        // once all four quadrants are in (hready); each lane takes its row's logits
        // and the first maximum
        float r[32];
        ptx::tmem_ld_32x32b_x32(tq, r);
        ptx::tc_fence_before();
        ptx::mbar_arrive(&tempty[acc]);
#if GROOT_HEAD_CERT
        float x[32];
        uint32_t xs[32];
#pragma unroll
        for (int c = 0; c < 32; c += 2) {  // column c holds output feature kcol_feature(c); pairs: FADD2
          const float2 z = ptx::fadd2(make_float2(r[c], r[c + 1]),
                                      make_float2(hw.bias[kcol_feature(c)], hw.bias[kcol_feature(c + 1)]));
          x[c] = fmaxf(z.x, 0.0f);
          x[c + 1] = fmaxf(z.y, 0.0f);
          xs[c] = __float_as_uint(x[c]);
          xs[c + 1] = __float_as_uint(x[c + 1]);
        }
        ptx::tmem_st_32x32b_x32(tmem_base + kHeadHiCol + ((q * 32u) << 16), xs);
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        ptx::mbar_arrive(hready);  // the MMA warp issues the head
        ptx::mbar_wait(hdone, e & 1);
        ptx::tc_fence_after();
        float lg[16];
        ptx::tmem_ld_32x32b_x16(tmem_base + kHeadDCol + ((q * 32u) << 16), lg);
        const uint32_t row = row0 + lane;
        float best = 0.f, second = -INFINITY, smax = 0.f;
        uint32_t arg = 0;
#pragma unroll
        for (int cl = 0; cl < kMaxClasses; ++cl) {
          if (cl < static_cast<int>(a.classes)) {
            const float sc = lg[cl] + hw.b[cl];
            smax = fmaxf(smax, lg[8 + cl]);
            if (cl == 0) {
              best = sc;
            } else if (sc > best) {
              second = fmaxf(second, best);
              best = sc;
              arg = cl;
            } else {
              second = fmaxf(second, sc);
            }
          }
        }
        // |logit - x.W| <= 2^-10 S_c (operand) + accumulation; margin must beat both bounds
        const float bound =
            a.head_cert * (smax * (2.0f * 1.125f / 1024.0f) + 1e-6f * (fabsf(best) + fabsf(second)) + 1e-30f);
        if (a.logits || !(best - second > bound)) {  // exact fp32 head from x (rare without logits)
          float l[kMaxClasses];
#pragma unroll
          for (int cl = 0; cl < kMaxClasses; ++cl) l[cl] = hw.b[cl];
#pragma unroll
          for (int c = 0; c < 32; ++c)
#pragma unroll
            for (int cl = 0; cl < kMaxClasses; ++cl)
              if (cl < static_cast<int>(a.classes)) l[cl] = fmaf(x[c], hw.w[kcol_feature(c)][cl], l[cl]);
          best = l[0];
          arg = 0;
#pragma unroll
          for (int cl = 0; cl < kMaxClasses; ++cl) {
            if (cl < static_cast<int>(a.classes)) {
              if (cl > 0 && l[cl] > best) { best = l[cl]; arg = cl; }
              if (a.logits && row < n) a.logits[static_cast<size_t>(row) * a.classes + cl] = l[cl];
            }
          }
        }
        if (row < n) a.cls[row] = static_cast<uint8_t>(arg);
#else
        uint32_t hi[32], lo[32];
#pragma unroll
        for (int c = 0; c < 32; c += 2) {  // column c holds output feature kcol_feature(c); pairs: FADD2
          const float2 z = ptx::fadd2(make_float2(r[c], r[c + 1]),
                                      make_float2(hw.bias[kcol_feature(c)], hw.bias[kcol_feature(c + 1)]));
          const float2 x = make_float2(fmaxf(z.x, 0.0f), fmaxf(z.y, 0.0f));
          hi[c] = __float_as_uint(x.x) & 0xFFFFE000u;
          hi[c + 1] = __float_as_uint(x.y) & 0xFFFFE000u;
          const float2 l = ptx::fsub2(x, make_float2(__uint_as_float(hi[c]), __uint_as_float(hi[c + 1])));
          lo[c] = __float_as_uint(l.x);
          lo[c + 1] = __float_as_uint(l.y);
        }
#if GROOT_LAST_PIPE
        // the previous tile's logits leave the head's columns before this tile's
        // head A operand is published (its MMA overwrites them)
        float lg[8];
        if (e > 0) {
          ptx::mbar_wait(hdone, (e - 1) & 1);
          ptx::tc_fence_after();
          ptx::tmem_ld_32x32b_x8(tmem_base + kHeadDCol + ((q * 32u) << 16), lg);
        }
        ptx::tmem_st_32x32b_x32(tmem_base + kHeadHiCol + ((q * 32u) << 16), hi);
        ptx::tmem_st_32x32b_x32(tmem_base + kHeadLoCol + ((q * 32u) << 16), lo);
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        ptx::mbar_arrive(hready);
        if (e > 0) head_out(prev_row, lg);
        prev_row = row0 + lane;
#else
        ptx::tmem_st_32x32b_x32(tmem_base + kHeadHiCol + ((q * 32u) << 16), hi);
        ptx::tmem_st_32x32b_x32(tmem_base + kHeadLoCol + ((q * 32u) << 16), lo);
        ptx::tmem_wait_st();
        ptx::tc_fence_before();
        ptx::mbar_arrive(hready);  // the MMA warp issues the head
        if (GROOT_EPI_POLL_NS) ptx::mbar_wait_poll(hdone, e & 1, 32);
        else ptx::mbar_wait(hdone, e & 1);
        ptx::tc_fence_after();
        float lg[8];
        ptx::tmem_ld_32x32b_x8(tmem_base + kHeadDCol + ((q * 32u) << 16), lg);
        const uint32_t row = row0 + lane;
        float best = 0.f;
        uint32_t arg = 0;
#pragma unroll
        for (int cl = 0; cl < kMaxClasses; ++cl) {
          if (cl < static_cast<int>(a.classes)) {
            const float sc = lg[cl] + hw.b[cl];
            if (cl == 0 || sc > best) { best = sc; arg = cl; }
            if (a.logits && row < n) a.logits[static_cast<size_t>(row) * a.classes + cl] = sc;
          }
        }
        if (row < n) a.cls[row] = static_cast<uint8_t>(arg);
#endif
#endif  // GROOT_HEAD_CERT
      }
      if (warp == 0 && lane == 0) tstamp(a.trace, e, 12);
    }
  }

  if (kMma) {
    ptx::tc_fence_before();
    __syncthreads();
    if (warp == kMmaWarp) {
      ptx::tc_fence_after();
      ptx::tmem_dealloc<kTmemCols>(tmem_base);
    }
  }
}

// ---------------------------------------------------------------------------
// Layer 0: 4 -> 32 from u8 features (one u32 word per node), thread per row:
// each neighbour costs a 4-byte gather, so one thread owns a row and a warp
// has 32 rows' gathers in flight. Neighbour feature words are summed as packed
// byte counters (exact for LD degree < 256); weights are kernel parameters
// (constant bank: free FFMA operands). The 32 outputs of a row are staged in
// shared memory so each warp store writes four full 128-byte rows.
// ---------------------------------------------------------------------------
struct Layer0W {
  float ws[4][kF], wn[4][kF], b[kF];
};

struct Layer0Args {
  uint32_t n;
  const uint32_t* rp;
  const uint32_t* col;
  const uint32_t* feat;
  HdInfo hd;  // mean width 4
  float* hout;
  uint32_t binary;  // every feature byte is 0/1: neighbour words summed as packed byte counters
};

constexpr int kL0Threads = 256;
constexpr int kL0Stride = 36;  // floats per staged row (144 B: conflict-free 16-B phases)

__global__ void __launch_bounds__(kL0Threads) sage_layer0_kernel(const Layer0Args a, const Layer0W w) {
  __shared__ __align__(16) float stage[kL0Threads / 32][32 * kL0Stride];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  float* sw = stage[wid];
  const uint32_t warps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t base = (blockIdx.x * (blockDim.x >> 5) + wid) * 32; base < a.n; base += warps * 32) {
    const uint32_t row = base + lane;
    uint32_t b = 0, d = 0;
    if (row < a.n) {
      b = __ldg(a.rp + row);
      d = __ldg(a.rp + row + 1) - b;
    }
    const bool is_hd = d >= a.hd.threshold;
    const uint32_t dl = is_hd ? 0u : d;
    // per-feature neighbour sums: binary features as packed byte counters
    // (exact: an LD row has < 256 neighbours), any other u8 values in four
    // separate u32 counters (the reference sums arbitrary u8 features)
    uint32_t cnt[4] = {0u, 0u, 0u, 0u};
    {
      uint32_t c[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) c[k] = (static_cast<uint32_t>(k) < dl) ? __ldg(a.col + b + k) : 0u;
      uint32_t f[8];
#pragma unroll
      for (int k = 0; k < 8; ++k) f[k] = (static_cast<uint32_t>(k) < dl) ? __ldg(a.feat + c[k]) : 0u;
      if (a.binary) {
        uint32_t packed = 0;
#pragma unroll
        for (int k = 0; k < 8; ++k) packed += f[k];
        for (uint32_t k = 8; k < dl; ++k) packed += __ldg(a.feat + __ldg(a.col + b + k));
#pragma unroll
        for (int q = 0; q < 4; ++q) cnt[q] = (packed >> (8 * q)) & 0xFFu;
      } else {
#pragma unroll
        for (int k = 0; k < 8; ++k)
#pragma unroll
          for (int q = 0; q < 4; ++q) cnt[q] += (f[k] >> (8 * q)) & 0xFFu;
        for (uint32_t k = 8; k < dl; ++k) {
          const uint32_t x = __ldg(a.feat + __ldg(a.col + b + k));
#pragma unroll
          for (int q = 0; q < 4; ++q) cnt[q] += (x >> (8 * q)) & 0xFFu;
        }
      }
    }
    float m[4];
    if (is_hd) {
      const float4 mm = ptx::ldg_f4(a.hd.mean + static_cast<size_t>(hd_slot(a.hd, row)) * 4);
      m[0] = mm.x; m[1] = mm.y; m[2] = mm.z; m[3] = mm.w;
    } else {
      const float inv = d > 0 ? 1.0f / static_cast<float>(d) : 0.0f;
#pragma unroll
      for (int k = 0; k < 4; ++k) m[k] = static_cast<float>(cnt[k]) * inv;
    }
    const uint32_t x = row < a.n ? __ldg(a.feat + row) : 0u;
    float xk[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) xk[k] = static_cast<float>((x >> (8 * k)) & 0xFFu);
#pragma unroll
    for (int c4 = 0; c4 < 8; ++c4) {
      float z[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const int o = 4 * c4 + i;
        float s1 = 0.f, s2 = 0.f;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          s1 = fmaf(xk[k], w.ws[k][o], s1);
          s2 = fmaf(m[k], w.wn[k][o], s2);
        }
        z[i] = fmaxf((s1 + s2) + w.b[o], 0.f);
      }
      *reinterpret_cast<float4*>(sw + lane * kL0Stride + 4 * c4) = make_float4(z[0], z[1], z[2], z[3]);
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      const uint32_t ri = k * 4 + (lane >> 3), c = lane & 7;
      const float4 v = *reinterpret_cast<const float4*>(sw + ri * kL0Stride + 4 * c);
      if (base + ri < a.n) *reinterpret_cast<float4*>(a.hout + static_cast<size_t>(base + ri) * kF + 4 * c) = v;
    }
    __syncwarp();
  }
}

// ---------------------------------------------------------------------------
// HD rows, L2-ordered (hd_chunk_kernel + hd_reduce_kernel): each HD row's
// neighbour list is cut into chunks of kHdChunk nonzeros, and the chunks of
// all HD rows are processed in the order of their first neighbour's row id
// (the per-graph HD plan, build_hd_plan). In a multiplier the PIs' neighbours
// are the partial products: a_i's are one array row, b_j's one per array
// row; ordered by position, the chunks that read the same partial-product
// rows run together, so each is fetched from DRAM about once instead of twice.
// A warp sums one chunk in nonzero order (4 row groups of 8 lanes, combined in
// fixed order) into a partial row; hd_reduce_kernel adds a row's partials in
// chunk order and scales by 1/deg: deterministic.
// ---------------------------------------------------------------------------
constexpr uint32_t kHdChunk = 64;

__global__ void __launch_bounds__(256) hd_chunk_kernel(const uint32_t* __restrict__ units, uint32_t nunits,
                                                       const uint32_t* __restrict__ unit_slot,
                                                       const uint32_t* __restrict__ unit_k,
                                                       const uint32_t* __restrict__ hd_rows,
                                                       const uint32_t* __restrict__ rp, const uint32_t* __restrict__ col,
                                                       const float* __restrict__ H, float* __restrict__ partial,
                                                       const uint32_t* __restrict__ unit_base,
                                                       const uint8_t* __restrict__ keys) {
  const uint32_t lane = threadIdx.x & 31, g = lane >> 3, j = lane & 7;
  // keys != null: row c of H is entry row keys[c] (keyed layer 1)
  auto row_of = [&](uint32_t c) -> const float* {
    return H + static_cast<size_t>(keys ? static_cast<uint32_t>(__ldg(keys + c)) : c) * kF + 4 * j;
  };
  const uint32_t warps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t w = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); w < nunits; w += warps) {
    const uint32_t u = units[w];
    const uint32_t slot = unit_slot[u], k = unit_k[u];
    const uint32_t r = hd_rows[slot];
    const uint32_t b = rp[r] + k * kHdChunk;
    const uint32_t e = min(b + kHdChunk, rp[r + 1]);
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    // group g takes nonzeros b+g, b+g+4, ...; 4 rows in flight per group
    uint32_t q = b + g;
    for (; q + 12 < e; q += 16) {
      const uint32_t c0 = __ldg(col + q), c1 = __ldg(col + q + 4), c2 = __ldg(col + q + 8), c3 = __ldg(col + q + 12);
      const float4 v0 = ptx::ldg_f4(row_of(c0));
      const float4 v1 = ptx::ldg_f4(row_of(c1));
      const float4 v2 = ptx::ldg_f4(row_of(c2));
      const float4 v3 = ptx::ldg_f4(row_of(c3));
      acc = f4add(f4add(acc, v0), v1);
      acc = f4add(f4add(acc, v2), v3);
    }
    for (; q < e; q += 4) acc = f4add(acc, ptx::ldg_f4(row_of(__ldg(col + q))));
    // fixed-order combine of the 4 groups: lane j of group 0 adds groups 1..3
    float4 o1, o2, o3;
    o1.x = __shfl_down_sync(0xffffffffu, acc.x, 8); o1.y = __shfl_down_sync(0xffffffffu, acc.y, 8);
    o1.z = __shfl_down_sync(0xffffffffu, acc.z, 8); o1.w = __shfl_down_sync(0xffffffffu, acc.w, 8);
    o2.x = __shfl_down_sync(0xffffffffu, acc.x, 16); o2.y = __shfl_down_sync(0xffffffffu, acc.y, 16);
    o2.z = __shfl_down_sync(0xffffffffu, acc.z, 16); o2.w = __shfl_down_sync(0xffffffffu, acc.w, 16);
    o3.x = __shfl_down_sync(0xffffffffu, acc.x, 24); o3.y = __shfl_down_sync(0xffffffffu, acc.y, 24);
    o3.z = __shfl_down_sync(0xffffffffu, acc.z, 24); o3.w = __shfl_down_sync(0xffffffffu, acc.w, 24);
    if (g == 0) {
      const float4 sum = f4add(f4add(f4add(acc, o1), o2), o3);
      *reinterpret_cast<float4*>(partial + static_cast<size_t>(unit_base[slot] + k) * kF + 4 * j) = sum;
    }
  }
}

__global__ void __launch_bounds__(256) hd_reduce_kernel(uint32_t count, const uint32_t* __restrict__ hd_rows,
                                                        const uint32_t* __restrict__ rp,
                                                        const uint32_t* __restrict__ unit_base,
                                                        const float* __restrict__ partial, float* __restrict__ out,
                                                        int out_by_row) {
  // 8 lanes per HD row (float4 each)
  const uint32_t groups = gridDim.x * (blockDim.x >> 3);
  const uint32_t j = threadIdx.x & 7;
  for (uint32_t slot = blockIdx.x * (blockDim.x >> 3) + (threadIdx.x >> 3); slot < count; slot += groups) {
    const uint32_t r = hd_rows[slot], d = rp[r + 1] - rp[r];
    const uint32_t u0 = unit_base[slot], u1 = unit_base[slot + 1];
    float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
    for (uint32_t u = u0; u < u1; ++u) acc = f4add(acc, *reinterpret_cast<const float4*>(partial + static_cast<size_t>(u) * kF + 4 * j));
    const float inv = d > 0 ? 1.0f / static_cast<float>(d) : 0.0f;
    *reinterpret_cast<float4*>(out + static_cast<size_t>(out_by_row ? r : slot) * kF + 4 * j) = f4scale(acc, inv);
  }
}

__global__ void hd_units_kernel(uint32_t count, const uint32_t* __restrict__ hd_rows, const uint32_t* __restrict__ rp,
                                const uint32_t* __restrict__ col, const uint32_t* __restrict__ unit_base,
                                uint32_t* __restrict__ unit_slot, uint32_t* __restrict__ unit_k,
                                uint32_t* __restrict__ keys, uint32_t* __restrict__ ids) {
  for (uint32_t slot = blockIdx.x * blockDim.x + threadIdx.x; slot < count; slot += gridDim.x * blockDim.x) {
    const uint32_t r = hd_rows[slot], b = rp[r];
    for (uint32_t u = unit_base[slot], k = 0; u < unit_base[slot + 1]; ++u, ++k) {
      unit_slot[u] = slot;
      unit_k[u] = k;
      keys[u] = col[b + k * kHdChunk];  // first neighbour of the chunk (rows are sorted)
      ids[u] = u;
    }
  }
}

__global__ void hd_chunk_count_kernel(uint32_t count, const uint32_t* __restrict__ hd_rows,
                                      const uint32_t* __restrict__ rp, uint32_t* __restrict__ chunks) {
  for (uint32_t slot = blockIdx.x * blockDim.x + threadIdx.x; slot < count; slot += gridDim.x * blockDim.x) {
    const uint32_t r = hd_rows[slot];
    chunks[slot] = (rp[r + 1] - rp[r] + kHdChunk - 1) / kHdChunk;
  }
}

// Layer-0 HD rows: exact integer feature counts, mean = count / deg.
__global__ void __launch_bounds__(256) hd_mean_feat_kernel(const uint32_t* __restrict__ hd_rows, uint32_t count,
                                                           const uint32_t* __restrict__ rp,
                                                           const uint32_t* __restrict__ col,
                                                           const uint32_t* __restrict__ feat, float* __restrict__ out) {
  __shared__ uint32_t red[8][4];
  for (uint32_t slot = blockIdx.x; slot < count; slot += gridDim.x) {
    const uint32_t r = hd_rows[slot], b = rp[r], d = rp[r + 1] - b;
    uint32_t c[4] = {0, 0, 0, 0};
    for (uint32_t e = threadIdx.x; e < d; e += blockDim.x) {
      const uint32_t x = __ldg(feat + __ldg(col + b + e));
#pragma unroll
      for (int k = 0; k < 4; ++k) c[k] += (x >> (8 * k)) & 0xFFu;
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
      for (int o = 16; o; o >>= 1) c[k] += __shfl_xor_sync(0xffffffffu, c[k], o);
    if ((threadIdx.x & 31) == 0)
#pragma unroll
      for (int k = 0; k < 4; ++k) red[threadIdx.x >> 5][k] = c[k];
    __syncthreads();
    if (threadIdx.x < 4) {
      uint32_t s = 0;
      for (int w = 0; w < 8; ++w) s += red[w][threadIdx.x];
      const float inv = d > 0 ? 1.0f / static_cast<float>(d) : 0.0f;
      out[static_cast<size_t>(slot) * 4 + threadIdx.x] = static_cast<float>(s) * inv;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// Keyed layer 0. A layer-0 row is a function of an exact integer record: own
// features, per-feature neighbour counts, degree (mean = count x 1/deg). AIG
// features are bits (node type, PI/PO, fan-in polarity), so a multiplier has a
// few dozen distinct records however many nodes it has. Per forward, on every
// row: the record (the layer-0 aggregation: CSR walk + feature gathers), a
// dictionary of the distinct records, layer 0's 4 -> 32 transform of each
// entry (the same FFMA sequence as sage_layer0_kernel: the rows are
// bit-identical), and a u8 entry id per row. Layer 1 expands ids into rows in
// shared memory instead of reading n x 128 B of materialized H1 that layer 0
// would have written. Graphs with non-binary features, HD degree > 4094 or
// more than 255 distinct records take the materialized path.
// Record: x (4 bits) | deg (12 bits) | count_k (12 bits each, k = 0..3).
// ---------------------------------------------------------------------------
constexpr uint32_t kDictCap = 255;     // entry ids are u8
constexpr uint32_t kDictSlots = 2048;  // global open-addressing table of records
constexpr uint32_t kDictLocal = 512;   // per-CTA table
constexpr uint32_t kDictLocalMax = 384;
constexpr unsigned long long kDictEmpty = ~0ull;

__device__ __forceinline__ uint32_t dict_hash(unsigned long long k) {
  return static_cast<uint32_t>((k * 0x9E3779B97F4A7C15ull) >> 40);
}
__device__ __forceinline__ unsigned long long l0_record(uint32_t x, uint32_t d, const uint32_t (&s)[4]) {
  const uint32_t x4 = (x & 1u) | ((x >> 7) & 2u) | ((x >> 14) & 4u) | ((x >> 21) & 8u);
  return x4 | (static_cast<unsigned long long>(d) << 4) | (static_cast<unsigned long long>(s[0]) << 16) |
         (static_cast<unsigned long long>(s[1]) << 28) | (static_cast<unsigned long long>(s[2]) << 40) |
         (static_cast<unsigned long long>(s[3]) << 52);
}
// flags[0]: not keyable (overflow / non-binary feature / degree); flags[1]: entries
__device__ void dict_insert_global(unsigned long long* tab, uint32_t* flags, unsigned long long k) {
  uint32_t h = dict_hash(k) & (kDictSlots - 1);
  for (uint32_t p = 0; p < kDictSlots; ++p, h = (h + 1) & (kDictSlots - 1)) {
    const unsigned long long cur = *reinterpret_cast<volatile unsigned long long*>(tab + h);
    if (cur == k) return;
    if (cur == kDictEmpty) {
      const unsigned long long prev = atomicCAS(tab + h, kDictEmpty, k);
      if (prev == kDictEmpty) {
        if (atomicAdd(flags + 1, 1u) >= kDictCap) flags[0] = 1;
        return;
      }
      if (prev == k) return;
    }
  }
  flags[0] = 1;
}

// Warp-collective: the first lane of each distinct record finds / inserts its
// slot in the CTA's table; every lane gets its record's slot (0xFFFF: table full).
__device__ __forceinline__ uint32_t l0_dedup_insert(unsigned long long key, unsigned long long* ltab, uint32_t* lcount,
                                                    uint32_t* lbad, int lane) {
  const uint32_t peers = __match_any_sync(0xffffffffu, key);
  const int leader = __ffs(peers) - 1;
  uint32_t slot = 0xFFFFu;
  if (key != kDictEmpty && leader == lane) {
    uint32_t h = dict_hash(key) & (kDictLocal - 1);
    for (;; h = (h + 1) & (kDictLocal - 1)) {
      const unsigned long long cur = *reinterpret_cast<volatile unsigned long long*>(ltab + h);
      if (cur == key) break;
      if (cur == kDictEmpty) {
        if (*reinterpret_cast<volatile uint32_t*>(lcount) >= kDictLocalMax) {
          *lbad = 1;
          h = 0xFFFFu;
          break;
        }
        const unsigned long long prev = atomicCAS(ltab + h, kDictEmpty, key);
        if (prev == kDictEmpty) {
          atomicAdd(lcount, 1u);
          break;
        }
        if (prev == key) break;
      }
    }
    slot = h;
  }
  return __shfl_sync(0xffffffffu, slot, leader);
}

// LD rows: kL0KeyRows rows per thread with their gathers interleaved (a row's
// chain row_ptr -> col -> features is three dependent memory round trips), the
// gather of sage_layer0_kernel; warp-deduplicated records go into a per-CTA
// table. A row stores its u16 slot in its CTA's table (the CTA is a function
// of the row: l0_ids_kernel); the tables stay in global memory and are merged
// into the global dictionary.
constexpr uint32_t kL0KeyRows = 1;  // rows per thread (measured: 4 rows per thread with 40 registers is slower: occupancy, not the chain, bounds the loads in flight)
__global__ void __launch_bounds__(256) l0_key_kernel(uint32_t n, const uint32_t* __restrict__ rp,
                                                     const uint32_t* __restrict__ col,
                                                     const uint32_t* __restrict__ feat, uint32_t thr,
                                                     uint16_t* __restrict__ lslot,
                                                     unsigned long long* __restrict__ ctab,
                                                     unsigned long long* __restrict__ gtab, uint32_t* flags) {
  __shared__ unsigned long long ltab[kDictLocal];
  __shared__ uint32_t lcount, lbad;
  for (uint32_t i = threadIdx.x; i < kDictLocal; i += blockDim.x) ltab[i] = kDictEmpty;
  if (threadIdx.x == 0) lcount = lbad = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const uint32_t warps = gridDim.x * (blockDim.x >> 5);
  constexpr uint32_t kR = kL0KeyRows;
  for (uint32_t base = (blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5)) * 32 * kR; base < n;
       base += warps * 32 * kR) {
    uint32_t b[kR], d[kR];
#pragma unroll
    for (uint32_t r = 0; r < kR; ++r) {
      const uint32_t row = base + 32 * r + lane;
      b[r] = row < n ? __ldg(rp + row) : 0u;
      d[r] = row < n ? __ldg(rp + row + 1) - b[r] : 0u;
      if (d[r] >= thr) d[r] = 0xFFFFFFFFu;  // HD row: hd_key_kernel
    }
    uint32_t c[kR][8];
#pragma unroll
    for (uint32_t r = 0; r < kR; ++r)
#pragma unroll
      for (uint32_t k = 0; k < 8; ++k) c[r][k] = (d[r] != 0xFFFFFFFFu && k < d[r]) ? __ldg(col + b[r] + k) : 0u;
    uint32_t packed[kR], x[kR];
#pragma unroll
    for (uint32_t r = 0; r < kR; ++r) {
      const uint32_t row = base + 32 * r + lane;
      x[r] = row < n ? __ldg(feat + row) : 0u;
      packed[r] = 0;
#pragma unroll
      for (uint32_t k = 0; k < 8; ++k)
        packed[r] += (d[r] != 0xFFFFFFFFu && k < d[r]) ? __ldg(feat + c[r][k]) : 0u;
    }
#pragma unroll
    for (uint32_t r = 0; r < kR; ++r) {
      const uint32_t row = base + 32 * r + lane;
      const bool ld = row < n && d[r] != 0xFFFFFFFFu;
      if (ld)
        for (uint32_t k = 8; k < d[r]; ++k) packed[r] += __ldg(feat + __ldg(col + b[r] + k));
      unsigned long long key = kDictEmpty;
      if (ld) {
        // every node's own word is checked here or in hd_key_kernel, so byte
        // counters of binary features (d < 256) are exact
        if ((x[r] & 0xFEFEFEFEu) != 0u) lbad = 1;
        const uint32_t s[4] = {packed[r] & 0xFFu, (packed[r] >> 8) & 0xFFu, (packed[r] >> 16) & 0xFFu,
                               packed[r] >> 24};
        key = l0_record(x[r], d[r], s);
      }
      const uint32_t slot = l0_dedup_insert(key, ltab, &lcount, &lbad, lane);
      if (row < n) lslot[row] = static_cast<uint16_t>(key != kDictEmpty ? slot : 0xFFFFu);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && lbad) flags[0] = 1;
  for (uint32_t i = threadIdx.x; i < kDictLocal; i += blockDim.x) {
    const unsigned long long k = ltab[i];
    ctab[static_cast<size_t>(blockIdx.x) * kDictLocal + i] = k;
    if (k != kDictEmpty) dict_insert_global(gtab, flags, k);
  }
}

// The key pass through the tile plan: a warp per 128-row tile stages the
// feature words of the tile's rows and of its halo rows in shared memory (the
// row records name each neighbour's slot), so a row's neighbour features are
// shared-memory reads instead of a CSR walk with 4-byte gathers from L2 (one
// 32-byte sector each). Rows of degree > 4 finish from the CSR; slow tiles
// take the CSR walk. Same records, dedup and tables as l0_key_kernel; the CTA
// of a row is the CTA of its tile's warp (l0_ids_kernel, tiled).
struct L0KeyPlan {
  const uint4* tmeta;
  const unsigned long long* rec;
  const uint32_t* halo;
  uint32_t period, period_rows;
};

#ifdef GROOT_L0_KEY_MINB  // experiment knob: min CTAs per SM (register cap) of the key pass
#define GROOT_L0_KEY_BOUNDS __launch_bounds__(256, GROOT_L0_KEY_MINB)
#else
#define GROOT_L0_KEY_BOUNDS __launch_bounds__(256)
#endif
__global__ void GROOT_L0_KEY_BOUNDS l0_key_tile_kernel(uint32_t n, const uint32_t* __restrict__ rp,
                                                          const uint32_t* __restrict__ col,
                                                          const uint32_t* __restrict__ feat, uint32_t thr,
                                                          const L0KeyPlan p, uint16_t* __restrict__ lslot,
                                                          unsigned long long* __restrict__ ctab,
                                                          unsigned long long* __restrict__ gtab, uint32_t* flags) {
  __shared__ unsigned long long ltab[kDictLocal];
  __shared__ uint32_t lcount, lbad;
  __shared__ __align__(16) uint32_t sF_all[8][kTpRows + kTpHaloCap];
  for (uint32_t i = threadIdx.x; i < kDictLocal; i += blockDim.x) ltab[i] = kDictEmpty;
  if (threadIdx.x == 0) lcount = lbad = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  uint32_t* sF = sF_all[threadIdx.x >> 5];
  const uint32_t ntiles = (n + kTpRows - 1) / kTpRows;
  // The warp's tiles t0, t0 + S, ... go through a three-stage pipeline of
  // global loads, so a tile's dependent chain (plan meta -> records, features,
  // halo list -> halo features) is in flight behind the previous tiles' work:
  //   meta of tile t + 2S | records, tile features, halo list of t + S |
  //   halo features of t (issued at the end of the previous iteration).
  constexpr uint32_t kPer = (kTpHaloCap + 31) / 32;  // halo entries per lane
  const uint32_t S = gridDim.x * (blockDim.x >> 5);
  struct Stage {
    uint32_t t;
    uint4 meta;
    unsigned long long r[kTpRows / 32];
    uint4 f;
    uint32_t h[kPer];  // halo row ids, then their feature words
  };
  auto meta_of = [&](uint32_t t) -> uint4 {
    return t < ntiles ? __ldg(p.tmeta + (p.period ? t % p.period : t)) : make_uint4(0, 0, 0, kTpSlow);
  };
  auto load_rows = [&](Stage& st) {  // records, tile features, halo list (needs st.meta)
    if (st.t >= ntiles || (st.meta.w & kTpSlow)) return;
    const uint32_t pt = p.period ? st.t % p.period : st.t;
    const uint32_t row0 = st.t * kTpRows;
#pragma unroll
    for (uint32_t i = 0; i < kTpRows / 32; ++i) st.r[i] = __ldg(p.rec + static_cast<size_t>(pt) * kTpRows + 32 * i + lane);
    if (row0 + kTpRows <= n) {
      st.f = __ldg(reinterpret_cast<const uint4*>(feat + row0) + lane);
    } else {
      uint32_t w[4];
#pragma unroll
      for (uint32_t i = 0; i < 4; ++i) w[i] = row0 + 4 * lane + i < n ? __ldg(feat + row0 + 4 * lane + i) : 0u;
      st.f = make_uint4(w[0], w[1], w[2], w[3]);
    }
#pragma unroll
    for (uint32_t u = 0; u < kPer; ++u) st.h[u] = lane + 32 * u < st.meta.w ? __ldg(p.halo + st.meta.y + lane + 32 * u) : 0u;
  };
  auto load_halo = [&](Stage& st) {  // halo feature words (needs the halo list)
    if (st.t >= ntiles || (st.meta.w & kTpSlow)) return;
    const uint32_t shift = p.period ? (st.t / p.period) * p.period_rows : 0u;
#pragma unroll
    for (uint32_t u = 0; u < kPer; ++u) st.h[u] = lane + 32 * u < st.meta.w ? __ldg(feat + shift + st.h[u]) : 0u;
  };
  const uint32_t t0 = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  Stage cur, nx1;
  uint4 nx2_meta;
  cur.t = t0;
  cur.meta = meta_of(cur.t);
  load_rows(cur);
  load_halo(cur);
  nx1.t = t0 + S;
  nx1.meta = meta_of(nx1.t);
  load_rows(nx1);
  nx2_meta = meta_of(t0 + 2 * S);
  for (uint32_t t = t0; t < ntiles; t += S) {
    const uint4 meta = cur.meta;
    const bool slow = (meta.w & kTpSlow) != 0;
    const uint32_t row0 = t * kTpRows;
    unsigned long long r[kTpRows / 32];
    if (!slow) {
#pragma unroll
      for (uint32_t i = 0; i < kTpRows / 32; ++i) r[i] = cur.r[i];
      reinterpret_cast<uint4*>(sF)[lane] = cur.f;
#pragma unroll
      for (uint32_t u = 0; u < kPer; ++u)
        if (lane + 32 * u < meta.w) sF[kTpRows + lane + 32 * u] = cur.h[u];
      if (lane == 0) sF[kTpZeroSlot] = 0u;
    }
    // advance the pipeline: the next tiles' loads go out before this tile's work
    cur = nx1;
    load_halo(cur);
    nx1.t = t + 2 * S;
    nx1.meta = nx2_meta;
    load_rows(nx1);
    nx2_meta = meta_of(t + 3 * S);
    __syncwarp();
#pragma unroll
    for (uint32_t i = 0; i < kTpRows / 32; ++i) {
      const uint32_t row = row0 + 32 * i + lane;
      unsigned long long key = kDictEmpty;
      if (row < n) {
        uint32_t x, d, packed = 0;
        bool hd;
        if (slow) {
          x = __ldg(feat + row);
          const uint32_t b = __ldg(rp + row);
          d = __ldg(rp + row + 1) - b;
          hd = d >= thr;
          for (uint32_t k = 0; k < d && !hd; ++k) packed += __ldg(feat + __ldg(col + b + k));
        } else {
          x = sF[32 * i + lane];
          const uint32_t lo32 = static_cast<uint32_t>(r[i]);
          hd = (lo32 & kTpRecHd) != 0;
          d = tp_rec_degree(lo32);
#pragma unroll
          for (uint32_t k = 0; k < kTpRecSlots; ++k) packed += sF[static_cast<uint32_t>(r[i] >> (16 * k + 7)) & 0x1FFu];
          if (lo32 & kTpRecLong) {
            const uint32_t b = __ldg(rp + row);
            for (uint32_t k = kTpRecSlots; k < d; ++k) packed += __ldg(feat + __ldg(col + b + k));
          }
        }
        if (!hd) {
          if ((x & 0xFEFEFEFEu) != 0u) lbad = 1;  // byte counters of binary features (d < 256) are exact
          const uint32_t sc[4] = {packed & 0xFFu, (packed >> 8) & 0xFFu, (packed >> 16) & 0xFFu, packed >> 24};
          key = l0_record(x, d, sc);
        }
      }
      const uint32_t slot = l0_dedup_insert(key, ltab, &lcount, &lbad, lane);
      if (row < n) lslot[row] = static_cast<uint16_t>(key != kDictEmpty ? slot : 0xFFFFu);
    }
    __syncwarp();  // sF is restaged for the warp's next tile
  }
  __syncthreads();
  if (threadIdx.x == 0 && lbad) flags[0] = 1;
  for (uint32_t i = threadIdx.x; i < kDictLocal; i += blockDim.x) {
    const unsigned long long k = ltab[i];
    ctab[static_cast<size_t>(blockIdx.x) * kDictLocal + i] = k;
    if (k != kDictEmpty) dict_insert_global(gtab, flags, k);
  }
}

// HD rows: CTA per row, exact integer counts (as hd_mean_feat_kernel).
__global__ void __launch_bounds__(256) hd_key_kernel(const uint32_t* __restrict__ hd_rows, uint32_t count,
                                                     const uint32_t* __restrict__ rp, const uint32_t* __restrict__ col,
                                                     const uint32_t* __restrict__ feat,
                                                     unsigned long long* __restrict__ hdkey,
                                                     unsigned long long* __restrict__ gtab, uint32_t* flags) {
  __shared__ uint32_t red[8][4];
  for (uint32_t slot = blockIdx.x; slot < count; slot += gridDim.x) {
    const uint32_t r = hd_rows[slot], b = rp[r], d = rp[r + 1] - b;
    uint32_t c[4] = {0, 0, 0, 0};
    // four neighbours per thread in flight: column loads, then the feature gathers
    constexpr uint32_t kU = 4;
    for (uint32_t e0 = threadIdx.x; e0 < d; e0 += kU * blockDim.x) {
      uint32_t ci[kU];
#pragma unroll
      for (uint32_t u = 0; u < kU; ++u) ci[u] = e0 + u * blockDim.x < d ? __ldg(col + b + e0 + u * blockDim.x) : 0u;
#pragma unroll
      for (uint32_t u = 0; u < kU; ++u) {
        const uint32_t x = e0 + u * blockDim.x < d ? __ldg(feat + ci[u]) : 0u;
#pragma unroll
        for (int k = 0; k < 4; ++k) c[k] += (x >> (8 * k)) & 0xFFu;
      }
    }
#pragma unroll
    for (int k = 0; k < 4; ++k)
      for (int o = 16; o; o >>= 1) c[k] += __shfl_xor_sync(0xffffffffu, c[k], o);
    if ((threadIdx.x & 31) == 0)
#pragma unroll
      for (int k = 0; k < 4; ++k) red[threadIdx.x >> 5][k] = c[k];
    __syncthreads();
    if (threadIdx.x == 0) {
      uint32_t s[4] = {0, 0, 0, 0};
      for (int w = 0; w < 8; ++w)
#pragma unroll
        for (int k = 0; k < 4; ++k) s[k] += red[w][k];
      const uint32_t x = __ldg(feat + r);
      if ((x & 0xFEFEFEFEu) != 0u || d > 4094u) {
        flags[0] = 1;
      } else {
        const unsigned long long key = l0_record(x, d, s);
        hdkey[slot] = key;
        dict_insert_global(gtab, flags, key);
      }
    }
    __syncthreads();
  }
}

// One CTA: entries sorted by record (ids are deterministic), slot -> id map,
// and H1 of every entry with sage_layer0_kernel's arithmetic.
__global__ void __launch_bounds__(1024) dict_finalize_kernel(const unsigned long long* __restrict__ gtab,
                                                             const uint32_t* __restrict__ flags, const Layer0W w,
                                                             float* __restrict__ table, uint8_t* __restrict__ idmap) {
  __shared__ unsigned long long ent[kDictCap], sorted[kDictCap];
  __shared__ uint32_t cnt;
  if (flags[0]) return;
  if (threadIdx.x == 0) cnt = 0;
  __syncthreads();
  for (uint32_t i = threadIdx.x; i < kDictSlots; i += blockDim.x) {
    const unsigned long long k = gtab[i];
    if (k != kDictEmpty) {
      const uint32_t e = atomicAdd(&cnt, 1u);
      if (e < kDictCap) ent[e] = k;
    }
  }
  __syncthreads();
  const uint32_t m = cnt;
  if (m > kDictCap) return;  // flags[0] is set too
  for (uint32_t i = threadIdx.x; i < kDictSlots; i += blockDim.x) {
    const unsigned long long k = gtab[i];
    if (k == kDictEmpty) continue;
    uint32_t rank = 0;
    for (uint32_t e = 0; e < m; ++e) rank += ent[e] < k;
    idmap[i] = static_cast<uint8_t>(rank);
    sorted[rank] = k;
  }
  __syncthreads();
  for (uint32_t e = threadIdx.x; e < m * kF; e += blockDim.x) {
    const uint32_t id = e / kF, o = e % kF;
    const unsigned long long k = sorted[id];
    const uint32_t d = static_cast<uint32_t>(k >> 4) & 0xFFFu;
    const float inv = d > 0 ? 1.0f / static_cast<float>(d) : 0.0f;
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const float xk = static_cast<float>((k >> q) & 1u);
      const float mk = static_cast<float>(static_cast<uint32_t>(k >> (16 + 12 * q)) & 0xFFFu) * inv;
      s1 = fmaf(xk, w.ws[q][o], s1);
      s2 = fmaf(mk, w.wn[q][o], s2);
    }
    table[id * kF + o] = fmaxf((s1 + s2) + w.b[o], 0.f);
  }
}

__device__ __forceinline__ uint32_t dict_lookup(const unsigned long long* t, unsigned long long k) {
  uint32_t h = dict_hash(k) & (kDictSlots - 1);
  while (t[h] != k) h = (h + 1) & (kDictSlots - 1);
  return h;
}

// Per-CTA slot -> entry id (kDictLocal per l0_key_kernel CTA).
__global__ void __launch_bounds__(256) l0_xlat_kernel(uint32_t ctas, const unsigned long long* __restrict__ ctab,
                                                      const unsigned long long* __restrict__ gtab,
                                                      const uint8_t* __restrict__ idmap,
                                                      const uint32_t* __restrict__ flags, uint8_t* __restrict__ xlat) {
  if (flags[0]) return;
  const uint32_t total = ctas * kDictLocal;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < total; i += gridDim.x * blockDim.x) {
    const unsigned long long k = ctab[i];
    xlat[i] = k == kDictEmpty ? 0u : idmap[dict_lookup(gtab, k)];
  }
}

// u8 entry id of every LD row (4 rows per thread, one 32-bit store): the row's
// l0_key_kernel CTA (warp-strided row groups: CTA = ((row / (32 kL0KeyRows)) % warps) / 8) and
// its slot there. HD rows are written afterwards by l0_hd_ids_kernel.
__global__ void __launch_bounds__(256) l0_ids_kernel(uint32_t n, uint32_t key_warps, uint32_t rows_per_group,
                                                     const uint16_t* __restrict__ lslot,
                                                     const uint8_t* __restrict__ xlat,
                                                     const uint32_t* __restrict__ flags, uint8_t* __restrict__ ids) {
  if (flags[0]) return;
  const uint32_t quads = (n + 3) / 4;
  // kU independent quads per thread and iteration: their slot loads are in
  // flight together (one DRAM round trip per kU quads, not per quad)
  constexpr uint32_t kU = 4;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t qb = blockIdx.x * blockDim.x + threadIdx.x; qb < quads; qb += stride * kU) {
    uint2 sl[kU];
#pragma unroll
    for (uint32_t i = 0; i < kU; ++i) {
      const uint32_t q = qb + i * stride;
      sl[i] = q < quads && 4 * q + 3 < n ? *reinterpret_cast<const uint2*>(lslot + 4 * q) : make_uint2(~0u, ~0u);
    }
#pragma unroll
    for (uint32_t i = 0; i < kU; ++i) {
      const uint32_t q = qb + i * stride;
      if (q >= quads) break;
      const uint32_t cta = (((4 * q) / rows_per_group) % key_warps) >> 3;  // the 4 rows share a row group
      const uint8_t* xl = xlat + static_cast<size_t>(cta) * kDictLocal;
      if (4 * q + 3 < n) {
        const uint32_t s4[4] = {sl[i].x & 0xFFFFu, sl[i].x >> 16, sl[i].y & 0xFFFFu, sl[i].y >> 16};
        uint32_t out = 0;
#pragma unroll
        for (int u = 0; u < 4; ++u) out |= static_cast<uint32_t>(s4[u] < kDictLocal ? __ldg(xl + s4[u]) : 0u) << (8 * u);
        reinterpret_cast<uint32_t*>(ids)[q] = out;
      } else {
        for (uint32_t r = 4 * q; r < n; ++r) {
          const uint32_t s1 = lslot[r];
          ids[r] = s1 < kDictLocal ? __ldg(xl + s1) : 0u;
        }
      }
    }
  }
}

__global__ void l0_hd_ids_kernel(uint32_t count, const uint32_t* __restrict__ hd_rows,
                                 const unsigned long long* __restrict__ hdkey,
                                 const unsigned long long* __restrict__ gtab, const uint8_t* __restrict__ idmap,
                                 const uint32_t* __restrict__ flags, uint8_t* __restrict__ ids) {
  if (flags[0]) return;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < count; i += gridDim.x * blockDim.x)
    ids[hd_rows[i]] = idmap[dict_lookup(gtab, hdkey[i])];
}

// Entry ids of every tile's halo rows, laid out like the halo list (tile t at
// t * kTpHaloCap), so the fused layer's loader stages them with the plan.
// Periodic plans: tile t uses plan tile t % period, rows shifted per period.
__global__ void __launch_bounds__(256) l0_halo_ids_kernel(uint32_t ntiles, const uint4* __restrict__ tmeta,
                                                          const uint32_t* __restrict__ halo, uint32_t period,
                                                          uint32_t period_rows, const uint8_t* __restrict__ ids,
                                                          const uint32_t* __restrict__ flags, uint8_t* __restrict__ hids) {
  if (flags[0]) return;
  constexpr uint32_t kPer = kTpHaloCap / 32;
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t warps = gridDim.x * (blockDim.x >> 5);
  for (uint32_t t = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); t < ntiles; t += warps) {
    const uint32_t pt = period ? t % period : t;
    const uint32_t shift = period ? (t / period) * period_rows : 0u;
    const uint4 m = __ldg(tmeta + pt);
    if (m.w & kTpSlow) continue;
    uint32_t hv[kPer];
#pragma unroll
    for (uint32_t u = 0; u < kPer; ++u) hv[u] = lane + 32 * u < m.w ? __ldg(halo + m.y + lane + 32 * u) : 0u;
    uint32_t iv[kPer];
#pragma unroll
    for (uint32_t u = 0; u < kPer; ++u) iv[u] = lane + 32 * u < m.w ? __ldg(ids + shift + hv[u]) : 0u;
#pragma unroll
    for (uint32_t u = 0; u < kPer; ++u)
      if (lane + 32 * u < m.w) hids[static_cast<size_t>(t) * kTpHaloCap + lane + 32 * u] = static_cast<uint8_t>(iv[u]);
  }
}

// kModeXform tables: Tn[k] = table[k] . W_neigh, Ts[k] = table[k] . W_self
// (fp64 accumulation, rounded once), CTA per entry, thread per output.
// Tn = table . W_neigh and Ts = table . W_self + b (the layer bias folded into
// the self table, so the layer adds one table row to the neighbour mean), fp64.
__global__ void __launch_bounds__(64) l1_xform_kernel(const float* __restrict__ table, const float* __restrict__ ws,
                                                      const float* __restrict__ wn, const float* __restrict__ bias,
                                                      const uint32_t* __restrict__ flags, float* __restrict__ tn,
                                                      float* __restrict__ ts) {
  const uint32_t k = blockIdx.x, o = threadIdx.x & 31;
  if (flags[0] || k >= flags[1]) return;
  const float* W = threadIdx.x < 32 ? wn : ws;
  double acc = threadIdx.x < 32 ? 0.0 : static_cast<double>(bias[o]);
  for (uint32_t i = 0; i < kF; ++i) acc = fma(static_cast<double>(table[k * kF + i]), static_cast<double>(W[i * kF + o]), acc);
  (threadIdx.x < 32 ? tn : ts)[k * kF + o] = static_cast<float>(acc);
}

// General CSR SpMM (spmm::execute over CsrMatrix<T>, T = float or double): 8
// lanes per row, columns strided by 8, nonzeros accumulated in order with
// separately rounded multiply and add (no FMA contraction), i.e. the
// reference's dst[c] += v * src[c] (inc/spmm.hpp:117-124) bit for bit.
// vals == nullptr -> 1/deg.
__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }

// hd_threshold > 0: rows of degree >= hd_threshold are summed as execute's HD
// band does (src/spmm.cpp:73-96, inc/spmm.hpp:141-157): 32 chunks, the
// remainder on the trailing chunks, each chunk summed from zero, the chunk
// partials added in ascending order -- bitwise the reference's execute for a
// plan with that threshold. hd_threshold == 0: the plain row loop
// (reference_spmm, inc/spmm.hpp:183-195).
template <class T>
__global__ void __launch_bounds__(256) spmm_generic_kernel(uint32_t rows, const uint32_t* __restrict__ rp,
                                                           const uint32_t* __restrict__ col,
                                                           const T* __restrict__ vals,
                                                           const T* __restrict__ dense, uint32_t f,
                                                           T* __restrict__ out, uint32_t hd_threshold) {
  const int j = threadIdx.x & 7;
  const uint32_t groups = gridDim.x * (blockDim.x >> 3);
  for (uint32_t r = blockIdx.x * (blockDim.x >> 3) + (threadIdx.x >> 3); r < rows; r += groups) {
    const uint32_t b = rp[r], e = rp[r + 1], d = e - b;
    const T inv = e > b ? T(1) / static_cast<T>(d) : T(0);
    auto sum = [&](uint32_t q0, uint32_t q1, uint32_t c) {
      T acc = T(0);
      for (uint32_t q = q0; q < q1; ++q) {
        const T v = vals ? vals[q] : inv;
        acc = add_rn(acc, mul_rn(v, dense[static_cast<size_t>(col[q]) * f + c]));
      }
      return acc;
    };
    const bool hd = hd_threshold && d >= hd_threshold;
    for (uint32_t c = j; c < f; c += 8) {
      T acc = T(0);
      if (hd) {
        const uint32_t qd = d / 32, rem = d % 32;
        uint32_t nz = b;
        for (uint32_t k = 0; k < 32; ++k) {
          const uint32_t len = qd + (k >= 32 - rem ? 1u : 0u);
          acc = add_rn(acc, sum(nz, nz + len, c));
          nz += len;
        }
      } else {
        acc = sum(b, e, c);
      }
      out[static_cast<size_t>(r) * f + c] = acc;
    }
  }
}

// ---------------------------------------------------------------------------
// Naive reference path (debug / differential tests only): thread per row.
// ---------------------------------------------------------------------------
__global__ void naive_layer_kernel(uint32_t n, const uint32_t* __restrict__ rp, const uint32_t* __restrict__ col,
                                   const float* __restrict__ hin, const uint32_t* __restrict__ feat, uint32_t fin,
                                   const float* __restrict__ ws, const float* __restrict__ wn,
                                   const float* __restrict__ b, float* __restrict__ hout) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    float h[32], m[32];
    for (uint32_t k = 0; k < fin; ++k) {
      h[k] = hin ? hin[static_cast<size_t>(r) * fin + k] : static_cast<float>((feat[r] >> (8 * k)) & 0xFF);
      m[k] = 0.f;
    }
    const uint32_t d = rp[r + 1] - rp[r];
    for (uint32_t q = rp[r]; q < rp[r + 1]; ++q) {
      const uint32_t u = col[q];
      for (uint32_t k = 0; k < fin; ++k)
        m[k] += hin ? hin[static_cast<size_t>(u) * fin + k] : static_cast<float>((feat[u] >> (8 * k)) & 0xFF);
    }
    const float inv = d ? 1.0f / static_cast<float>(d) : 0.0f;
    for (uint32_t k = 0; k < fin; ++k) m[k] *= inv;
    for (uint32_t o = 0; o < 32; ++o) {
      float s1 = 0.f, s2 = 0.f;
      for (uint32_t k = 0; k < fin; ++k) {
        s1 = fmaf(h[k], ws[k * 32 + o], s1);
        s2 = fmaf(m[k], wn[k * 32 + o], s2);
      }
      hout[static_cast<size_t>(r) * 32 + o] = fmaxf((s1 + s2) + b[o], 0.f);
    }
  }
}

__global__ void head_kernel(uint32_t n, const float* __restrict__ h, const float* __restrict__ head, uint32_t C,
                            uint8_t* __restrict__ cls, float* __restrict__ logits, const uint8_t* __restrict__ labels,
                            unsigned long long* __restrict__ confusion) {
  for (uint32_t r = blockIdx.x * blockDim.x + threadIdx.x; r < n; r += gridDim.x * blockDim.x) {
    float best = 0.f;
    uint32_t arg = 0;
    for (uint32_t c = 0; c < C; ++c) {
      float s = 0.f;
      for (int k = 0; k < 32; ++k) s = fmaf(h[static_cast<size_t>(r) * 32 + k], head[k * C + c], s);
      s += head[32 * C + c];
      if (c == 0 || s > best) { best = s; arg = c; }
      if (logits) logits[static_cast<size_t>(r) * C + c] = s;
    }
    cls[r] = static_cast<uint8_t>(arg);
    if (confusion && labels && labels[r] < 5 && arg < 5) atomicAdd(&confusion[labels[r] * 5 + arg], 1ull);
  }
}

// confusion[truth][pred] (finish_prediction, src/gnn.cpp:268-276): 16 rows
// per thread and iteration (128-bit loads of classes and labels). Per truth
// class t a register holds five 6-bit counters (prediction p at bits 6p), so a
// row costs a shift and five predicated adds; every 48 rows they are flushed
// into 25 u32 totals, then warp-, block- and grid-reduced.
__global__ void __launch_bounds__(256) confusion_kernel(uint32_t n, const uint8_t* __restrict__ cls,
                                                        const uint8_t* __restrict__ labels,
                                                        unsigned long long* __restrict__ conf) {
  __shared__ uint32_t h[25];
  if (threadIdx.x < 25) h[threadIdx.x] = 0;
  __syncthreads();
  uint32_t tot[25], acc[5];
#pragma unroll
  for (int k = 0; k < 25; ++k) tot[k] = 0;
#pragma unroll
  for (int r = 0; r < 5; ++r) acc[r] = 0;
  auto count = [&](uint32_t p, uint32_t t) {
    const uint32_t inc = p < 5 ? 1u << (6 * p) : 0u;
#pragma unroll
    for (uint32_t r = 0; r < 5; ++r) acc[r] += t == r ? inc : 0u;
  };
  auto flush = [&]() {
#pragma unroll
    for (int r = 0; r < 5; ++r) {
#pragma unroll
      for (int q = 0; q < 5; ++q) tot[5 * r + q] += (acc[r] >> (6 * q)) & 63u;
      acc[r] = 0;
    }
  };
  const uint32_t stride = gridDim.x * blockDim.x;
  const bool aligned = ((reinterpret_cast<uintptr_t>(cls) | reinterpret_cast<uintptr_t>(labels)) & 15u) == 0;
  const uint32_t vecs = aligned ? n / 16 : 0u;  // caller buffers may be unaligned: scalar path
  uint32_t since = 0;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < vecs; v += stride) {
    const uint4 pc = __ldg(reinterpret_cast<const uint4*>(cls) + v);
    const uint4 tl = __ldg(reinterpret_cast<const uint4*>(labels) + v);
    const uint32_t pw[4] = {pc.x, pc.y, pc.z, pc.w}, tw[4] = {tl.x, tl.y, tl.z, tl.w};
#pragma unroll
    for (int w = 0; w < 4; ++w)
#pragma unroll
      for (int b = 0; b < 4; ++b) count((pw[w] >> (8 * b)) & 0xFFu, (tw[w] >> (8 * b)) & 0xFFu);
    if (++since == 3) {  // 48 rows < 64: no 6-bit counter overflows
      flush();
      since = 0;
    }
  }
  flush();
  for (uint32_t i = vecs * 16 + blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    count(cls[i], labels[i]);
    flush();
  }
#pragma unroll
  for (uint32_t k = 0; k < 25; ++k) {
    uint32_t c = tot[k];
    for (int o = 16; o; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
    if ((threadIdx.x & 31) == 0 && c) atomicAdd(&h[k], c);
  }
  __syncthreads();
  if (threadIdx.x < 25 && h[threadIdx.x]) atomicAdd(&conf[threadIdx.x], static_cast<unsigned long long>(h[threadIdx.x]));
}

// ---------------------------------------------------------------------------
// Row classifier (K10): rows with degree >= threshold, ascending.
// ---------------------------------------------------------------------------
__global__ void hd_flag_kernel(uint32_t n, const uint32_t* __restrict__ rp, uint32_t thr, uint8_t* __restrict__ flag) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    flag[v] = (rp[v + 1] - rp[v]) >= thr;
}

void classify_rows(groot_graph* g, uint32_t thr) {
  if (g->hd_threshold == thr && (g->num_hd == 0 || g->hd_rows.p)) return;
  ProfScope ps("classify_rows");
  DevBuf<uint8_t> flag(g->n);
  DevBuf<uint32_t> out(g->n), cnt(1);
  if (g->n) GROOT_LAUNCH(hd_flag_kernel, blocks_for(g->n, 256), 256, 0, g->n, g->rp.p, thr, flag.p);
  size_t bytes = 0;
  cub::CountingInputIterator<uint32_t> it(0);
  cub::DeviceSelect::Flagged(nullptr, bytes, it, flag.p, out.p, cnt.p, g->n, stream());
  DevBuf<uint8_t> tmp(bytes);
  GROOT_CUDA(cub::DeviceSelect::Flagged(tmp.p, bytes, it, flag.p, out.p, cnt.p, g->n, stream()));
  uint32_t num = 0;
  cnt.download(&num, 1);
  stream_sync();
  g->num_hd = num;
  g->hdp_valid = false;
  g->hd_rows.alloc(num);
  if (num)
    GROOT_CUDA(cudaMemcpyAsync(g->hd_rows.p, out.p, num * 4ull, cudaMemcpyDeviceToDevice, stream()));
  g->hd_mean.alloc(static_cast<size_t>(num) * kF);
  g->hd_threshold = thr;
  // (no synchronisation: the temporaries return to the stream-ordered pool)
}

void build_tile_plan(groot_graph* g, uint32_t thr);

// Kernel arguments common to the fused layer and the SpMM: CSR (slow tiles),
// input rows, HD band, tile plan.
static LayerArgs plan_args(groot_graph* g, const float* hin, const HdInfo& hd) {
  LayerArgs a{};
  a.n = g->n;
  a.rp = g->rp.p;
  a.col = g->col.p;
  a.hin = hin;
  a.hd = hd;
  a.tmeta = reinterpret_cast<const TileMeta*>(g->tp_meta.p);
  a.lrp = g->tp_lrp.p;
  a.lcol = g->tp_lcol.p;
  a.halo = g->tp_halo.p;
  a.rec = g->tp_rec.p;
  a.plan_period = g->tp_period;
  if (!g->tile_ctr.p) g->tile_ctr.alloc(1);
  static const bool dyn = env_u32("GROOT_DYNAMIC_TILES", 1) != 0;
  a.tile_counter = dyn ? g->tile_ctr.p : nullptr;
  if (a.tile_counter) GROOT_CUDA(cudaMemsetAsync(a.tile_counter, 0, sizeof(uint32_t), stream()));
  a.period_rows = g->tp_period_rows;
  return a;
}

// Per-graph HD plan (see hd_chunk_kernel): chunk units of every HD row,
// sorted by their first neighbour's row id. Cached on the graph.
static void build_hd_plan(groot_graph* g) {
  if (g->hdp_valid || g->num_hd == 0) return;
  const uint32_t count = g->num_hd;
  g->hdp_base.alloc(count + 1ull);
  DevBuf<uint32_t> chunks(count + 1ull);
  GROOT_LAUNCH(hd_chunk_count_kernel, blocks_for(count, 256), 256, 0, count, g->hd_rows.p, g->rp.p, chunks.p);
  exclusive_scan_u32(chunks.p, g->hdp_base.p, count);
  uint32_t nunits = 0;
  GROOT_CUDA(cudaMemcpyAsync(&nunits, g->hdp_base.p + count, 4, cudaMemcpyDeviceToHost, stream()));
  stream_sync();
  DevBuf<uint32_t> keys(nunits), keys2(nunits), ids(nunits);
  g->hdp_slot.alloc(nunits);
  g->hdp_k.alloc(nunits);
  g->hdp_units.alloc(nunits);
  GROOT_LAUNCH(hd_units_kernel, blocks_for(count, 256), 256, 0, count, g->hd_rows.p, g->rp.p, g->col.p,
               g->hdp_base.p, g->hdp_slot.p, g->hdp_k.p, keys.p, ids.p);
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, keys.p, keys2.p, ids.p, g->hdp_units.p, nunits, 0, 32, stream());
  DevBuf<uint8_t> tmp(bytes);
  GROOT_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, keys.p, keys2.p, ids.p, g->hdp_units.p, nunits, 0, 32,
                                             stream()));
  g->hdp_partial.alloc(static_cast<size_t>(nunits) * kF);
  g->hdp_nunits = nunits;
  g->hdp_valid = true;
}

__global__ void replicate_hd_units_kernel(uint32_t nunits1, uint32_t nhd1, uint32_t copies,
                                          const uint32_t* __restrict__ units1, const uint32_t* __restrict__ slot1,
                                          const uint32_t* __restrict__ k1, uint32_t* __restrict__ units,
                                          uint32_t* __restrict__ slot, uint32_t* __restrict__ kk) {
  const uint64_t total = static_cast<uint64_t>(nunits1) * copies;
  for (uint64_t i = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t c = static_cast<uint32_t>(i / nunits1), u = static_cast<uint32_t>(i - static_cast<uint64_t>(c) * nunits1);
    units[i] = units1[u] + c * nunits1;  // copy c's chunks come after copy c-1's in first-neighbour order
    slot[i] = slot1[u] + c * nhd1;
    kk[i] = k1[u];
  }
}

// HD plan of a tile-aligned batch from its copy 0's (see replicate_forward_plan).
void replicate_hd_plan(groot_graph* src, groot_graph* dst, uint32_t copies) {
  if (src->num_hd == 0 || dst->num_hd != src->num_hd * copies) return;
  build_hd_plan(src);
  const uint32_t nu1 = src->hdp_nunits;
  dst->hdp_nunits = nu1 * copies;
  dst->hdp_base.alloc(dst->num_hd + 1ull);
  GROOT_LAUNCH(replicate_offset_kernel, blocks_for(dst->num_hd / 4 + 1, 256), 256, 0,
               static_cast<uint64_t>(src->num_hd), copies, nu1, src->hdp_base.p, dst->hdp_base.p);
  const uint32_t last = dst->hdp_nunits;
  GROOT_CUDA(cudaMemcpyAsync(dst->hdp_base.p + dst->num_hd, &last, 4, cudaMemcpyHostToDevice, stream()));
  dst->hdp_slot.alloc(dst->hdp_nunits);
  dst->hdp_k.alloc(dst->hdp_nunits);
  dst->hdp_units.alloc(dst->hdp_nunits);
  GROOT_LAUNCH(replicate_hd_units_kernel, blocks_for(dst->hdp_nunits, 256), 256, 0, nu1, src->num_hd, copies,
               src->hdp_units.p, src->hdp_slot.p, src->hdp_k.p, dst->hdp_units.p, dst->hdp_slot.p, dst->hdp_k.p);
  dst->hdp_partial.alloc(static_cast<size_t>(dst->hdp_nunits) * kF);
  stream_sync();  // `last` lives on this stack frame
  dst->hdp_valid = true;
}

// HD rows' 32-wide neighbour means of H (L2-ordered chunks + fixed-order reduce).
static void hd_means32(groot_graph* g, const float* H, float* out, int out_by_row, const uint8_t* keys = nullptr) {
  build_hd_plan(g);
  const unsigned sms = static_cast<unsigned>(num_sms());
  GROOT_LAUNCH(hd_chunk_kernel, blocks_for(g->hdp_nunits * 32ull, 256, sms * 8), 256, 0, g->hdp_units.p,
               g->hdp_nunits, g->hdp_slot.p, g->hdp_k.p, g->hd_rows.p, g->rp.p, g->col.p, H, g->hdp_partial.p,
               g->hdp_base.p, keys);
  GROOT_LAUNCH(hd_reduce_kernel, blocks_for(g->num_hd * 8ull, 256, sms * 8), 256, 0, g->num_hd, g->hd_rows.p, g->rp.p,
               g->hdp_base.p, g->hdp_partial.p, out, out_by_row);
}

static void ensure_activations(groot_graph* g) {
  const size_t need = static_cast<size_t>(g->n) * kF;
  for (auto& b : g->act)
    if (b.n < need) b.alloc(need);
}

// TMA descriptor for an n x 32 fp32 row-major activation matrix: 32 x box_rows
// boxes, unswizzled (row i of the box at i * 128 B); rows past n read as zeros.
static CUtensorMap make_rows32_tmap(float* base, uint32_t n, uint32_t box_rows) {
  using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  static EncodeFn encode = [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    GROOT_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
    if (!fn || q != cudaDriverEntryPointSuccess) fail(GROOT_ECUDA, "cuTensorMapEncodeTiled unavailable");
    return reinterpret_cast<EncodeFn>(fn);
  }();
  CUtensorMap m;
  const cuuint64_t dims[2] = {kF, n};
  const cuuint64_t strides[1] = {kF * sizeof(float)};
  const cuuint32_t box[2] = {kF, box_rows};
  const cuuint32_t estr[2] = {1, 1};
  const CUresult r = encode(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) fail(GROOT_ECUDA, "cuTensorMapEncodeTiled failed: " + std::to_string(static_cast<int>(r)));
  return m;
}

static void set_tc_smem() {  // a per-device function attribute: once per device
  static std::atomic<bool> done[kMaxDevices];
  const int dev = current_device();
  if (done[dev].load()) return;
  constexpr uint32_t kS0 = TkCfg<false>::kSmem, kS1 = TkCfg<true>::kSmem;
  GROOT_CUDA(cudaFuncSetAttribute(sage_tile_kernel<kModeLayer>, cudaFuncAttributeMaxDynamicSharedMemorySize, kS0));
  GROOT_CUDA(cudaFuncSetAttribute(sage_tile_kernel<kModeLast>, cudaFuncAttributeMaxDynamicSharedMemorySize, kS0));
  GROOT_CUDA(cudaFuncSetAttribute(sage_tile_kernel<kModeSpmm>, cudaFuncAttributeMaxDynamicSharedMemorySize, kS0));
  GROOT_CUDA(cudaFuncSetAttribute(sage_tile_kernel<kModeLayer, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kS1));
  GROOT_CUDA(cudaFuncSetAttribute(sage_tile_kernel<kModeLast, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kS1));
  GROOT_CUDA(cudaFuncSetAttribute(sage_tile_kernel<kModeXform, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kS1));
  done[dev].store(true);
}

// Per-graph preparation shared by the whole forward and the layer API:
// row classifier (HD band) and, for models with tensor-core layers, the tile plan.
static void prepare_graph(const groot_model* m, groot_graph* g) {
  require(m->in_dim == 4 && m->hidden == kF, "forward: model shape unsupported (in_dim 4, hidden 32)");
  static const bool host_timing = std::getenv("GROOT_HOST_TIMING") != nullptr;
  auto now = [] { return std::chrono::steady_clock::now(); };
  const auto h0 = now();
  set_tc_smem();
  classify_rows(g, hd_threshold());
  const auto h1 = now();
  if (m->depth > 1) build_tile_plan(g, g->hd_threshold);
  const auto h2 = now();
  if (host_timing) {
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    std::fprintf(stderr, "[forward] classify %.2f ms, tile plan %.2f ms (host)\n", ms(h0, h1), ms(h1, h2));
  }
}

// One layer of run_forward (src/gnn.cpp:37-52) on a resident graph:
//   l = 0            features (u8) -> hout (n x 32)
//   0 < l < depth-1  hin (n x 32)  -> hout (n x 32)
//   l = depth-1      hin -> head + first-max argmax: cls (u8[n]), logits (n x classes, optional)
// (depth 1: layer 0 writes hout, then the head kernel). Rows are computed for
// every row of g, each from its own neighbour list in g.
// Keyed layer 0 (see l0_key_kernel) of a forward: records, dictionary, entry
// rows and ids. Returns false (nothing materialized) when the graph is not
// keyable; the first forward on a graph finds that out (one host sync).
static bool layer0_keyed(const groot_model* m, groot_graph* g) {
  const char* e = std::getenv("GROOT_L0_KEYED");
  if ((e && std::atoi(e) == 0) || m->depth < 2 || g->n == 0 || g->l0_mode == 2 || !g->binary_feat) return false;
  // small graphs: the key passes' fixed launch cost exceeds the layer-0 rows they save
  const char* mr = std::getenv("GROOT_L0_KEYED_MIN_ROWS");
  if (g->n < (mr ? std::strtoull(mr, nullptr, 10) : (1ull << 20))) return false;
  const uint32_t n = g->n;
  const uint32_t ntiles = (n + kTileM - 1) / kTileM;
  const unsigned sms = static_cast<unsigned>(num_sms());
  static const bool tiled_env = env_u32("GROOT_L0_KEY_TILED", 1) != 0;
  const bool key_tiled = tiled_env && g->tp_meta.p && g->tp_rec.p && g->tp_threshold == g->hd_threshold;
  static const uint32_t key_per_sm = env_u32("GROOT_L0_KEY_CTAS_PER_SM", 8);
  const unsigned key_ctas = key_tiled ? blocks_for(ntiles, 8, sms * key_per_sm)  // a warp per tile
                                      : blocks_for((n + kL0KeyRows - 1) / kL0KeyRows, 256, sms * 8);
  if (g->l0_slot.n < n) g->l0_slot.alloc(n);
  if (g->l0_id.n < static_cast<size_t>(ntiles) * kTileM) g->l0_id.alloc(static_cast<size_t>(ntiles) * kTileM);
  if (g->l0_hid.n < static_cast<size_t>(ntiles) * kTpHaloCap) g->l0_hid.alloc(static_cast<size_t>(ntiles) * kTpHaloCap);
  if (g->l0_ctab.n < static_cast<size_t>(key_ctas) * kDictLocal) {
    g->l0_ctab.alloc(static_cast<size_t>(key_ctas) * kDictLocal);
    g->l0_xlat.alloc(static_cast<size_t>(key_ctas) * kDictLocal);
  }
  if (g->l0_key.n < std::max<uint32_t>(g->num_hd, 1u)) g->l0_key.alloc(std::max<uint32_t>(g->num_hd, 1u));
  if (!g->l0_dict.p) {
    g->l0_dict.alloc(kDictSlots);
    g->l0_idmap.alloc(kDictSlots);
    g->l0_table.alloc(kTkTableRows * kF);
    g->l0_table.zero();
    g->l0_flags.alloc(2);
  }
  const uint32_t* feat = reinterpret_cast<const uint32_t*>(g->feat.p);
  {
    ProfScope ps("l0_keys");
    GROOT_CUDA(cudaMemsetAsync(g->l0_dict.p, 0xFF, kDictSlots * sizeof(unsigned long long), stream()));
    GROOT_CUDA(cudaMemsetAsync(g->l0_flags.p, 0, 2 * sizeof(uint32_t), stream()));
    if (g->num_hd)
      GROOT_LAUNCH(hd_key_kernel, std::min<uint32_t>(g->num_hd, sms * 8), 256, 0, g->hd_rows.p, g->num_hd, g->rp.p,
                   g->col.p, feat, g->l0_key.p, g->l0_dict.p, g->l0_flags.p);
    if (key_tiled) {
      const L0KeyPlan kp{reinterpret_cast<const uint4*>(g->tp_meta.p), g->tp_rec.p, g->tp_halo.p, g->tp_period,
                         g->tp_period_rows};
      GROOT_LAUNCH(l0_key_tile_kernel, key_ctas, 256, 0, n, g->rp.p, g->col.p, feat, g->hd_threshold, kp, g->l0_slot.p,
                   g->l0_ctab.p, g->l0_dict.p, g->l0_flags.p);
    } else {
      GROOT_LAUNCH(l0_key_kernel, key_ctas, 256, 0, n, g->rp.p, g->col.p, feat, g->hd_threshold, g->l0_slot.p,
                   g->l0_ctab.p, g->l0_dict.p, g->l0_flags.p);
    }
    GROOT_LAUNCH(dict_finalize_kernel, 1, 1024, 0, g->l0_dict.p, g->l0_flags.p, *reinterpret_cast<const Layer0W*>(m->l0w),
                 g->l0_table.p, g->l0_idmap.p);
    GROOT_LAUNCH(l0_xlat_kernel, blocks_for(key_ctas * kDictLocal, 256), 256, 0, key_ctas, g->l0_ctab.p, g->l0_dict.p,
                 g->l0_idmap.p, g->l0_flags.p, g->l0_xlat.p);
    GROOT_LAUNCH(l0_ids_kernel, blocks_for((n + 3) / 4, 256, sms * 8), 256, 0, n, key_ctas * 8u,
                 key_tiled ? kTpRows : 32u * kL0KeyRows, g->l0_slot.p,
                 g->l0_xlat.p, g->l0_flags.p, g->l0_id.p);
    if (g->num_hd)
      GROOT_LAUNCH(l0_hd_ids_kernel, blocks_for(g->num_hd, 256), 256, 0, g->num_hd, g->hd_rows.p, g->l0_key.p,
                   g->l0_dict.p, g->l0_idmap.p, g->l0_flags.p, g->l0_id.p);
    GROOT_LAUNCH(l0_halo_ids_kernel, blocks_for(ntiles * 32ull, 256, sms * 16), 256, 0,
                 ntiles, reinterpret_cast<const uint4*>(g->tp_meta.p), g->tp_halo.p, g->tp_period, g->tp_period_rows,
                 g->l0_id.p, g->l0_flags.p, g->l0_hid.p);
  }
  if (g->l0_mode == 0) {
    uint32_t fl[2] = {0, 0};
    g->l0_flags.download(fl, 2);
    stream_sync();
    g->l0_mode = fl[0] ? 2 : 1;
  }
  return g->l0_mode == 1;
}

void layer_device(const groot_model* m, groot_graph* g, uint32_t l, const float* hin, float* hout, uint8_t* cls,
                  float* logits, uint32_t tile_begin, uint32_t tile_end, bool hd_means, bool keyed_in) {
  const uint32_t n = g->n;
  if (n == 0) return;
  keyed_in = keyed_in && l == 1;
  if (keyed_in) hin = g->l0_table.p;
  HdInfo hd{g->hd_rows.p, g->num_hd, g->hd_threshold, g->hd_mean.p};
  const unsigned sms = static_cast<unsigned>(num_sms());
  if (l == 0) {
    if (g->num_hd) {
      ProfScope ps("hd_mean_feat");
      GROOT_LAUNCH(hd_mean_feat_kernel, std::min<uint32_t>(g->num_hd, sms * 8), 256, 0, g->hd_rows.p, g->num_hd,
                   g->rp.p, g->col.p, reinterpret_cast<const uint32_t*>(g->feat.p), g->hd_mean.p);
    }
    Layer0Args l0{n, g->rp.p, g->col.p, reinterpret_cast<const uint32_t*>(g->feat.p), hd, hout, g->binary_feat ? 1u : 0u};
    {
      ProfScope ps("sage_layer0");
      GROOT_LAUNCH(sage_layer0_kernel, blocks_for(n, kL0Threads, sms * 8), kL0Threads, 0, l0,
                   *reinterpret_cast<const Layer0W*>(m->l0w));
    }
    if (m->depth == 1)
      GROOT_LAUNCH(head_kernel, blocks_for(n, 256), 256, 0, n, hout, m->head.p, m->classes, cls, logits,
                   g->labels.p, nullptr);
    return;
  }
  const uint32_t ntiles = (n + kTileM - 1) / kTileM;
  // keyed layer 1 with layers after it: transform first (kModeXform)
  const char* xe = std::getenv("GROOT_L1_XFORM");
  const bool xform = keyed_in && l + 1 < m->depth && !(xe && std::atoi(xe) == 0);
  if (xform) {
    if (!g->l0_xtab.p) g->l0_xtab.alloc(2ull * kTkTableRows * kF);
    g->l0_xtab.zero();
    const float* w1 = m->naive_w.p + (2 * m->in_dim * kF + kF);  // layer 1: W_self, W_neigh, b
    ProfScope ps("l1_xform");
    GROOT_LAUNCH(l1_xform_kernel, kTkTableRows, 64, 0, g->l0_table.p, w1, w1 + kF * kF, w1 + 2 * kF * kF, g->l0_flags.p,
                 g->l0_xtab.p,
                 g->l0_xtab.p + kTkTableRows * kF);
  }
  const float* hd_src = xform ? g->l0_xtab.p : hin;  // (xform: HD means of Tn rows)
  if (g->num_hd && hd_means) {
    ProfScope ps("hd_mean32");
    hd_means32(g, hd_src, g->hd_mean.p, 0, keyed_in ? g->l0_id.p : nullptr);
  }
  LayerArgs a = plan_args(g, hin, hd);
  if (keyed_in) {
    a.keys = g->l0_id.p;
    a.hids = g->l0_hid.p;
    a.ktable = xform ? g->l0_xtab.p : g->l0_table.p;
    a.ktable_self = g->l0_xtab.p + kTkTableRows * kF;
  }
  a.tile_begin = std::min(tile_begin, ntiles);
  a.tile_end = std::min(tile_end, ntiles);
  a.hout = hout;
  a.bimg = m->bimg.p + static_cast<size_t>(l - 1) * (kBBytes / 4);
  a.hbimg = m->hbimg.p;
  {
    const char* hc = std::getenv("GROOT_HEAD_CERT_SCALE");  // test knob: route rows to the exact head
    a.head_cert = hc ? static_cast<float>(std::atof(hc)) : 1.0f;
  }
  a.classes = m->classes;
  a.cls = cls;
  a.logits = logits;
  const unsigned grid = std::max<uint32_t>(1u, std::min<uint32_t>(a.tile_end - a.tile_begin, sms));
  const CUtensorMap tmap_in = make_rows32_tmap(const_cast<float*>(hin), keyed_in ? kTkTableRows : n, kTileM);
  HeadW hw = *reinterpret_cast<const HeadW*>(m->headw);
  std::memcpy(hw.bias, m->bias_h.data() + static_cast<size_t>(l - 1) * kF, sizeof(hw.bias));
  static const char* trace_path = std::getenv("GROOT_TRACE");
  DevBuf<unsigned long long> trace;
  static const uint32_t trace_layer = env_u32("GROOT_TRACE_LAYER", 1);
  if (trace_path && l == trace_layer) {
    trace.alloc(64 * 16);
    trace.zero();
    a.trace = trace.p;
  }
  if (xform) {
    ProfScope ps("sage_layer1_xform");
    GROOT_LAUNCH((sage_tile_kernel<kModeXform, true>), grid, kThreads, TkCfg<true>::kSmem, a, hw, tmap_in);
  } else if (l + 1 == m->depth) {
    ProfScope ps("sage_layer_tc_last");
    if (keyed_in)
      GROOT_LAUNCH((sage_tile_kernel<kModeLast, true>), grid, kThreads, TkCfg<true>::kSmem, a, hw, tmap_in);
    else
      GROOT_LAUNCH(sage_tile_kernel<kModeLast>, grid, kThreads, TkCfg<false>::kSmem, a, hw, tmap_in);
  } else {
    ProfScope ps(keyed_in ? "sage_layer_tc_keyed" : "sage_layer_tc");
    if (keyed_in)
      GROOT_LAUNCH((sage_tile_kernel<kModeLayer, true>), grid, kThreads, TkCfg<true>::kSmem, a, hw, tmap_in);
    else
      GROOT_LAUNCH(sage_tile_kernel<kModeLayer>, grid, kThreads, TkCfg<false>::kSmem, a, hw, tmap_in);
  }
  if (a.trace) {
    std::vector<unsigned long long> h(64 * 16);
    trace.download(h.data(), h.size());
    stream_sync();
    if (FILE* fp = std::fopen(trace_path, "w")) {
      for (int i = 0; i < 64; ++i) {
        for (int k = 0; k < 16; ++k) std::fprintf(fp, "%llu ", h[i * 16 + k]);
        std::fprintf(fp, "\n");
      }
      std::fclose(fp);
    }
  }
}

void layer_prepare(const groot_model* m, groot_graph* g) {
  if (g->n) prepare_graph(m, g);
}

// Full forward + classify on a resident graph. cls: u8[n] device; logits:
// f32[n*classes] device or null; confusion: u64[25] device or null.
void forward_device(const groot_model* m, groot_graph* g, uint8_t* cls, float* logits, unsigned long long* confusion) {
  require(m->in_dim == 4 && m->hidden == kF, "forward: model shape unsupported (in_dim 4, hidden 32)");
  if (g->n == 0) return;
  prepare_graph(m, g);
  ensure_activations(g);
  const bool keyed = layer0_keyed(m, g);
  for (uint32_t l = keyed ? 1 : 0; l < m->depth; ++l)
    layer_device(m, g, l, l ? g->act[(l - 1) & 1].p : nullptr, l + 1 < m->depth || m->depth == 1 ? g->act[l & 1].p : nullptr,
                 cls, logits, 0, ~0u, true, keyed);
  if (confusion) {
    ProfScope ps("confusion");
    GROOT_LAUNCH(confusion_kernel, blocks_for(g->n / 16 + 1, 256, static_cast<unsigned>(num_sms()) * 8), 256, 0, g->n, cls,
                 g->labels.p, confusion);
  }
}

// Copy stream of the current device (created once, non-blocking): class
// read-back of the e2e call and encode's label upload overlap the main stream.
cudaStream_t side_stream() {
  static std::mutex side_mu;
  static cudaStream_t side_of[kMaxDevices] = {};
  const int dev = current_device();
  std::lock_guard<std::mutex> lk(side_mu);
  if (!side_of[dev]) GROOT_CUDA(cudaStreamCreateWithFlags(&side_of[dev], cudaStreamNonBlocking));
  return side_of[dev];
}

// Forward + classify of a tile-aligned batch (batch_padded: copy k at rows
// k*P .. k*P + n1) with the class read-back overlapped: the last layer runs
// as kReadbackParts launches over consecutive tile ranges, and the classes of
// the rows each range completes go to the host on a side stream while the
// next range computes. labels_out is in the reference's numbering (k*n1 + v).
void forward_classify_to_host(const groot_model* m, groot_graph* g, uint8_t* cls, unsigned long long* confusion,
                              uint32_t copies, uint32_t n1, uint32_t P, uint8_t* labels_out) {
  require(m->in_dim == 4 && m->hidden == kF, "forward: model shape unsupported (in_dim 4, hidden 32)");
  if (g->n == 0) return;
  prepare_graph(m, g);
  ensure_activations(g);
  const uint32_t D = m->depth;
  const bool keyed = layer0_keyed(m, g);
  for (uint32_t l = keyed ? 1 : 0; l + 1 < D; ++l)
    layer_device(m, g, l, l ? g->act[(l - 1) & 1].p : nullptr, g->act[l & 1].p, cls, nullptr, 0, ~0u, true, keyed);
  // read-back stream: one per device (created once); events per call, so
  // concurrent calls on different devices or threads share nothing
  cudaStream_t side = side_stream();
  Event evh, evs;
  cudaEvent_t ev_half = evh.e, ev_side = evs.e;
  // the last layer in tile ranges of shrinking size: the classes of the rows a
  // range completes go to the host on the side stream while the next ranges
  // compute, so only the last (3 %) range's classes are read after the layer
  // (beside the confusion count).
  // Row r of copy k (device row k*P + r) is host row k*n1 + r.
  static const uint32_t single = env_u32("GROOT_READBACK_SINGLE", 0);  // experiment: one launch, read-back after it
  const uint32_t kReadbackParts = single ? 1u : 9u;
  static constexpr uint16_t kEnd9[9] = {250, 450, 600, 720, 820, 890, 940, 970, 1000};  // per mille of tiles
  const uint16_t* kEnd = single ? kEnd9 + 8 : kEnd9;
  auto readback = [&](uint64_t r0, uint64_t r1, cudaStream_t st) {  // device rows [r0, r1), padding rows skipped
    for (uint64_t k = r0 / P; k < copies && k * P < r1; ++k) {
      const uint64_t a = std::max<uint64_t>(r0, k * P), b = std::min<uint64_t>(r1, k * P + n1);
      if (a < b)
        GROOT_CUDA(cudaMemcpyAsync(labels_out + k * n1 + (a - k * P), cls + a, b - a, cudaMemcpyDeviceToHost, st));
    }
  };
  uint64_t done = 0;  // device rows whose classes are on their way to the host
  if (D == 1) {
    layer_device(m, g, 0, nullptr, g->act[0].p, cls, nullptr, 0, ~0u, true, false);
  } else {
    const float* hin = g->act[(D - 2) & 1].p;
    const uint32_t ntiles = (g->n + kTileM - 1) / kTileM;
    bool first = true;  // the first launch also computes the layer's HD-row means
    for (uint32_t part = 0; part < kReadbackParts; ++part) {
      const uint32_t tb = part ? static_cast<uint32_t>(static_cast<uint64_t>(ntiles) * kEnd[part - 1] / 1000) : 0u;
      const uint32_t te = part + 1 == kReadbackParts ? ~0u : static_cast<uint32_t>(static_cast<uint64_t>(ntiles) * kEnd[part] / 1000);
      if (te != ~0u && te <= tb) continue;  // empty range (small graphs)
      layer_device(m, g, D - 1, hin, nullptr, cls, nullptr, tb, te, first, keyed);
      first = false;
      if (!labels_out) continue;
      const uint64_t rows_done =
          part + 1 == kReadbackParts ? g->n : std::min<uint64_t>(static_cast<uint64_t>(te) * kTileM, g->n);
      GROOT_CUDA(cudaEventRecord(ev_half, stream()));
      GROOT_CUDA(cudaStreamWaitEvent(side, ev_half, 0));
      readback(done, rows_done, side);
      done = rows_done;
    }
    if (done) GROOT_CUDA(cudaEventRecord(ev_side, side));
  }
  if (labels_out && done < g->n) readback(done, g->n, stream());  // depth 1: one launch
  if (confusion) {  // overlaps the read-back of the last range
    ProfScope ps("confusion");
    GROOT_LAUNCH(confusion_kernel, blocks_for(g->n / 16 + 1, 256, static_cast<unsigned>(num_sms()) * 8), 256, 0, g->n, cls,
                 g->labels.p, confusion);
  }
  if (done) GROOT_CUDA(cudaStreamWaitEvent(stream(), ev_side, 0));
}

// confusion[truth][pred] += over rows (device counts; labels >= 5 are skipped)
void confusion_device(uint32_t n, const uint8_t* cls, const uint8_t* labels, unsigned long long* conf) {
  if (n == 0) return;
  ProfScope ps("confusion");
  GROOT_LAUNCH(confusion_kernel, blocks_for(n / 16 + 1, 256, static_cast<unsigned>(num_sms()) * 8), 256, 0, n, cls,
               labels, conf);
}

// Naive path (tests): same math, thread per row, plain loads.
void forward_naive_device(const groot_model* m, groot_graph* g, uint8_t* cls, float* logits,
                          unsigned long long* confusion) {
  ensure_activations(g);
  const uint32_t n = g->n;
  if (n == 0) return;
  const float* w = m->naive_w.p;
  uint32_t in = m->in_dim;
  size_t off = 0;
  for (uint32_t l = 0; l < m->depth; ++l) {
    const float* ws = w + off;
    const float* wn = ws + in * 32;
    const float* b = wn + in * 32;
    off += 2 * in * 32 + 32;
    GROOT_LAUNCH(naive_layer_kernel, blocks_for(n, 128), 128, 0, n, g->rp.p, g->col.p,
                 l ? g->act[(l - 1) & 1].p : nullptr, reinterpret_cast<const uint32_t*>(g->feat.p), in, ws, wn, b,
                 g->act[l & 1].p);
    in = 32;
  }
  GROOT_LAUNCH(head_kernel, blocks_for(n, 256), 256, 0, n, g->act[(m->depth - 1) & 1].p, m->head.p, m->classes, cls,
               logits, g->labels.p, confusion);
}

void spmm_mean_device(groot_graph* g, const float* dense, uint32_t f, float* out) {
  if (g->n == 0) return;
  if (f == kF) {
    classify_rows(g, hd_threshold());
    HdInfo hd{g->hd_rows.p, g->num_hd, g->hd_threshold, g->hd_mean.p};
    const unsigned sms = static_cast<unsigned>(num_sms());
    if (g->num_hd) {
      ProfScope ps("spmm_hd_mean32");
      hd_means32(g, dense, out, 1);
    }
    set_tc_smem();
    build_tile_plan(g, hd.threshold);
    ProfScope ps("spmm_mean32");
    LayerArgs a = plan_args(g, dense, hd);
    a.spmm_out = out;
    a.tile_begin = 0;
    a.tile_end = (g->n + kTileM - 1) / kTileM;
    const CUtensorMap tmap_in = make_rows32_tmap(const_cast<float*>(dense), g->n, kTileM);
    const uint32_t ntiles = (g->n + kTileM - 1) / kTileM;
    HeadW hw{};
    GROOT_LAUNCH(sage_tile_kernel<kModeSpmm>, std::min<uint32_t>(ntiles, sms), kThreads, TkCfg<false>::kSmem, a, hw, tmap_in);
  } else {
    GROOT_LAUNCH(spmm_generic_kernel<float>, blocks_for(g->n, 32, num_sms() * 16), 256, 0, g->n, g->rp.p, g->col.p,
                 nullptr, dense, f, out, 0u);
  }
}

void spmm_csr_device(uint32_t rows, const uint32_t* rp, const uint32_t* col, const float* vals, const float* dense,
                     uint32_t f, float* out, uint32_t hd_threshold) {
  if (rows == 0) return;
  GROOT_LAUNCH(spmm_generic_kernel<float>, blocks_for(rows, 32, num_sms() * 16), 256, 0, rows, rp, col, vals, dense, f, out,
               hd_threshold);
}

void spmm_csr_device_f64(uint32_t rows, const uint32_t* rp, const uint32_t* col, const double* vals,
                         const double* dense, uint32_t f, double* out, uint32_t hd_threshold) {
  if (rows == 0) return;
  GROOT_LAUNCH(spmm_generic_kernel<double>, blocks_for(rows, 32, num_sms() * 16), 256, 0, rows, rp, col, vals, dense, f,
               out, hd_threshold);
}

// make_context (src/gnn.cpp:140-170) on the device: everything the forward
// derives from the graph alone -- the row classifier (HD band), the tile plan,
// the HD chunk plan and the activation buffers -- built once and cached on the
// handle until graph_release_context.
void graph_prepare(groot_graph* g) {
  set_tc_smem();
  classify_rows(g, hd_threshold());
  if (g->n) {
    build_tile_plan(g, g->hd_threshold);
    build_hd_plan(g);
  }
  ensure_activations(g);
  stream_sync();
}

void graph_release_context(groot_graph* g) {
  stream_sync();
  g->hd_threshold = 0;
  g->num_hd = 0;
  g->hd_rows.release();
  g->hd_mean.release();
  for (auto& b : g->act) b.release();
  g->tp_threshold = g->tp_halo_cap = g->tp_slow = 0;
  g->tp_period = g->tp_period_rows = 0;
  g->tp_meta.release();
  g->tp_lrp.release();
  g->tp_lcol.release();
  g->tp_rec.release();
  g->tp_halo.release();
  g->hdp_valid = false;
  g->hdp_nunits = 0;
  g->hdp_base.release();
  g->hdp_slot.release();
  g->hdp_k.release();
  g->hdp_units.release();
  g->hdp_partial.release();
  g->l0_mode = 0;
}

// Host-side TF32 split (round-to-nearest, ties away — same as cvt.rna.tf32.f32).
static float tf32_rna_host(float x) {
  uint32_t u;
  std::memcpy(&u, &x, 4);
  if ((u & 0x7F800000u) != 0x7F800000u) u = (u + 0x1000u) & 0xFFFFE000u;
  float r;
  std::memcpy(&r, &u, 4);
  return r;
}

// Build device weights: layer 0 fp32, layers >= 1 as swizzled smem images
// (B operand K-major: row n = output feature, K = input feature).
void model_upload(groot_model* m) {
  const uint32_t D = m->depth, H = m->hidden, C = m->classes, I = m->in_dim;
  const double* p = m->params.data();
  std::vector<float> l0(2 * I * H + H);
  for (size_t i = 0; i < l0.size(); ++i) l0[i] = static_cast<float>(p[i]);
  static_assert(sizeof(Layer0W) == sizeof(m->l0w), "layer-0 parameter block");
  std::memcpy(m->l0w, l0.data(), sizeof(m->l0w));
  m->l0.alloc(l0.size());
  m->l0.upload(l0.data(), l0.size());
  // naive path: all layers fp32 row-major, then head
  std::vector<float> nw;
  size_t off = 0;
  uint32_t in = I;
  std::vector<uint32_t> img(static_cast<size_t>(D > 1 ? D - 1 : 0) * (kBBytes / 4), 0);
  std::vector<float> bias(static_cast<size_t>(D > 1 ? D - 1 : 0) * H);
  for (uint32_t l = 0; l < D; ++l) {
    const double* ws = p + off;
    const double* wn = ws + in * H;
    const double* b = wn + in * H;
    for (uint32_t i = 0; i < 2 * in * H + H; ++i) nw.push_back(static_cast<float>(ws[i]));
    if (l > 0) {
      uint8_t* base = reinterpret_cast<uint8_t*>(img.data()) + static_cast<size_t>(l - 1) * kBBytes;
      for (int kb = 0; kb < 2; ++kb) {
        const double* W = kb ? wn : ws;
        for (uint32_t nn = 0; nn < 32; ++nn)
          for (uint32_t k = 0; k < 32; ++k) {
            const float v = static_cast<float>(W[kcol_feature(k) * H + kcol_feature(nn)]);  // K and N permuted
            const float hi = tf32_rna_host(v), lo = v - hi;
            const uint32_t o = nn * 128 + (((k >> 2) ^ (nn & 7)) << 4) + (k & 3) * 4;
            std::memcpy(base + kb * 8192 + o, &hi, 4);
            std::memcpy(base + kb * 8192 + 4096 + o, &lo, 4);
          }
      }
      for (uint32_t o = 0; o < H; ++o) bias[(l - 1) * H + o] = static_cast<float>(b[o]);
    }
    off += 2 * in * H + H;
    in = H;
  }
  std::vector<float> head(H * C + C);
  for (uint32_t i = 0; i < H * C + C; ++i) head[i] = static_cast<float>(p[off + i]);
  static_assert(sizeof(HeadW) == sizeof(m->headw), "head parameter block");
  m->bias_h = bias;
  HeadW hw{};
  for (uint32_t k = 0; k < H; ++k)
    for (uint32_t c = 0; c < C; ++c) hw.w[k][c] = head[k * C + c];
  for (uint32_t c = 0; c < C; ++c) hw.b[c] = head[H * C + c];
  std::memcpy(m->headw, &hw, sizeof(hw));
  // head B image for the last layer's tensor-core head: row n = class (zero
  // rows past C), K element c = hidden feature kcol_feature(c) (the
  // accumulator's column order), TF32 hi | lo, K-major 128-B swizzle
  std::vector<uint32_t> himg(kHeadBBytes / 4, 0);
  for (uint32_t nn = 0; nn < kHeadN; ++nn)
    for (uint32_t k = 0; k < 32; ++k) {
      // rows 8 + c: |W_c| (the certified head's bound sums, GROOT_HEAD_CERT)
      const float v = nn < C ? head[kcol_feature(k) * C + nn]
                             : (nn >= 8 && nn - 8 < C ? std::fabs(head[kcol_feature(k) * C + nn - 8]) : 0.0f);
      const float hi = tf32_rna_host(v), lo = v - hi;
      const uint32_t o = nn * 128 + (((k >> 2) ^ (nn & 7)) << 4) + (k & 3) * 4;
      std::memcpy(reinterpret_cast<uint8_t*>(himg.data()) + o, &hi, 4);
      std::memcpy(reinterpret_cast<uint8_t*>(himg.data()) + kHeadN * 128 + o, &lo, 4);
    }
  m->hbimg.alloc(himg.size());
  m->hbimg.upload(himg.data(), himg.size());
  m->bimg.alloc(img.size());
  m->bimg.upload(img.data(), img.size());
  m->bias.alloc(bias.size());
  m->bias.upload(bias.data(), bias.size());
  m->head.alloc(head.size());
  m->head.upload(head.data(), head.size());
  m->naive_w.alloc(nw.size());
  m->naive_w.upload(nw.data(), nw.size());
  stream_sync();
}

}  // namespace groot
