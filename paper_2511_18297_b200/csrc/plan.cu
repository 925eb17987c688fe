// plan.cu — build_plan (src/spmm.cpp:37-127) for API parity.
//
// The device hot path does not permute rows: it keeps the natural (index-local)
// row order for LD rows and routes only the HD band through classify_rows()
// (forward.cu). This entry point reproduces the reference's SpmmPlan exactly —
// the stable degree sort runs on the device (radix sort of (degree,row) pairs,
// stable == counting sort order), the band/unit enumeration over the sorted
// degrees runs on the host (O(rows/budget) units).
#include <cub/cub.cuh>

#include <algorithm>

#include "common.cuh"

namespace groot {

__global__ void degree_pairs_kernel(uint32_t n, const uint32_t* __restrict__ rp, uint32_t* __restrict__ deg,
                                    uint32_t* __restrict__ ids) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    deg[v] = rp[v + 1] - rp[v];
    ids[v] = v;
  }
}

}  // namespace groot

using namespace groot;

// degree_sort (src/spmm.cpp:9-35): stable ascending order of rows by degree
// on the device (radix sort of (degree, row) pairs; stable == counting-sort
// order). Returns sorted degrees and perm[sorted] = original row on the host.
static void degree_sort_dev(uint32_t n, const uint32_t* d_rp, std::vector<uint32_t>& hdeg,
                            std::vector<uint32_t>& hperm) {
  hdeg.assign(n, 0);
  hperm.assign(n, 0);
  if (!n) return;
  DevBuf<uint32_t> deg(n), ids(n), sdeg(n), perm(n);
  GROOT_LAUNCH(degree_pairs_kernel, blocks_for(n, 256), 256, 0, n, d_rp, deg.p, ids.p);
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, deg.p, sdeg.p, ids.p, perm.p, n, 0, 32, stream());
  DevBuf<uint8_t> tmp(bytes);
  GROOT_CUDA(cub::DeviceRadixSort::SortPairs(tmp.p, bytes, deg.p, sdeg.p, ids.p, perm.p, n, 0, 32, stream()));
  sdeg.download(hdeg.data(), n);
  perm.download(hperm.data(), n);
  stream_sync();
}

// Host row_ptr (u64, the reference's CsrMatrix::row_ptr) -> validated device u32 copy.
static void upload_row_ptr(uint32_t rows, const uint64_t* row_ptr, DevBuf<uint32_t>& d_rp) {
  if (!row_ptr) fail(GROOT_EINVAL, "build_plan: null row_ptr");
  if (row_ptr[rows] >= 0xFFFFFFFFull) fail(GROOT_EINVAL, "build_plan: nnz must be < 2^32");
  std::vector<uint32_t> rp32(rows + 1ull);
  for (uint32_t r = 0; r <= rows; ++r) {
    if (r && row_ptr[r] < row_ptr[r - 1]) fail(GROOT_EINVAL, "CsrMatrix: row_ptr not monotone");
    rp32[r] = static_cast<uint32_t>(row_ptr[r]);
  }
  d_rp.alloc(rows + 1ull);
  d_rp.upload(rp32.data(), rows + 1ull);
}

static void build_plan_impl(uint32_t n, const uint32_t* d_rp, uint32_t hd, uint32_t ld, uint32_t budget,
                            uint64_t* counts, uint32_t* perm_out, uint32_t* hd_rows, uint32_t* mid_rows,
                            uint32_t* ld_groups, uint64_t* units) {
    if (ld < 1 || budget < 1) fail(GROOT_EINVAL, "build_plan: thresholds must be >= 1");
    if (hd <= ld) fail(GROOT_EINVAL, "build_plan: hd_threshold must exceed ld_threshold");
    std::vector<uint32_t> hdeg, hperm;
    degree_sort_dev(n, d_rp, hdeg, hperm);
    std::vector<uint32_t> rp(n + 1ull);
    if (n) {
      GROOT_CUDA(cudaMemcpyAsync(rp.data(), d_rp, (n + 1ull) * 4, cudaMemcpyDeviceToHost, stream()));
      stream_sync();
    }
    uint32_t z = 0;
    while (z < n && hdeg[z] == 0) ++z;
    uint32_t le = z;
    while (le < n && hdeg[le] <= ld) ++le;
    uint32_t me = le;
    while (me < n && hdeg[me] < hd) ++me;
    std::vector<uint64_t> u;
    std::vector<uint32_t> hdv, midv, ldg;
    for (uint32_t s = me; s < n; ++s) hdv.push_back(s);
    for (size_t i = 0; i < hdv.size(); ++i) {  // 32 chunks per HD row, remainder on trailing chunks
      const uint32_t r = hperm[hdv[i]];
      const uint32_t wid = rp[r + 1] - rp[r], q = wid / 32, rem = wid % 32;
      uint64_t nz = rp[r];
      for (uint32_t c = 0; c < 32; ++c) {
        const uint32_t len = q + (c >= 32 - rem ? 1 : 0);
        u.insert(u.end(), {0ull, hdv[i], 1ull, nz, nz + len, i * 32ull + c});
        nz += len;
      }
    }
    for (uint32_t s = me; s-- > le;) {  // MID rows, largest degree first
      midv.push_back(s);
      u.insert(u.end(), {2ull, s, 1ull, 0ull, 0ull, 0ull});
    }
    for (uint32_t s = z; s < le;) {  // LD groups: floor(budget/d) rows per unit
      const uint32_t d = hdeg[s];
      uint32_t ge = s;
      while (ge < le && hdeg[ge] == d) ++ge;
      ldg.insert(ldg.end(), {d, s, ge});
      const uint32_t per = std::max<uint32_t>(1, budget / d);
      for (uint32_t r0 = s; r0 < ge; r0 += per)
        u.insert(u.end(), {1ull, r0, static_cast<uint64_t>(std::min(per, ge - r0)), 0ull, 0ull, 0ull});
      s = ge;
    }
    if (counts) {
      counts[0] = hdv.size();
      counts[1] = midv.size();
      counts[2] = ldg.size() / 3;
      counts[3] = u.size() / 6;
      counts[4] = z;
      counts[5] = le;
    }
    if (perm_out) std::copy(hperm.begin(), hperm.end(), perm_out);
    if (hd_rows) std::copy(hdv.begin(), hdv.end(), hd_rows);
    if (mid_rows) std::copy(midv.begin(), midv.end(), mid_rows);
    if (ld_groups) std::copy(ldg.begin(), ldg.end(), ld_groups);
    if (units) std::copy(u.begin(), u.end(), units);
}

extern "C" int groot_build_plan(const groot_graph* g, uint32_t hd, uint32_t ld, uint32_t budget, uint64_t* counts,
                                uint32_t* perm_out, uint32_t* hd_rows, uint32_t* mid_rows, uint32_t* ld_groups,
                                uint64_t* units) {
  return guarded([&] {
    if (!g) fail(GROOT_EINVAL, "groot_build_plan: null argument");
    DeviceScope ds(g->device);
    build_plan_impl(g->n, g->rp.p, hd, ld, budget, counts, perm_out, hd_rows, mid_rows, ld_groups, units);
  });
}

extern "C" int groot_build_plan_rows(uint32_t rows, const uint64_t* row_ptr, uint32_t hd, uint32_t ld,
                                     uint32_t budget, uint64_t* counts, uint32_t* perm_out, uint32_t* hd_rows,
                                     uint32_t* mid_rows, uint32_t* ld_groups, uint64_t* units) {
  return guarded([&] {
    DevBuf<uint32_t> d_rp;
    upload_row_ptr(rows, row_ptr, d_rp);
    build_plan_impl(rows, d_rp.p, hd, ld, budget, counts, perm_out, hd_rows, mid_rows, ld_groups, units);
  });
}

extern "C" int groot_degree_sort(uint32_t rows, const uint64_t* row_ptr, uint32_t* perm_out,
                                 uint64_t* sorted_row_ptr) {
  return guarded([&] {
    DevBuf<uint32_t> d_rp;
    upload_row_ptr(rows, row_ptr, d_rp);
    std::vector<uint32_t> hdeg, hperm;
    degree_sort_dev(rows, d_rp.p, hdeg, hperm);
    if (perm_out) std::copy(hperm.begin(), hperm.end(), perm_out);
    if (sorted_row_ptr) {  // row pointers in the sorted order (src/spmm.cpp:28-33)
      sorted_row_ptr[0] = 0;
      for (uint32_t s = 0; s < rows; ++s) sorted_row_ptr[s + 1] = sorted_row_ptr[s] + hdeg[s];
    }
  });
}
