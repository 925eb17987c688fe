// oracle.cpp — CPU restatement of the reference hot path (TEST INFRASTRUCTURE).
//
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg load
// this library, and only as the checker. The product never calls it.
//
// Each function below restates one reference function; citations are
// /root/reference/proj/core/{src,include/aigsage}/<file>:<line>. The code is
// written over flat arrays (AIGER literals 2v+inv, CSR with u64 row pointers)
// rather than the reference's classes, but it keeps every ordering rule that
// the reference's outputs depend on (node creation order, edge order, per-row
// sort, boundary order, accumulation order of the SpMM).
#include "oracle.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <optional>
#include <random>
#include <stdexcept>
#include <string>
#include <thread>
#include <utility>
#include <vector>

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

constexpr uint8_t kPo = 0, kMaj = 1, kXor = 2, kAnd = 3, kPi = 4;

inline uint32_t lit_not(uint32_t l) { return l ^ 1u; }

// ---------------------------------------------------------------------------
// circuitgen (src/circuitgen.cpp:13-133)
// ---------------------------------------------------------------------------
struct CsaBuilder {
  uint32_t inputs;
  std::vector<uint32_t> ands;  // left, right literal pairs
  std::vector<uint8_t> labels;
  uint32_t half = 0, full = 0;

  explicit CsaBuilder(uint32_t ni) : inputs(ni) {
    // AigBuilder ctor (src/circuitgen.cpp:13-17): node 0 labelled AND, PIs PI.
    labels.assign(1 + ni, kAnd);
    for (uint32_t i = 1; i <= ni; ++i) labels[i] = kPi;
  }
  uint32_t make(uint32_t l, uint32_t r, uint8_t cls) {  // AigBuilder::add_and
    const uint32_t v = 1 + inputs + static_cast<uint32_t>(ands.size() / 2);
    ands.push_back(l);
    ands.push_back(r);
    labels.push_back(cls);
    return 2 * v;
  }
  // gen_half_adder (src/circuitgen.cpp:44-51): returns {sum, carry}
  std::pair<uint32_t, uint32_t> ha(uint32_t a, uint32_t b) {
    const uint32_t carry = make(a, b, kMaj);
    const uint32_t nor_ = make(lit_not(a), lit_not(b), kAnd);
    const uint32_t sum = make(lit_not(carry), lit_not(nor_), kXor);
    return {sum, carry};
  }
  // gen_full_adder (src/circuitgen.cpp:53-64): carry literal is ~MAJ root.
  std::pair<uint32_t, uint32_t> fa(uint32_t a, uint32_t b, uint32_t c) {
    const uint32_t c1 = make(a, b, kAnd);
    const uint32_t n1 = make(lit_not(a), lit_not(b), kAnd);
    const uint32_t x1 = make(lit_not(c1), lit_not(n1), kAnd);
    const uint32_t c2 = make(x1, c, kAnd);
    const uint32_t n2 = make(lit_not(x1), lit_not(c), kAnd);
    const uint32_t sum = make(lit_not(c2), lit_not(n2), kXor);
    const uint32_t mj = make(lit_not(c1), lit_not(c2), kMaj);
    return {sum, lit_not(mj)};
  }
  // `reduce` lambda (src/circuitgen.cpp:78-88)
  std::pair<uint32_t, std::optional<uint32_t>> reduce(const std::vector<uint32_t>& in) {
    if (in.size() == 1) return {in[0], std::nullopt};
    if (in.size() == 2) {
      ++half;
      auto [s, c] = ha(in[0], in[1]);
      return {s, c};
    }
    if (in.size() != 3) throw std::runtime_error("gen_csa: column reduction with no inputs");
    ++full;
    auto [s, c] = fa(in[0], in[1], in[2]);
    return {s, c};
  }
};

struct CsaResult {
  uint32_t inputs;
  std::vector<uint32_t> ands, outs;
  std::vector<uint8_t> labels;
};

CsaResult gen_csa(uint32_t w) {
  if (w < 2) throw std::invalid_argument("gen_csa_multiplier: width must be >= 2");
  CsaBuilder b(2 * w);
  auto pp = [&](uint32_t i, uint32_t j) { return b.make(2 * (i + 1), 2 * (w + j + 1), kAnd); };
  std::vector<std::optional<uint32_t>> sums(2 * w), carries(2 * w);
  std::vector<uint32_t> m(2 * w, 0);
  m[0] = pp(0, 0);
  for (uint32_t j = 1; j < w; ++j) sums[j] = pp(0, j);
  for (uint32_t i = 1; i < w; ++i) {
    std::vector<std::optional<uint32_t>> ns(2 * w), nc(2 * w);
    for (uint32_t j = 0; j < w; ++j) {
      const uint32_t col = i + j;
      std::vector<uint32_t> in;
      if (sums[col]) in.push_back(*sums[col]);
      in.push_back(pp(i, j));  // partial product is created before the adder
      if (carries[col]) in.push_back(*carries[col]);
      auto [s, c] = b.reduce(in);
      if (j == 0) m[i] = s; else ns[col] = s;
      if (c) nc[col + 1] = *c;
    }
    sums.swap(ns);
    carries.swap(nc);
  }
  std::optional<uint32_t> ripple;
  for (uint32_t col = w; col < 2 * w; ++col) {
    std::vector<uint32_t> in;
    if (sums[col]) in.push_back(*sums[col]);
    if (carries[col]) in.push_back(*carries[col]);
    if (ripple) in.push_back(*ripple);
    auto [s, c] = b.reduce(in);
    m[col] = s;
    ripple = c;
  }
  CsaResult r;
  r.inputs = 2 * w;
  r.ands = std::move(b.ands);
  r.outs = m;
  r.labels = std::move(b.labels);
  for (size_t k = 0; k < m.size(); ++k) r.labels.push_back(kPo);  // AigBuilder::finish
  return r;
}

// ---------------------------------------------------------------------------
// encode (src/encode.cpp:14-68)
// ---------------------------------------------------------------------------
void build_csr(uint32_t n, uint64_t ne, const uint32_t* e, uint64_t* rp, uint32_t* ci) {
  std::fill(rp, rp + n + 1, 0);
  for (uint64_t i = 0; i < ne; ++i) {
    ++rp[e[2 * i] + 1];
    ++rp[e[2 * i + 1] + 1];
  }
  for (uint32_t v = 0; v < n; ++v) rp[v + 1] += rp[v];
  std::vector<uint64_t> cur(rp, rp + n);
  for (uint64_t i = 0; i < ne; ++i) {
    const uint32_t u = e[2 * i], v = e[2 * i + 1];
    ci[cur[u]++] = v;
    ci[cur[v]++] = u;
  }
  for (uint32_t v = 0; v < n; ++v) std::sort(ci + rp[v], ci + rp[v + 1]);
}

// ---------------------------------------------------------------------------
// partition (src/partition.cpp:402-456)
// ---------------------------------------------------------------------------
struct Part {
  std::vector<uint32_t> core, boundary;
  std::vector<uint32_t> edges;  // local-id pairs
};

// ---------------------------------------------------------------------------
// spmm (src/spmm.cpp:9-127; inc/spmm.hpp:51-181)
// ---------------------------------------------------------------------------
enum UnitKind : uint64_t { kHdChunk = 0, kLdBatch = 1, kMidRow = 2 };
struct Unit {
  uint64_t kind, sorted_row, row_count, nz_begin, nz_end, partial_slot;
};

void degree_sort(uint32_t rows, const uint64_t* rp, uint32_t* perm, uint64_t* srp) {
  uint32_t maxd = 0;
  for (uint32_t r = 0; r < rows; ++r) maxd = std::max<uint32_t>(maxd, static_cast<uint32_t>(rp[r + 1] - rp[r]));
  std::vector<uint32_t> slot(static_cast<size_t>(maxd) + 2, 0);
  for (uint32_t r = 0; r < rows; ++r) ++slot[(rp[r + 1] - rp[r]) + 1];
  for (size_t d = 1; d < slot.size(); ++d) slot[d] += slot[d - 1];
  for (uint32_t r = 0; r < rows; ++r) perm[slot[rp[r + 1] - rp[r]]++] = r;  // stable
  srp[0] = 0;
  for (uint32_t s = 0; s < rows; ++s) srp[s + 1] = srp[s] + (rp[perm[s] + 1] - rp[perm[s]]);
}

}  // namespace

struct orc_parts {
  std::vector<Part> parts;
};

struct orc_plan {
  uint32_t rows = 0;
  uint64_t nnz = 0;
  std::vector<uint32_t> perm;
  std::vector<uint64_t> srp;
  std::vector<uint32_t> hd_rows, mid_rows, ld_groups;
  std::vector<Unit> units;
  uint32_t ld_begin = 0, ld_end = 0;
};

namespace {

constexpr uint32_t kChunks = 32;  // kHdChunksPerRow, inc/spmm.hpp:90

orc_plan* make_plan(uint32_t rows, const uint64_t* rp, uint32_t hd, uint32_t ld, uint32_t budget) {
  if (ld < 1 || budget < 1) throw std::invalid_argument("build_plan: thresholds must be >= 1");
  if (hd <= ld) throw std::invalid_argument("build_plan: hd_threshold must exceed ld_threshold");
  auto* p = new orc_plan;
  p->rows = rows;
  p->nnz = rows ? rp[rows] : 0;
  p->perm.resize(rows);
  p->srp.resize(static_cast<size_t>(rows) + 1);
  degree_sort(rows, rp, p->perm.data(), p->srp.data());
  auto deg = [&](uint32_t s) { return static_cast<uint32_t>(p->srp[s + 1] - p->srp[s]); };
  uint32_t z = 0;
  while (z < rows && deg(z) == 0) ++z;
  uint32_t le = z;
  while (le < rows && deg(le) <= ld) ++le;
  uint32_t me = le;
  while (me < rows && deg(me) < hd) ++me;
  p->ld_begin = z;
  p->ld_end = le;
  for (uint32_t s = me; s < rows; ++s) p->hd_rows.push_back(s);
  for (size_t i = 0; i < p->hd_rows.size(); ++i) {
    const uint32_t r = p->perm[p->hd_rows[i]];
    const uint32_t wid = static_cast<uint32_t>(rp[r + 1] - rp[r]);
    const uint32_t q = wid / kChunks, rem = wid % kChunks;
    uint64_t nz = rp[r];
    for (uint32_t c = 0; c < kChunks; ++c) {
      const uint32_t len = q + (c >= kChunks - rem ? 1 : 0);  // remainder on trailing chunks
      p->units.push_back({kHdChunk, p->hd_rows[i], 1, nz, nz + len, i * kChunks + c});
      nz += len;
    }
  }
  for (uint32_t s = me; s-- > le;) {  // MID rows, largest degree first
    p->mid_rows.push_back(s);
    p->units.push_back({kMidRow, s, 1, 0, 0, 0});
  }
  for (uint32_t s = z; s < le;) {
    const uint32_t d = deg(s);
    uint32_t ge = s;
    while (ge < le && deg(ge) == d) ++ge;
    p->ld_groups.insert(p->ld_groups.end(), {d, s, ge});
    const uint32_t per = std::max<uint32_t>(1, budget / d);
    for (uint32_t r0 = s; r0 < ge; r0 += per)
      p->units.push_back({kLdBatch, r0, std::min(per, ge - r0), 0, 0, 0});
    s = ge;
  }
  return p;
}

// accumulate lambda (inc/spmm.hpp:117-124): dst = 0; dst += v*src in nonzero order.
inline void accum(double* dst, uint64_t b, uint64_t e, const uint32_t* ci, const double* val,
                  const double* dense, uint32_t f) {
  for (uint32_t c = 0; c < f; ++c) dst[c] = 0.0;
  for (uint64_t k = b; k < e; ++k) {
    const double v = val[k];
    const double* src = dense + static_cast<size_t>(ci[k]) * f;
    for (uint32_t c = 0; c < f; ++c) dst[c] += v * src[c];
  }
}

void plan_execute(const orc_plan& p, const uint64_t* rp, const uint32_t* ci, const double* val,
                  const double* dense, uint32_t f, double* out) {
  const size_t n_ld = p.ld_end - p.ld_begin;
  std::vector<double> staging(n_ld * f);
  std::vector<double> partials(p.hd_rows.size() * kChunks * f);
  std::fill(out, out + static_cast<size_t>(p.rows) * f, 0.0);
  for (const Unit& u : p.units) {  // phase 1 (inc/spmm.hpp:126-146)
    if (u.kind == kLdBatch) {
      for (uint64_t s = u.sorted_row; s < u.sorted_row + u.row_count; ++s) {
        const uint32_t r = p.perm[s];
        accum(staging.data() + (s - p.ld_begin) * f, rp[r], rp[r + 1], ci, val, dense, f);
      }
    } else if (u.kind == kMidRow) {
      const uint32_t r = p.perm[u.sorted_row];
      accum(out + static_cast<size_t>(r) * f, rp[r], rp[r + 1], ci, val, dense, f);
    } else {
      accum(partials.data() + u.partial_slot * f, u.nz_begin, u.nz_end, ci, val, dense, f);
    }
  }
  for (size_t i = 0; i < p.hd_rows.size(); ++i) {  // phase 2 (inc/spmm.hpp:150-157)
    double* dst = out + static_cast<size_t>(p.perm[p.hd_rows[i]]) * f;
    const double* pp = partials.data() + i * kChunks * f;
    for (uint32_t c = 0; c < kChunks; ++c)
      for (uint32_t j = 0; j < f; ++j) dst[j] += pp[c * f + j];
  }
  for (size_t s = p.ld_begin; s < p.ld_end; ++s)  // LD scatter (inc/spmm.hpp:158-160)
    std::memcpy(out + static_cast<size_t>(p.perm[s]) * f, staging.data() + (s - p.ld_begin) * f,
                f * sizeof(double));
}

// ---------------------------------------------------------------------------
// gnn (src/gnn.cpp)
// ---------------------------------------------------------------------------
struct Layer {
  uint32_t in, out;
  const double *ws, *wn, *b;  // row-major in x out
};
struct ModelView {
  std::vector<Layer> layers;
  const double *wout, *bout;
  uint32_t hidden, classes;
};

ModelView view_model(const double* prm, uint32_t depth, uint32_t in_dim, uint32_t hidden,
                     uint32_t classes) {
  ModelView m;
  m.hidden = hidden;
  m.classes = classes;
  uint32_t in = in_dim;
  const double* q = prm;
  for (uint32_t l = 0; l < depth; ++l) {
    Layer L{in, hidden, q, q + in * hidden, q + 2 * in * hidden};
    q += 2 * in * hidden + hidden;
    m.layers.push_back(L);
    in = hidden;
  }
  m.wout = q;
  m.bout = q + static_cast<size_t>(in) * classes;
  return m;
}

template <class F>
void parallel_rows(uint32_t n, unsigned threads, F&& f) {
  if (threads <= 1 || n < 4096) {
    f(0u, n);
    return;
  }
  std::vector<std::thread> pool;
  for (unsigned t = 0; t < threads; ++t) {
    const uint32_t b = static_cast<uint32_t>(static_cast<uint64_t>(n) * t / threads);
    const uint32_t e = static_cast<uint32_t>(static_cast<uint64_t>(n) * (t + 1) / threads);
    pool.emplace_back([&, b, e] { f(b, e); });
  }
  for (auto& th : pool) th.join();
}

// dense = a*W (row-major, k ascending), the Eigen product (src/gnn.cpp:46) restated.
inline void matvec(const double* a, const double* w, uint32_t in, uint32_t out, double* z) {
  for (uint32_t j = 0; j < out; ++j) {
    double s = 0.0;
    for (uint32_t k = 0; k < in; ++k) s += a[k] * w[static_cast<size_t>(k) * out + j];
    z[j] = s;
  }
}

struct Graph {
  uint32_t n;
  const uint64_t* rp;
  const uint32_t* ci;
};

// make_context values (src/gnn.cpp:147-157): a_mean = 1/deg(v) on row v.
std::vector<double> mean_values(const Graph& g) {
  std::vector<double> v(g.rp[g.n]);
  for (uint32_t r = 0; r < g.n; ++r) {
    const uint64_t d = g.rp[r + 1] - g.rp[r];
    const double inv = d > 0 ? 1.0 / static_cast<double>(d) : 0.0;
    for (uint64_t k = g.rp[r]; k < g.rp[r + 1]; ++k) v[k] = inv;
  }
  return v;
}

// Planned SpMM restated row-wise: rows below the HD threshold accumulate in
// nonzero order; HD rows sum 32 chunk partials in ascending chunk order. This
// equals plan_execute for the default plan, without materialising the plan.
void mean_aggregate(const Graph& g, const double* val, const double* h, uint32_t f, double* m,
                    unsigned threads) {
  parallel_rows(g.n, threads, [&](uint32_t b, uint32_t e) {
    std::vector<double> part(f);
    for (uint32_t r = b; r < e; ++r) {
      const uint64_t rb = g.rp[r], re = g.rp[r + 1];
      const uint32_t wid = static_cast<uint32_t>(re - rb);
      double* dst = m + static_cast<size_t>(r) * f;
      if (wid < 512) {
        accum(dst, rb, re, g.ci, val, h, f);
        continue;
      }
      for (uint32_t c = 0; c < f; ++c) dst[c] = 0.0;
      const uint32_t q = wid / kChunks, rem = wid % kChunks;
      uint64_t nz = rb;
      for (uint32_t c = 0; c < kChunks; ++c) {
        const uint32_t len = q + (c >= kChunks - rem ? 1 : 0);
        accum(part.data(), nz, nz + len, g.ci, val, h, f);
        for (uint32_t j = 0; j < f; ++j) dst[j] += part[j];
        nz += len;
      }
    }
  });
}

struct Cache {
  std::vector<std::vector<double>> h, m, z;
  std::vector<double> logits;
};

// run_forward (src/gnn.cpp:37-52)
void run_forward(const Graph& g, const uint8_t* feat, const ModelView& mv, uint32_t in_dim,
                 Cache& c, unsigned threads, bool keep) {
  const uint32_t n = g.n;
  const std::vector<double> val = mean_values(g);
  std::vector<double> h(static_cast<size_t>(n) * in_dim);
  for (size_t i = 0; i < h.size(); ++i) h[i] = feat[i];
  if (keep) c.h.push_back(h);
  for (const Layer& L : mv.layers) {
    std::vector<double> m(static_cast<size_t>(n) * L.in);
    mean_aggregate(g, val.data(), h.data(), L.in, m.data(), threads);
    std::vector<double> z(static_cast<size_t>(n) * L.out), hn(z.size());
    parallel_rows(n, threads, [&](uint32_t b, uint32_t e) {
      std::vector<double> t1(L.out), t2(L.out);
      for (uint32_t r = b; r < e; ++r) {
        matvec(&h[static_cast<size_t>(r) * L.in], L.ws, L.in, L.out, t1.data());
        matvec(&m[static_cast<size_t>(r) * L.in], L.wn, L.in, L.out, t2.data());
        for (uint32_t j = 0; j < L.out; ++j) {
          const double zz = (t1[j] + t2[j]) + L.b[j];
          z[static_cast<size_t>(r) * L.out + j] = zz;
          hn[static_cast<size_t>(r) * L.out + j] = zz > 0.0 ? zz : 0.0;  // cwiseMax(0)
        }
      }
    });
    if (keep) {
      c.m.push_back(std::move(m));
      c.z.push_back(std::move(z));
      c.h.push_back(hn);
    }
    h.swap(hn);
  }
  const uint32_t hid = mv.layers.back().out;
  c.logits.assign(static_cast<size_t>(n) * mv.classes, 0.0);
  parallel_rows(n, threads, [&](uint32_t b, uint32_t e) {
    for (uint32_t r = b; r < e; ++r) {
      double* o = &c.logits[static_cast<size_t>(r) * mv.classes];
      matvec(&h[static_cast<size_t>(r) * hid], mv.wout, hid, mv.classes, o);
      for (uint32_t j = 0; j < mv.classes; ++j) o[j] += mv.bout[j];
    }
  });
}

uint64_t param_count(uint32_t depth, uint32_t in_dim, uint32_t hidden, uint32_t classes) {
  uint64_t c = 0;
  uint32_t in = in_dim;
  for (uint32_t l = 0; l < depth; ++l) {
    c += 2ull * in * hidden + hidden;
    in = hidden;
  }
  return c + static_cast<uint64_t>(in) * classes + classes;
}

// init_model (src/gnn.cpp:113-138): Glorot U(+-sqrt(6/(in+out))) from
// mt19937_64(seed), row-major, order W_self, W_neigh per layer, then W_out.
void init_model(uint64_t seed, uint32_t in_dim, uint32_t hidden, uint32_t classes, uint32_t depth,
                double* prm) {
  if (depth < 1) throw std::invalid_argument("init_model: depth must be >= 1");
  std::mt19937_64 rng(seed);
  auto glorot = [&](uint32_t rows, uint32_t cols, double* dst) {
    const double lim = std::sqrt(6.0 / (rows + cols));
    std::uniform_real_distribution<double> dist(-lim, lim);
    for (uint32_t i = 0; i < rows * cols; ++i) dst[i] = dist(rng);
  };
  double* q = prm;
  uint32_t in = in_dim;
  for (uint32_t l = 0; l < depth; ++l) {
    glorot(in, hidden, q);
    glorot(in, hidden, q + in * hidden);
    std::fill(q + 2 * in * hidden, q + 2 * in * hidden + hidden, 0.0);
    q += 2 * in * hidden + hidden;
    in = hidden;
  }
  glorot(in, classes, q);
  std::fill(q + in * classes, q + in * classes + classes, 0.0);
}

// Transposed mean aggregation (a_mean_t, src/gnn.cpp:158-166): row v sums
// x[u]/deg(u) over its neighbours in nonzero order (same plan rules).
void mean_aggregate_t(const Graph& g, const double* x, uint32_t f, double* out) {
  std::vector<double> val(g.rp[g.n]);
  for (uint32_t r = 0; r < g.n; ++r)
    for (uint64_t k = g.rp[r]; k < g.rp[r + 1]; ++k) {
      const uint32_t u = g.ci[k];
      const uint64_t d = g.rp[u + 1] - g.rp[u];
      val[k] = d > 0 ? 1.0 / static_cast<double>(d) : 0.0;
    }
  mean_aggregate(g, val.data(), x, f, out, 1);
}

// loss_and_grads (src/gnn.cpp:180-209) + Adam (src/gnn.cpp:211-255).
void train(const Graph& g, const uint8_t* feat, const uint8_t* labels, uint32_t epochs, double lr,
           uint64_t seed, double* prm, double* final_loss, double* final_acc) {
  if (lr <= 0) throw std::invalid_argument("train: learning rate must be positive");
  const uint32_t depth = 4, in_dim = 4, hidden = 32, classes = 5;
  const uint64_t np = param_count(depth, in_dim, hidden, classes);
  init_model(seed, in_dim, hidden, classes, depth, prm);
  std::vector<double> m1(np, 0.0), m2(np, 0.0), grad(np);
  const uint32_t n = g.n;
  const double b1 = 0.9, b2 = 0.999, eps = 1e-8;
  double last_loss = 0, last_acc = 0;
  for (uint32_t ep = 1; ep <= epochs; ++ep) {
    const ModelView mv = view_model(prm, depth, in_dim, hidden, classes);
    Cache c;
    run_forward(g, feat, mv, in_dim, c, 1, true);
    // softmax_loss (src/gnn.cpp:56-68)
    std::vector<double> prob(static_cast<size_t>(n) * classes);
    double loss = 0.0;
    uint64_t hit = 0;
    for (uint32_t i = 0; i < n; ++i) {
      const double* lg = &c.logits[static_cast<size_t>(i) * classes];
      double mx = lg[0];
      uint32_t arg = 0;
      for (uint32_t j = 1; j < classes; ++j)
        if (lg[j] > mx) { mx = lg[j]; arg = j; }
      hit += arg == labels[i];
      double den = 0.0;
      double e[8];
      for (uint32_t j = 0; j < classes; ++j) { e[j] = std::exp(lg[j] - mx); den += e[j]; }
      loss -= std::log(e[labels[i]] / den);
      for (uint32_t j = 0; j < classes; ++j) prob[static_cast<size_t>(i) * classes + j] = e[j] / den;
    }
    loss /= static_cast<double>(n);
    if (!std::isfinite(loss)) throw std::runtime_error("train: loss diverged (non-finite)");
    last_loss = loss;
    last_acc = static_cast<double>(hit) / n;
    // backward
    std::vector<double> dl = prob;
    for (uint32_t i = 0; i < n; ++i) dl[static_cast<size_t>(i) * classes + labels[i]] -= 1.0;
    for (double& v : dl) v /= static_cast<double>(n);
    std::fill(grad.begin(), grad.end(), 0.0);
    // offsets of each parameter block in ASG1 order
    std::vector<uint64_t> off;
    {
      uint64_t o = 0;
      uint32_t in = in_dim;
      for (uint32_t l = 0; l < depth; ++l) {
        off.push_back(o);
        o += 2ull * in * hidden + hidden;
        in = hidden;
      }
      off.push_back(o);
    }
    const std::vector<double>& hl = c.h[depth];
    double* gwo = &grad[off[depth]];
    double* gbo = gwo + hidden * classes;
    for (uint32_t i = 0; i < n; ++i)
      for (uint32_t a = 0; a < hidden; ++a)
        for (uint32_t j = 0; j < classes; ++j)
          gwo[a * classes + j] += hl[static_cast<size_t>(i) * hidden + a] * dl[static_cast<size_t>(i) * classes + j];
    for (uint32_t i = 0; i < n; ++i)
      for (uint32_t j = 0; j < classes; ++j) gbo[j] += dl[static_cast<size_t>(i) * classes + j];
    std::vector<double> dh(static_cast<size_t>(n) * hidden, 0.0);
    for (uint32_t i = 0; i < n; ++i)
      for (uint32_t a = 0; a < hidden; ++a) {
        double s = 0.0;
        for (uint32_t j = 0; j < classes; ++j) s += dl[static_cast<size_t>(i) * classes + j] * mv.wout[a * classes + j];
        dh[static_cast<size_t>(i) * hidden + a] = s;
      }
    for (uint32_t l = depth; l-- > 0;) {
      const Layer& L = mv.layers[l];
      std::vector<double> dz(static_cast<size_t>(n) * L.out);
      for (size_t t = 0; t < dz.size(); ++t) dz[t] = c.z[l][t] > 0.0 ? dh[t] : 0.0;
      double* gws = &grad[off[l]];
      double* gwn = gws + L.in * L.out;
      double* gb = gwn + L.in * L.out;
      for (uint32_t i = 0; i < n; ++i)
        for (uint32_t a = 0; a < L.in; ++a) {
          const double hv = c.h[l][static_cast<size_t>(i) * L.in + a];
          const double mvv = c.m[l][static_cast<size_t>(i) * L.in + a];
          for (uint32_t j = 0; j < L.out; ++j) {
            gws[a * L.out + j] += hv * dz[static_cast<size_t>(i) * L.out + j];
            gwn[a * L.out + j] += mvv * dz[static_cast<size_t>(i) * L.out + j];
          }
        }
      for (uint32_t i = 0; i < n; ++i)
        for (uint32_t j = 0; j < L.out; ++j) gb[j] += dz[static_cast<size_t>(i) * L.out + j];
      if (l > 0) {
        std::vector<double> a1(static_cast<size_t>(n) * L.in), a2(static_cast<size_t>(n) * L.in);
        for (uint32_t i = 0; i < n; ++i)
          for (uint32_t a = 0; a < L.in; ++a) {
            double s1 = 0.0, s2 = 0.0;
            for (uint32_t j = 0; j < L.out; ++j) {
              s1 += dz[static_cast<size_t>(i) * L.out + j] * L.ws[a * L.out + j];
              s2 += dz[static_cast<size_t>(i) * L.out + j] * L.wn[a * L.out + j];
            }
            a1[static_cast<size_t>(i) * L.in + a] = s1;
            a2[static_cast<size_t>(i) * L.in + a] = s2;
          }
        std::vector<double> t(static_cast<size_t>(n) * L.in);
        mean_aggregate_t(g, a2.data(), L.in, t.data());
        dh.assign(a1.size(), 0.0);
        for (size_t q = 0; q < dh.size(); ++q) dh[q] = a1[q] + t[q];
      }
    }
    const double bc1 = 1.0 - std::pow(b1, ep), bc2 = 1.0 - std::pow(b2, ep);
    for (uint64_t i = 0; i < np; ++i) {
      m1[i] = b1 * m1[i] + (1.0 - b1) * grad[i];
      m2[i] = b2 * m2[i] + (1.0 - b2) * grad[i] * grad[i];
      prm[i] -= lr * (m1[i] / bc1) / (std::sqrt(m2[i] / bc2) + eps);
    }
  }
  if (final_loss) *final_loss = last_loss;
  if (final_acc) *final_acc = last_acc;
}

}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

int orc_csa_sizes(uint32_t width, uint32_t* ni, uint32_t* na, uint32_t* no) {
  return guarded([&] {
    if (width < 2) throw std::invalid_argument("gen_csa_multiplier: width must be >= 2");
    // Closed form of the generator's node count: w^2 partial products, and per
    // reduction step 3 ANDs (half adder) or 7 ANDs (full adder).
    const CsaResult r = gen_csa(width);
    *ni = r.inputs;
    *na = static_cast<uint32_t>(r.ands.size() / 2);
    *no = static_cast<uint32_t>(r.outs.size());
  });
}

int orc_gen_csa(uint32_t width, uint32_t* and_lits, uint32_t* out_lits, uint8_t* labels) {
  return guarded([&] {
    const CsaResult r = gen_csa(width);
    std::copy(r.ands.begin(), r.ands.end(), and_lits);
    std::copy(r.outs.begin(), r.outs.end(), out_lits);
    std::copy(r.labels.begin(), r.labels.end(), labels);
  });
}

int orc_encode(uint32_t ni, uint32_t na, const uint32_t* al, uint32_t no, const uint32_t* ol,
               uint8_t* feat, uint32_t* edges, uint64_t* rp, uint32_t* ci, uint32_t* deg) {
  return guarded([&] {
    const uint32_t nodes = 1 + ni + na, n = nodes + no;
    std::fill(feat, feat + 4ull * n, 0);
    uint64_t e = 0;
    for (uint32_t a = 0; a < na; ++a) {  // src/encode.cpp:45-53
      const uint32_t v = 1 + ni + a, l = al[2 * a], r = al[2 * a + 1];
      if ((l >> 1) >= v || (r >> 1) >= v) throw std::invalid_argument("encode: fanin >= node");
      feat[4ull * v] = 1;
      feat[4ull * v + 1] = 1;
      feat[4ull * v + 2] = l & 1;
      feat[4ull * v + 3] = r & 1;
      edges[e++] = l >> 1; edges[e++] = v;
      edges[e++] = r >> 1; edges[e++] = v;
    }
    for (uint32_t k = 0; k < no; ++k) {  // src/encode.cpp:54-60, po_feature :10-12
      const uint32_t po = nodes + k;
      feat[4ull * po] = 0;
      feat[4ull * po + 1] = ol[k] & 1;
      feat[4ull * po + 2] = 1;
      feat[4ull * po + 3] = 1;
      edges[e++] = ol[k] >> 1; edges[e++] = po;
    }
    build_csr(n, e / 2, edges, rp, ci);
    for (uint32_t v = 0; v < n; ++v) deg[v] = static_cast<uint32_t>(rp[v + 1] - rp[v]);
  });
}

int orc_build_csr(uint32_t n, uint64_t ne, const uint32_t* edges, uint64_t* rp, uint32_t* ci) {
  return guarded([&] { build_csr(n, ne, edges, rp, ci); });
}

int orc_batch(uint32_t n, uint64_t ne, const uint64_t* rp, const uint32_t* ci, const uint8_t* feat,
              const uint8_t* lab, const uint32_t* edges, uint32_t copies, uint64_t* orp,
              uint32_t* oci, uint8_t* ofeat, uint8_t* olab, uint32_t* odeg, uint32_t* oedges) {
  return guarded([&] {
    if (copies < 1) throw std::invalid_argument("batch: copy count must be >= 1");
    const uint64_t nnz = rp[n];
    for (uint32_t k = 0; k < copies; ++k) {
      const uint32_t no = k * n;
      const uint64_t zo = k * nnz;
      for (uint32_t v = 0; v < n; ++v) {
        orp[no + v] = zo + rp[v];
        odeg[no + v] = static_cast<uint32_t>(rp[v + 1] - rp[v]);
        olab[no + v] = lab[v];
        std::memcpy(ofeat + 4ull * (no + v), feat + 4ull * v, 4);
      }
      for (uint64_t q = 0; q < nnz; ++q) oci[zo + q] = ci[q] + no;
      for (uint64_t q = 0; q < ne; ++q) {
        oedges[2 * (k * ne + q)] = edges[2 * q] + no;
        oedges[2 * (k * ne + q) + 1] = edges[2 * q + 1] + no;
      }
    }
    orp[static_cast<uint64_t>(n) * copies] = nnz * copies;
  });
}

int orc_topo_chunks(uint32_t n, uint32_t k, uint32_t* part_of) {
  return guarded([&] {
    if (k < 1) throw std::invalid_argument("partition: k must be >= 1");
    if (k > n) throw std::invalid_argument("partition: k exceeds node count");
    for (uint32_t p = 0; p < k; ++p) {
      const uint64_t b = static_cast<uint64_t>(n) * p / k, e = static_cast<uint64_t>(n) * (p + 1) / k;
      for (uint64_t v = b; v < e; ++v) part_of[v] = p;
    }
  });
}

orc_parts* orc_regrow(uint32_t n, const uint64_t* rp, const uint32_t* ci, uint64_t ne,
                      const uint32_t* edges, const uint32_t* part_of, uint32_t k, int with_b) {
  orc_parts* out = nullptr;
  const int st = guarded([&] {
    auto* h = new orc_parts;
    h->parts.resize(k);
    for (uint32_t v = 0; v < n; ++v) {
      if (part_of[v] >= k) throw std::invalid_argument("regrow: part id out of range");
      h->parts[part_of[v]].core.push_back(v);
    }
    if (with_b) {  // src/partition.cpp:410-426
      for (uint32_t v = 0; v < n; ++v)
        for (uint64_t q = rp[v]; q < rp[v + 1]; ++q)
          if (part_of[ci[q]] != part_of[v]) h->parts[part_of[v]].boundary.push_back(ci[q]);
      for (Part& p : h->parts) {
        std::sort(p.boundary.begin(), p.boundary.end());
        p.boundary.erase(std::unique(p.boundary.begin(), p.boundary.end()), p.boundary.end());
      }
    }
    // local ids: cores ascending then boundary ascending (src/partition.cpp:428-438)
    auto local = [&](const Part& p, uint32_t v) -> uint32_t {
      auto it = std::lower_bound(p.core.begin(), p.core.end(), v);
      if (it != p.core.end() && *it == v) return static_cast<uint32_t>(it - p.core.begin());
      auto jt = std::lower_bound(p.boundary.begin(), p.boundary.end(), v);
      if (jt == p.boundary.end() || *jt != v) throw std::out_of_range("local_index.at");
      return static_cast<uint32_t>(p.core.size() + (jt - p.boundary.begin()));
    };
    for (uint64_t q = 0; q < ne; ++q) {  // src/partition.cpp:442-454
      const uint32_t u = edges[2 * q], v = edges[2 * q + 1];
      const uint32_t pu = part_of[u], pv = part_of[v];
      if (pu == pv) {
        Part& p = h->parts[pu];
        p.edges.push_back(local(p, u));
        p.edges.push_back(local(p, v));
      } else if (with_b) {
        for (uint32_t pp : {pu, pv}) {
          Part& p = h->parts[pp];
          p.edges.push_back(local(p, u));
          p.edges.push_back(local(p, v));
        }
      }
    }
    out = h;
  });
  return st == 0 ? out : nullptr;
}

uint32_t orc_parts_count(const orc_parts* h) { return static_cast<uint32_t>(h->parts.size()); }

void orc_parts_sizes(const orc_parts* h, uint32_t p, uint32_t* nc, uint32_t* nb, uint64_t* ne) {
  const Part& q = h->parts[p];
  *nc = static_cast<uint32_t>(q.core.size());
  *nb = static_cast<uint32_t>(q.boundary.size());
  *ne = q.edges.size() / 2;
}

void orc_parts_copy(const orc_parts* h, uint32_t p, uint32_t* core, uint32_t* bnd, uint32_t* edges) {
  const Part& q = h->parts[p];
  if (core) std::copy(q.core.begin(), q.core.end(), core);
  if (bnd) std::copy(q.boundary.begin(), q.boundary.end(), bnd);
  if (edges) std::copy(q.edges.begin(), q.edges.end(), edges);
}

void orc_parts_free(orc_parts* h) { delete h; }

uint64_t orc_edge_cut(uint64_t ne, const uint32_t* edges, const uint32_t* part_of) {
  uint64_t c = 0;
  for (uint64_t q = 0; q < ne; ++q) c += part_of[edges[2 * q]] != part_of[edges[2 * q + 1]];
  return c;
}

double orc_crossing_fraction(uint64_t ne, const uint32_t* edges, const uint32_t* part_of) {
  if (ne == 0) return 0.0;
  return static_cast<double>(orc_edge_cut(ne, edges, part_of)) / static_cast<double>(ne);
}

int orc_degree_sort(uint32_t rows, const uint64_t* rp, uint32_t* perm, uint64_t* srp) {
  return guarded([&] { degree_sort(rows, rp, perm, srp); });
}

orc_plan* orc_build_plan(uint32_t rows, const uint64_t* rp, uint32_t hd, uint32_t ld, uint32_t budget) {
  orc_plan* out = nullptr;
  const int st = guarded([&] { out = make_plan(rows, rp, hd, ld, budget); });
  return st == 0 ? out : nullptr;
}

void orc_plan_counts(const orc_plan* p, uint64_t c[6]) {
  c[0] = p->hd_rows.size();
  c[1] = p->mid_rows.size();
  c[2] = p->ld_groups.size() / 3;
  c[3] = p->units.size();
  c[4] = p->ld_begin;
  c[5] = p->ld_end;
}

void orc_plan_copy(const orc_plan* p, uint32_t* hd, uint32_t* mid, uint32_t* ldg, uint64_t* units,
                   uint32_t* perm) {
  if (hd) std::copy(p->hd_rows.begin(), p->hd_rows.end(), hd);
  if (mid) std::copy(p->mid_rows.begin(), p->mid_rows.end(), mid);
  if (ldg) std::copy(p->ld_groups.begin(), p->ld_groups.end(), ldg);
  if (units)
    for (size_t i = 0; i < p->units.size(); ++i) {
      const Unit& u = p->units[i];
      const uint64_t row[6] = {u.kind, u.sorted_row, u.row_count, u.nz_begin, u.nz_end, u.partial_slot};
      std::copy(row, row + 6, units + 6 * i);
    }
  if (perm) std::copy(p->perm.begin(), p->perm.end(), perm);
}

int orc_plan_execute(const orc_plan* p, uint32_t rows, const uint64_t* rp, const uint32_t* ci,
                     const double* val, const double* dense, uint32_t f, double* out) {
  return guarded([&] {
    if (rows != p->rows || (rows ? rp[rows] : 0) != p->nnz)
      throw std::invalid_argument("spmm::execute: plan does not match matrix");
    plan_execute(*p, rp, ci, val, dense, f, out);
  });
}

void orc_plan_free(orc_plan* p) { delete p; }

int orc_reference_spmm(uint32_t rows, const uint64_t* rp, const uint32_t* ci, const double* val,
                       const double* dense, uint32_t f, double* out) {
  return guarded([&] {
    for (uint32_t r = 0; r < rows; ++r) accum(out + static_cast<size_t>(r) * f, rp[r], rp[r + 1], ci, val, dense, f);
  });
}

uint64_t orc_param_count(uint32_t depth, uint32_t in_dim, uint32_t hidden, uint32_t classes) {
  return param_count(depth, in_dim, hidden, classes);
}

int orc_init_model(uint64_t seed, uint32_t in_dim, uint32_t hidden, uint32_t classes,
                   uint32_t depth, double* prm) {
  return guarded([&] { init_model(seed, in_dim, hidden, classes, depth, prm); });
}

int orc_forward(uint32_t n, const uint64_t* rp, const uint32_t* ci, const uint8_t* feat,
                uint32_t depth, uint32_t in_dim, uint32_t hidden, uint32_t classes,
                const double* prm, double* logits, unsigned threads) {
  return guarded([&] {
    if (depth < 1) throw std::invalid_argument("forward: depth must be >= 1");
    if (threads == 0) threads = std::max(1u, std::thread::hardware_concurrency());
    const Graph g{n, rp, ci};
    const ModelView mv = view_model(prm, depth, in_dim, hidden, classes);
    Cache c;
    run_forward(g, feat, mv, in_dim, c, threads, false);
    std::copy(c.logits.begin(), c.logits.end(), logits);
  });
}

int orc_classify(uint32_t n, uint32_t classes, const double* lg, const uint8_t* truth,
                 uint8_t* pred, uint64_t* conf, double* acc) {
  return guarded([&] {
    if (conf) std::fill(conf, conf + 25, 0);
    uint64_t hit = 0;
    for (uint32_t i = 0; i < n; ++i) {
      const double* row = lg + static_cast<size_t>(i) * classes;
      uint32_t arg = 0;
      for (uint32_t j = 1; j < classes; ++j)
        if (row[j] > row[arg]) arg = j;  // first maximum wins (Eigen maxCoeff)
      pred[i] = static_cast<uint8_t>(arg);
      if (truth) {
        if (conf) ++conf[truth[i] * 5 + arg];
        hit += truth[i] == arg;
      }
    }
    if (acc) *acc = n == 0 ? 0.0 : static_cast<double>(hit) / n;
  });
}

int orc_train(uint32_t n, const uint64_t* rp, const uint32_t* ci, const uint8_t* feat,
              const uint8_t* lab, uint32_t epochs, double lr, uint64_t seed, double* prm,
              double* fl, double* fa) {
  return guarded([&] { train(Graph{n, rp, ci}, feat, lab, epochs, lr, seed, prm, fl, fa); });
}

}  // extern "C"
