// ref_shim.cpp — extern "C" access to the REAL reference code (TEST INFRASTRUCTURE).
//
// Linked with the reference's own translation units compiled from
// /root/reference/proj/core/src/{aig,circuitgen,encode,partition,spmm,
// worker_pool,matrix_io}.cpp by oracle/Makefile into oracle/_ref/libaigsage_ref.so.
// Nothing here is product code. It serves three purposes:
//   1. pin the restatement in oracle.cpp (tests/test_oracle_vs_ref.py),
//   2. generate golden fixtures (tests/golden/make_golden.py),
//   3. time the reference CPU path (bench.py --impl reference / cpu_baseline).
// src/gnn.cpp needs Eigen (absent), so the forward below restates
// run_forward (src/gnn.cpp:37-52) around the reference's compiled
// spmm::build_plan / spmm::execute / default_pool — the only part that is
// not the reference's own object code is the dense h*W product.
#include <algorithm>
#include <cstring>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "aigsage/aig.hpp"
#include "aigsage/circuitgen.hpp"
#include "aigsage/encode.hpp"
#include "aigsage/partition.hpp"
#include "aigsage/spmm.hpp"
#include "aigsage/worker_pool.hpp"

using namespace aigsage;

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
}  // namespace

struct ref_graph {
  EdaGraph g;
};
struct ref_parts {
  std::vector<AugmentedPartition> parts;
};
struct ref_aig {
  Aig aig;
  GroundTruth gt;
};

// Restated dense step of run_forward (src/gnn.cpp:46-49: z = h*W_self + m*W_neigh,
// + bias, ReLU) for rows [r0, r1). Per output j the two products are summed
// over k ascending and combined as (s1 + s2) + b -- the same operation order
// as a naive triple loop, but with j innermost so the compiler vectorises it
// (no FMA contraction: -ffp-contract=off in oracle/Makefile).
static void dense_rows(const double* h, const double* m, uint32_t in, const double* ws, const double* wn,
                       const double* b, uint32_t hidden, size_t r0, size_t r1, double* hn) {
  std::vector<double> s1(hidden), s2(hidden);
  for (size_t r = r0; r < r1; ++r) {
    std::fill(s1.begin(), s1.end(), 0.0);
    std::fill(s2.begin(), s2.end(), 0.0);
    const double* hr = h + r * in;
    const double* mr = m + r * in;
    for (uint32_t k = 0; k < in; ++k) {
      const double hk = hr[k], mk = mr[k];
      const double* wsk = ws + static_cast<size_t>(k) * hidden;
      const double* wnk = wn + static_cast<size_t>(k) * hidden;
      for (uint32_t j = 0; j < hidden; ++j) {
        s1[j] += hk * wsk[j];
        s2[j] += mk * wnk[j];
      }
    }
    double* o = hn + r * hidden;
    for (uint32_t j = 0; j < hidden; ++j) {
      const double z = (s1[j] + s2[j]) + b[j];
      o[j] = z > 0.0 ? z : 0.0;
    }
  }
}

// the dense step over all n rows, split into row blocks on `pool` (null: inline)
static void dense_layer(const double* h, const double* m, uint32_t in, const double* ws, const double* wn,
                        const double* b, uint32_t hidden, size_t n, double* hn, WorkerPool* pool) {
  constexpr size_t kBlock = 4096;
  const size_t blocks = (n + kBlock - 1) / kBlock;
  auto run = [&](std::size_t i) {
    const size_t r0 = i * kBlock, r1 = std::min(n, r0 + kBlock);
    dense_rows(h, m, in, ws, wn, b, hidden, r0, r1, hn);
  };
  if (pool && blocks > 1) pool->for_each(blocks, run);
  else for (size_t i = 0; i < blocks; ++i) run(i);
}

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }
unsigned ref_default_workers(void) { return WorkerPool::default_workers(); }

// gen_csa_multiplier (src/circuitgen.cpp:66)
ref_aig* ref_gen_csa(uint32_t width) {
  ref_aig* out = nullptr;
  guarded([&] {
    CsaCircuit c = gen_csa_multiplier(width);
    out = new ref_aig{std::move(c.aig), std::move(c.gt)};
  });
  return out;
}
// parse_aiger (src/aig.cpp:47); labels are all AND except PIs/POs (no GroundTruth in a file)
ref_aig* ref_parse_aiger(const char* text) {
  ref_aig* out = nullptr;
  guarded([&] {
    std::istringstream in(text);
    Aig a = parse_aiger(in);
    GroundTruth gt;
    gt.labels.assign(a.num_nodes() + a.outputs().size(), 3);
    for (uint32_t i = 1; i <= a.num_inputs(); ++i) gt.labels[i] = 4;
    for (size_t k = 0; k < a.outputs().size(); ++k) gt.labels[a.num_nodes() + k] = 0;
    out = new ref_aig{std::move(a), std::move(gt)};
  });
  return out;
}
// Aig from literal arrays through the reference's own Aig::add_and / add_output
// (src/aig.cpp:10-22) — no text parsing; labels as in ref_parse_aiger.
ref_aig* ref_aig_from_lits(uint32_t ni, uint32_t na, const uint32_t* ands, uint32_t no, const uint32_t* outs) {
  ref_aig* out = nullptr;
  guarded([&] {
    Aig a(ni);
    for (uint32_t k = 0; k < na; ++k)
      a.add_and(Literal{ands[2 * k] >> 1, (ands[2 * k] & 1) != 0}, Literal{ands[2 * k + 1] >> 1, (ands[2 * k + 1] & 1) != 0});
    for (uint32_t k = 0; k < no; ++k) a.add_output(Literal{outs[k] >> 1, (outs[k] & 1) != 0});
    GroundTruth gt;
    gt.labels.assign(a.num_nodes() + a.outputs().size(), 3);
    for (uint32_t i = 1; i <= a.num_inputs(); ++i) gt.labels[i] = 4;
    for (size_t k = 0; k < a.outputs().size(); ++k) gt.labels[a.num_nodes() + k] = 0;
    out = new ref_aig{std::move(a), std::move(gt)};
  });
  return out;
}
void ref_aig_sizes(const ref_aig* a, uint32_t* ni, uint32_t* na, uint32_t* no) {
  *ni = a->aig.num_inputs();
  *na = a->aig.num_ands();
  *no = static_cast<uint32_t>(a->aig.outputs().size());
}
void ref_aig_copy(const ref_aig* a, uint32_t* and_lits, uint32_t* out_lits, uint8_t* labels) {
  const auto& ands = a->aig.and_nodes();
  for (size_t i = 0; i < ands.size(); ++i) {
    and_lits[2 * i] = 2 * ands[i].left.node + (ands[i].left.inverted ? 1 : 0);
    and_lits[2 * i + 1] = 2 * ands[i].right.node + (ands[i].right.inverted ? 1 : 0);
  }
  for (size_t k = 0; k < a->aig.outputs().size(); ++k)
    out_lits[k] = 2 * a->aig.outputs()[k].node + (a->aig.outputs()[k].inverted ? 1 : 0);
  if (labels) std::copy(a->gt.labels.begin(), a->gt.labels.end(), labels);
}
void ref_aig_free(ref_aig* a) { delete a; }

// encode (src/encode.cpp:33)
ref_graph* ref_encode(const ref_aig* a) {
  ref_graph* out = nullptr;
  guarded([&] { out = new ref_graph{encode(a->aig, a->gt)}; });
  return out;
}
// batch (src/encode.cpp:70)
ref_graph* ref_batch(const ref_graph* g, uint32_t copies) {
  ref_graph* out = nullptr;
  guarded([&] { out = new ref_graph{batch(g->g, copies)}; });
  return out;
}
void ref_graph_sizes(const ref_graph* g, uint32_t* n, uint64_t* nnz, uint64_t* ne) {
  *n = g->g.n;
  *nnz = g->g.col_idx.size();
  *ne = g->g.fwd_edges.size();
}
void ref_graph_copy(const ref_graph* g, uint64_t* rp, uint32_t* ci, uint8_t* feat, uint8_t* lab,
                    uint32_t* deg, uint32_t* edges) {
  const EdaGraph& e = g->g;
  if (rp) std::copy(e.row_ptr.begin(), e.row_ptr.end(), rp);
  if (ci) std::copy(e.col_idx.begin(), e.col_idx.end(), ci);
  if (feat) std::copy(e.features.begin(), e.features.end(), feat);
  if (lab) std::copy(e.labels.begin(), e.labels.end(), lab);
  if (deg) std::copy(e.degree.begin(), e.degree.end(), deg);
  if (edges)
    for (size_t i = 0; i < e.fwd_edges.size(); ++i) {
      edges[2 * i] = e.fwd_edges[i].first;
      edges[2 * i + 1] = e.fwd_edges[i].second;
    }
}
void ref_graph_free(ref_graph* g) { delete g; }

// partition_topo_chunks (src/partition.cpp:301)
int ref_topo_chunks(const ref_graph* g, uint32_t k, uint32_t* part_of) {
  return guarded([&] {
    const PartitionAssignment pa = partition_topo_chunks(g->g, k);
    std::copy(pa.part_of.begin(), pa.part_of.end(), part_of);
  });
}
// partition_multilevel (src/partition.cpp:314-367). Livelocks in rebalance for
// k >= 8 on multiplier graphs: callers run it under a time limit.
int ref_partition_multilevel(const ref_graph* g, uint32_t k, uint64_t seed, uint32_t* part_of) {
  return guarded([&] {
    const PartitionAssignment pa = partition_multilevel(g->g, k, seed);
    std::copy(pa.part_of.begin(), pa.part_of.end(), part_of);
  });
}
// load_assignment (src/partition.cpp:369)
int ref_load_assignment(const char* path, uint32_t n, uint32_t* part_of, uint32_t* k) {
  return guarded([&] {
    const PartitionAssignment pa = load_assignment(path, n);
    std::copy(pa.part_of.begin(), pa.part_of.end(), part_of);
    *k = pa.k;
  });
}
// regrow / core_subgraphs (src/partition.cpp:460-466)
ref_parts* ref_regrow(const ref_graph* g, const uint32_t* part_of, uint32_t k, int with_b) {
  ref_parts* out = nullptr;
  guarded([&] {
    PartitionAssignment pa;
    pa.part_of.assign(part_of, part_of + g->g.n);
    pa.k = k;
    out = new ref_parts{with_b ? regrow(g->g, pa) : core_subgraphs(g->g, pa)};
  });
  return out;
}
void ref_parts_sizes(const ref_parts* h, uint32_t p, uint32_t* nc, uint32_t* nb, uint64_t* ne) {
  const AugmentedPartition& a = h->parts[p];
  *nc = a.num_core();
  *nb = static_cast<uint32_t>(a.boundary_nodes.size());
  *ne = a.edges.size();
}
void ref_parts_copy(const ref_parts* h, uint32_t p, uint32_t* core, uint32_t* bnd, uint32_t* edges) {
  const AugmentedPartition& a = h->parts[p];
  if (core) std::copy(a.core_nodes.begin(), a.core_nodes.end(), core);
  if (bnd) std::copy(a.boundary_nodes.begin(), a.boundary_nodes.end(), bnd);
  if (edges)
    for (size_t i = 0; i < a.edges.size(); ++i) {
      edges[2 * i] = a.edges[i].first;
      edges[2 * i + 1] = a.edges[i].second;
    }
}
uint64_t ref_footprint_proxy(const ref_parts* h) { return footprint_proxy(h->parts); }
// materialize (src/partition.cpp:488)
ref_graph* ref_materialize(const ref_graph* g, const ref_parts* h, uint32_t p) {
  ref_graph* out = nullptr;
  guarded([&] { out = new ref_graph{materialize(g->g, h->parts[p])}; });
  return out;
}
void ref_parts_free(ref_parts* h) { delete h; }
double ref_crossing_fraction(const ref_graph* g, const uint32_t* part_of, uint32_t k) {
  PartitionAssignment pa;
  pa.part_of.assign(part_of, part_of + g->g.n);
  pa.k = k;
  return crossing_fraction(g->g, pa);
}

// spmm::build_plan (src/spmm.cpp:37) — counts + arrays in the oracle's layout.
struct ref_plan {
  spmm::SpmmPlan plan;
};
ref_plan* ref_build_plan(uint32_t rows, const uint64_t* rp, uint32_t hd, uint32_t ld, uint32_t budget) {
  ref_plan* out = nullptr;
  guarded([&] {
    out = new ref_plan{spmm::build_plan(rows, std::span<const uint64_t>(rp, rows + 1ull), 1, hd, ld, budget)};
  });
  return out;
}
void ref_plan_counts(const ref_plan* p, uint64_t c[6]) {
  c[0] = p->plan.hd_rows.size();
  c[1] = p->plan.mid_rows.size();
  c[2] = p->plan.ld_groups.size();
  c[3] = p->plan.work_units.size();
  c[4] = p->plan.ld_row_begin;
  c[5] = p->plan.ld_row_end;
}
void ref_plan_copy(const ref_plan* p, uint32_t* hd, uint32_t* mid, uint32_t* ldg, uint64_t* units,
                   uint32_t* perm) {
  const spmm::SpmmPlan& q = p->plan;
  if (hd) std::copy(q.hd_rows.begin(), q.hd_rows.end(), hd);
  if (mid) std::copy(q.mid_rows.begin(), q.mid_rows.end(), mid);
  if (ldg)
    for (size_t i = 0; i < q.ld_groups.size(); ++i) {
      ldg[3 * i] = q.ld_groups[i].degree;
      ldg[3 * i + 1] = q.ld_groups[i].row_begin;
      ldg[3 * i + 2] = q.ld_groups[i].row_end;
    }
  if (units)
    for (size_t i = 0; i < q.work_units.size(); ++i) {
      const spmm::WorkUnit& u = q.work_units[i];
      const uint64_t kind = u.kind == spmm::WorkKind::HdChunk ? 0 : (u.kind == spmm::WorkKind::LdBatch ? 1 : 2);
      const uint64_t row[6] = {kind, u.sorted_row, u.row_count, u.nz_begin, u.nz_end, u.partial_slot};
      std::copy(row, row + 6, units + 6 * i);
    }
  if (perm) std::copy(q.perm.begin(), q.perm.end(), perm);
}
// spmm::execute (inc/spmm.hpp:106), fp64; threads: 0 => inline, else a pool of that size
int ref_plan_execute(const ref_plan* p, uint32_t rows, const uint64_t* rp, const uint32_t* ci,
                     const double* val, const double* dense, uint32_t f, double* out, unsigned threads) {
  return guarded([&] {
    spmm::CsrMatrix<double> m;
    m.rows = m.cols = rows;
    m.row_ptr.assign(rp, rp + rows + 1ull);
    m.col_idx.assign(ci, ci + rp[rows]);
    m.values.assign(val, val + rp[rows]);
    if (threads == 0) {
      spmm::execute(p->plan, m, dense, f, out, nullptr);
    } else {
      WorkerPool pool(threads);
      spmm::execute(p->plan, m, dense, f, out, &pool);
    }
  });
}
void ref_plan_free(ref_plan* p) { delete p; }

// predict_full (src/gnn.cpp:293-300) over the reference's compiled make_context
// pieces: CsrMatrix a_mean with values 1/deg (src/gnn.cpp:147-157), plan from
// spmm::build_plan, aggregation by spmm::execute on default_pool() when
// nnz*f >= 65536 (src/gnn.cpp:16-28). Dense product restated (Eigen absent).
// params in ASG1 order. logits may be NULL. Returns the number of threads used.
int ref_predict_full(const ref_graph* g, uint32_t depth, uint32_t in_dim, uint32_t hidden,
                     uint32_t classes, const double* prm, double* logits, uint8_t* pred,
                     uint64_t* confusion, double* accuracy) {
  return guarded([&] {
    const EdaGraph& e = g->g;
    const uint32_t n = e.n;
    spmm::CsrMatrix<double> a;
    a.rows = a.cols = n;
    a.row_ptr = e.row_ptr;
    a.col_idx = e.col_idx;
    a.values.resize(e.col_idx.size());
    for (uint32_t v = 0; v < n; ++v) {
      const double inv = e.degree[v] > 0 ? 1.0 / e.degree[v] : 0.0;
      for (uint64_t q = e.row_ptr[v]; q < e.row_ptr[v + 1]; ++q) a.values[q] = inv;
    }
    const spmm::SpmmPlan plan = spmm::build_plan(a, 0);
    std::vector<double> h(static_cast<size_t>(n) * in_dim);
    for (size_t i = 0; i < h.size(); ++i) h[i] = e.features[i];
    uint32_t in = in_dim;
    const double* q = prm;
    for (uint32_t l = 0; l < depth; ++l) {
      const double* ws = q;
      const double* wn = q + in * hidden;
      const double* b = q + 2 * in * hidden;
      q += 2 * in * hidden + hidden;
      std::vector<double> m(static_cast<size_t>(n) * in);
      WorkerPool* pool = a.nnz() * in >= (1u << 16) ? &default_pool() : nullptr;
      spmm::execute(plan, a, h.data(), in, m.data(), pool);
      std::vector<double> hn(static_cast<size_t>(n) * hidden);
      dense_layer(h.data(), m.data(), in, ws, wn, b, hidden, n, hn.data(), &default_pool());
      h.swap(hn);
      in = hidden;
    }
    const double* wo = q;
    const double* bo = q + in * classes;
    if (confusion) std::fill(confusion, confusion + 25, 0);
    uint64_t hit = 0;
    std::vector<double> row(classes);
    for (uint32_t r = 0; r < n; ++r) {
      for (uint32_t j = 0; j < classes; ++j) {
        double s = 0.0;
        for (uint32_t k = 0; k < in; ++k) s += h[static_cast<size_t>(r) * in + k] * wo[k * classes + j];
        row[j] = s + bo[j];
      }
      uint32_t arg = 0;
      for (uint32_t j = 1; j < classes; ++j)
        if (row[j] > row[arg]) arg = j;
      if (logits) std::copy(row.begin(), row.end(), logits + static_cast<size_t>(r) * classes);
      if (pred) pred[r] = static_cast<uint8_t>(arg);
      if (confusion) ++confusion[e.labels[r] * 5 + arg];
      hit += e.labels[r] == arg;
    }
    if (accuracy) *accuracy = n ? static_cast<double>(hit) / n : 0.0;
  });
}

// predict (src/gnn.cpp:280-291) over parts [first, first+count): default_pool()
// runs one part per item (the nested SpMM then runs inline, src/worker_pool.cpp:55-60),
// each part = forward(materialize(g, part)) with the restated dense product,
// scored on core rows. pred (global, n entries) receives the core labels and
// logits (global, n x classes, may be NULL) the core rows' logits.
int ref_predict_parts(const ref_graph* g, const ref_parts* h, uint32_t first, uint32_t count,
                      uint32_t depth, uint32_t in_dim, uint32_t hidden, uint32_t classes,
                      const double* prm, uint8_t* pred, double* logits) {
  return guarded([&] {
    if (first + count > h->parts.size()) throw std::invalid_argument("ref_predict_parts: range");
    default_pool().for_each(count, [&](std::size_t i) {
      const AugmentedPartition& part = h->parts[first + i];
      const EdaGraph e = materialize(g->g, part);
      const uint32_t n = e.n;
      spmm::CsrMatrix<double> a;
      a.rows = a.cols = n;
      a.row_ptr = e.row_ptr;
      a.col_idx = e.col_idx;
      a.values.resize(e.col_idx.size());
      for (uint32_t v = 0; v < n; ++v) {
        const double inv = e.degree[v] > 0 ? 1.0 / e.degree[v] : 0.0;
        for (uint64_t q = e.row_ptr[v]; q < e.row_ptr[v + 1]; ++q) a.values[q] = inv;
      }
      const spmm::SpmmPlan plan = spmm::build_plan(a, 0);
      std::vector<double> x(static_cast<size_t>(n) * in_dim);
      for (size_t k = 0; k < x.size(); ++k) x[k] = e.features[k];
      uint32_t in = in_dim;
      const double* q = prm;
      for (uint32_t l = 0; l < depth; ++l) {
        const double* ws = q;
        const double* wn = q + in * hidden;
        const double* b = q + 2 * in * hidden;
        q += 2 * in * hidden + hidden;
        std::vector<double> m(static_cast<size_t>(n) * in);
        spmm::execute(plan, a, x.data(), in, m.data(), &default_pool());  // nested: runs inline
        std::vector<double> hn(static_cast<size_t>(n) * hidden);
        dense_layer(x.data(), m.data(), in, ws, wn, b, hidden, n, hn.data(), nullptr);  // part-parallel already
        x.swap(hn);
        in = hidden;
      }
      const double* wo = q;
      const double* bo = q + in * classes;
      for (uint32_t r = 0; r < part.num_core(); ++r) {
        uint32_t arg = 0;
        double best = 0.0;
        for (uint32_t c = 0; c < classes; ++c) {
          double s = 0.0;
          for (uint32_t k = 0; k < in; ++k) s += x[static_cast<size_t>(r) * in + k] * wo[k * classes + c];
          s += bo[c];
          if (logits) logits[static_cast<size_t>(part.core_nodes[r]) * classes + c] = s;
          if (c == 0 || s > best) { best = s; arg = c; }
        }
        if (pred) pred[part.core_nodes[r]] = static_cast<uint8_t>(arg);
      }
    });
  });
}

}  // extern "C"
