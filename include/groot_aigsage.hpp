// groot_aigsage.hpp — drop-in C++ mirror of the reference's aigsage operator API
// for the GNN verification hot path, implemented over the C ABI (groot.h) of
// libgroot_b200.so. Same names, argument meaning and exception types as
// /root/reference/proj/core/include/aigsage/{aig,circuitgen,encode,partition,
// spmm,gnn}.hpp; compute runs on the B200 (no CPU fallback).
//
// Differences a caller can observe, all deliberate:
//  * RowMat is a minimal row-major dense matrix (rows(), cols(), data(),
//    operator()(i,j)) instead of Eigen::Matrix (Eigen is not a dependency).
//  * forward() returns fp32 logits widened to double (the device path computes
//    in fp32 with a 3xTF32 tensor-core transform).
//  * VerifyReport carries the residual polynomial as text plus its term count
//    (the reference's Polynomial is a Boost.Multiprecision type).
//  * aigsage::gpu::DeviceGraph keeps a graph resident in HBM across calls;
//    the value-returning functions copy to the host like the reference does.
//
// Link: -I include -L paper_2511_18297_b200 -lgroot_b200
#pragma once

#include <algorithm>
#include <array>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstdlib>
#include <fstream>
#include <functional>
#include <iterator>
#include <map>
#include <memory>
#include <random>
#include <span>
#include <sstream>
#include <stdexcept>
#include <string>
#include <thread>
#include <type_traits>
#include <unordered_map>
#include <utility>
#include <vector>

#include "groot.h"

namespace aigsage {

namespace detail {
inline void check(int st) {
  if (st == GROOT_OK) return;
  const std::string msg = groot_last_error();
  if (st == GROOT_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}
}  // namespace detail

// ---- inc/aig.hpp --------------------------------------------------------------
struct Literal {
  std::uint32_t node = 0;
  bool inverted = false;
  friend bool operator==(const Literal&, const Literal&) = default;
};
inline Literal lit(std::uint32_t node, bool inverted = false) { return {node, inverted}; }
inline Literal operator~(Literal l) { return {l.node, !l.inverted}; }
inline std::uint32_t encode_lit(Literal l) { return 2 * l.node + (l.inverted ? 1u : 0u); }
inline Literal decode_lit(std::uint32_t v) { return {v >> 1, (v & 1u) != 0}; }

struct AndNode {
  Literal left, right;
  friend bool operator==(const AndNode&, const AndNode&) = default;
};

class Aig {
 public:
  Aig() = default;
  explicit Aig(std::uint32_t num_inputs) : num_inputs_(num_inputs) {}
  std::uint32_t num_inputs() const { return num_inputs_; }
  std::uint32_t num_ands() const { return static_cast<std::uint32_t>(ands_.size()); }
  std::uint32_t num_nodes() const { return 1 + num_inputs_ + num_ands(); }
  std::uint32_t first_and() const { return 1 + num_inputs_; }
  bool is_constant(std::uint32_t v) const { return v == 0; }
  bool is_input(std::uint32_t v) const { return v >= 1 && v <= num_inputs_; }
  bool is_and(std::uint32_t v) const { return v >= first_and() && v < num_nodes(); }
  const AndNode& and_node(std::uint32_t v) const { return ands_[v - first_and()]; }
  const std::vector<AndNode>& and_nodes() const { return ands_; }
  const std::vector<Literal>& outputs() const { return outputs_; }
  std::uint32_t add_and(Literal left, Literal right) {  // src/aig.cpp:10-16
    const std::uint32_t index = num_nodes();
    if (left.node >= index || right.node >= index)
      throw std::invalid_argument("Aig::add_and: fanin index must be strictly below the new node");
    ands_.push_back({left, right});
    return index;
  }
  void add_output(Literal driver) {
    if (driver.node >= num_nodes()) throw std::invalid_argument("Aig::add_output: driver references unknown node");
    outputs_.push_back(driver);
  }
  // Flips the inversion flag of one fanin of an AND node (inc/aig.hpp:57, src/aig.cpp:24-29):
  // the verifier's mutated-multiplier tests.
  void flip_and_fanin(std::uint32_t node, bool right_side) {
    if (!is_and(node)) throw std::invalid_argument("Aig::flip_and_fanin: not an AND node");
    AndNode& a = ands_[node - first_and()];
    Literal& l = right_side ? a.right : a.left;
    l.inverted = !l.inverted;
  }
  // Flat AIGER literal arrays for the C ABI.
  std::vector<std::uint32_t> and_lits() const {
    std::vector<std::uint32_t> v(2 * ands_.size());
    for (size_t i = 0; i < ands_.size(); ++i) {
      v[2 * i] = encode_lit(ands_[i].left);
      v[2 * i + 1] = encode_lit(ands_[i].right);
    }
    return v;
  }
  std::vector<std::uint32_t> out_lits() const {
    std::vector<std::uint32_t> v(outputs_.size());
    for (size_t i = 0; i < outputs_.size(); ++i) v[i] = encode_lit(outputs_[i]);
    return v;
  }
  static Aig from_lits(std::uint32_t ni, const std::vector<std::uint32_t>& ands, const std::vector<std::uint32_t>& outs) {
    Aig g(ni);
    g.ands_.reserve(ands.size() / 2);
    for (size_t i = 0; i + 1 < ands.size(); i += 2) g.ands_.push_back({decode_lit(ands[i]), decode_lit(ands[i + 1])});
    for (std::uint32_t o : outs) g.outputs_.push_back(decode_lit(o));
    return g;
  }
  friend bool operator==(const Aig&, const Aig&) = default;

 private:
  std::uint32_t num_inputs_ = 0;
  std::vector<AndNode> ands_;
  std::vector<Literal> outputs_;
};

// parse_aiger (src/aig.cpp:47-88): same checks and messages (std::runtime_error).
inline Aig parse_aiger(std::istream& in) {
  const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  std::uint32_t ni, na, no;
  detail::check(groot_aiger_sizes(text.data(), text.size(), &ni, &na, &no));
  std::vector<std::uint32_t> ands(2ull * na), outs(no);
  detail::check(groot_aiger_fill(text.data(), text.size(), ands.data(), outs.data()));
  return Aig::from_lits(ni, ands, outs);
}
inline Aig parse_aiger_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open AIGER file: " + path);
  return parse_aiger(in);
}
inline void write_aiger(const Aig& g, std::ostream& out) {  // src/aig.cpp:96-113
  const std::uint32_t i = g.num_inputs(), a = g.num_ands();
  out << "aag " << (i + a) << ' ' << i << " 0 " << g.outputs().size() << ' ' << a << '\n';
  for (std::uint32_t n = 1; n <= i; ++n) out << 2 * n << '\n';
  for (const Literal& d : g.outputs()) out << encode_lit(d) << '\n';
  for (std::uint32_t n = 0; n < a; ++n)
    out << 2 * (i + 1 + n) << ' ' << encode_lit(g.and_nodes()[n].left) << ' ' << encode_lit(g.and_nodes()[n].right) << '\n';
}

inline void write_aiger_file(const Aig& g, const std::string& path) {  // inc/aig.hpp:73, src/aig.cpp:109-113
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot write AIGER file: " + path);
  write_aiger(g, out);
}

// ---- inc/circuitgen.hpp ---------------------------------------------------------
enum class NodeClass : std::uint8_t { Po = 0, Maj = 1, Xor = 2, And = 3, Pi = 4 };
inline constexpr std::uint32_t kNumClasses = 5;

struct GroundTruth {
  std::vector<std::uint8_t> labels;
  std::vector<std::uint32_t> po_nodes;
  std::map<std::uint32_t, std::vector<Literal>> supports;  // adder roots -> support literals (CSA generator)
};

struct CsaCircuit {
  Aig aig;
  GroundTruth gt;
  std::uint32_t width = 0;
  std::uint32_t half_adders = 0;
  std::uint32_t full_adders = 0;
};

// Radix-4 Booth multiplier (BASELINE config 3; not in the reference):
// same conventions as gen_csa_multiplier; adder counts are not tracked (0).
inline CsaCircuit gen_booth_multiplier(std::uint32_t width) {
  std::uint32_t ni, na, no;
  detail::check(groot_booth_sizes(width, &ni, &na, &no));
  std::vector<std::uint32_t> ands(2ull * na), outs(no);
  CsaCircuit c;
  c.width = width;
  c.gt.labels.resize(1ull + ni + na + no);
  detail::check(groot_gen_booth(width, ands.data(), outs.data(), c.gt.labels.data()));
  c.aig = Aig::from_lits(ni, ands, outs);
  for (std::uint32_t k = 0; k < no; ++k) c.gt.po_nodes.push_back(c.aig.num_nodes() + k);
  return c;
}

// gen_csa_multiplier (src/circuitgen.cpp:66-133): bit-identical AIG and labels.
inline CsaCircuit gen_csa_multiplier(std::uint32_t width) {
  std::uint32_t ni, na, no;
  detail::check(groot_csa_sizes(width, &ni, &na, &no));
  std::vector<std::uint32_t> ands(2ull * na), outs(no);
  CsaCircuit c;
  c.width = width;
  c.gt.labels.resize(1ull + ni + na + no);
  detail::check(groot_gen_csa(width, ands.data(), outs.data(), c.gt.labels.data()));
  c.aig = Aig::from_lits(ni, ands, outs);
  for (std::uint32_t k = 0; k < no; ++k) c.gt.po_nodes.push_back(c.aig.num_nodes() + k);
  std::uint32_t nsup = 0;  // GroundTruth::supports (src/circuitgen.cpp:30-32, 50-62)
  detail::check(groot_csa_supports(width, &nsup, nullptr));
  std::vector<std::uint32_t> rec(5ull * nsup);
  detail::check(groot_csa_supports(width, &nsup, rec.data()));
  for (std::uint32_t i = 0; i < nsup; ++i) {
    std::vector<Literal>& sup = c.gt.supports[rec[5 * i]];
    for (std::uint32_t a = 0; a < rec[5 * i + 1]; ++a) sup.push_back(decode_lit(rec[5 * i + 2 + a]));
  }
  // Adder counts by replaying the column-slot occupancy of the generator
  // (src/circuitgen.cpp:90-127); reduce() makes a HA for 2 inputs, a FA for 3.
  const std::uint32_t w = width;
  std::vector<std::uint8_t> sums(2 * w, 0), carries(2 * w, 0), ns(2 * w), nc(2 * w);
  for (std::uint32_t j = 1; j < w; ++j) sums[j] = 1;
  auto add = [&](std::uint32_t cnt) {
    if (cnt == 2) ++c.half_adders;
    if (cnt == 3) ++c.full_adders;
    return cnt >= 2;
  };
  for (std::uint32_t i = 1; i < w; ++i) {
    std::fill(ns.begin(), ns.end(), 0);
    std::fill(nc.begin(), nc.end(), 0);
    for (std::uint32_t j = 0; j < w; ++j) {
      const std::uint32_t col = i + j;
      const bool carry = add(sums[col] + 1u + carries[col]);
      if (j != 0) ns[col] = 1;
      if (carry) nc[col + 1] = 1;
    }
    sums.swap(ns);
    carries.swap(nc);
  }
  bool ripple = false;
  for (std::uint32_t col = w; col < 2 * w; ++col) ripple = add(sums[col] + carries[col] + (ripple ? 1u : 0u));
  return c;
}

// load_labels / write_labels (src/circuitgen.cpp:173-198)
inline std::vector<std::uint8_t> load_labels(const std::string& path, std::size_t expected_nodes) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open label file: " + path);
  std::vector<std::uint8_t> labels(expected_nodes, 0), seen(expected_nodes, 0);
  std::uint64_t node, label;
  while (in >> node >> label) {
    if (node >= expected_nodes) throw std::runtime_error("label file: node id out of range: " + std::to_string(node));
    if (seen[node]) throw std::runtime_error("label file: duplicate node " + std::to_string(node));
    if (label >= kNumClasses) throw std::runtime_error("label file: label out of range for node " + std::to_string(node));
    labels[node] = static_cast<std::uint8_t>(label);
    seen[node] = 1;
  }
  for (std::size_t i = 0; i < expected_nodes; ++i)
    if (!seen[i]) throw std::runtime_error("label file: missing node " + std::to_string(i));
  return labels;
}
inline void write_labels(const std::string& path, const std::vector<std::uint8_t>& labels) {
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot write label file: " + path);
  for (std::size_t i = 0; i < labels.size(); ++i) out << i << ' ' << static_cast<int>(labels[i]) << '\n';
}

// write_supports / load_supports (src/circuitgen.cpp:200-227): "root arity lit..." lines
inline void write_supports(const std::string& path, const std::map<std::uint32_t, std::vector<Literal>>& supports) {
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot write support file: " + path);
  for (const auto& [root, sup] : supports) {
    out << root << ' ' << sup.size();
    for (const Literal& l : sup) out << ' ' << encode_lit(l);
    out << '\n';
  }
}
inline std::map<std::uint32_t, std::vector<Literal>> load_supports(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open support file: " + path);
  std::map<std::uint32_t, std::vector<Literal>> supports;
  std::uint32_t root;
  std::size_t arity;
  while (in >> root >> arity) {
    std::vector<Literal> sup;
    for (std::size_t i = 0; i < arity; ++i) {
      std::uint64_t enc;
      if (!(in >> enc)) throw std::runtime_error("support file: truncated entry");
      sup.push_back(decode_lit(static_cast<std::uint32_t>(enc)));
    }
    supports[root] = std::move(sup);
  }
  return supports;
}

// ---- inc/verify.hpp: the consumer of the classes ------------------------------------
struct VerifyOptions {
  std::size_t monomial_cap = 2'000'000;
};
// The residual polynomial is returned as text (first 64 terms) with its term
// count: the reference's Polynomial is a Boost.Multiprecision type.
struct VerifyReport {
  bool equivalent = false;
  bool inconclusive = false;
  std::string residual;
  std::uint64_t residual_terms = 0;
  std::uint64_t substitution_count = 0;
  std::uint64_t shortcut_count = 0;
  std::uint64_t fallback_count = 0;
};
// backward_rewrite (src/verify.cpp:220-395), host.
inline VerifyReport backward_rewrite(const Aig& g, const std::vector<std::uint8_t>& labels,
                                     const std::map<std::uint32_t, std::vector<Literal>>& supports, std::uint32_t width,
                                     const VerifyOptions& opts = {}) {
  const auto ands = g.and_lits();
  const auto outs = g.out_lits();
  std::vector<std::uint32_t> off(g.num_nodes() + 1ull, 0), nodes;
  for (std::uint32_t v = 0; v < g.num_nodes(); ++v) {
    if (auto it = supports.find(v); it != supports.end())
      for (const Literal& l : it->second) nodes.push_back(l.node);
    off[v + 1] = static_cast<std::uint32_t>(nodes.size());
  }
  VerifyReport r;
  std::int32_t eq = 0, inc = 0;
  std::uint64_t counts[3];
  detail::check(groot_backward_rewrite(g.num_inputs(), g.num_ands(), ands.data(), static_cast<std::uint32_t>(outs.size()),
                                       outs.data(), labels.data(), static_cast<std::uint32_t>(labels.size()), off.data(),
                                       nodes.data(), width, opts.monomial_cap, &eq, &inc, &r.residual_terms, counts));
  r.equivalent = eq != 0;
  r.inconclusive = inc != 0;
  r.residual = groot_backward_rewrite_residual();
  r.substitution_count = counts[0];
  r.shortcut_count = counts[1];
  r.fallback_count = counts[2];
  return r;
}
inline bool truth_table_equiv(const Aig& g, std::uint32_t width) {  // src/verify.cpp:398-416
  const auto ands = g.and_lits();
  const auto outs = g.out_lits();
  std::int32_t eq = 0;
  detail::check(groot_truth_table_equiv(g.num_inputs(), g.num_ands(), ands.data(), static_cast<std::uint32_t>(outs.size()),
                                        outs.data(), width, &eq));
  return eq != 0;
}
inline std::vector<std::uint8_t> simulate(const Aig& g, const std::vector<std::uint8_t>& assignment) {  // src/aig.cpp:130
  if (assignment.size() != g.num_inputs()) throw std::invalid_argument("simulate: assignment length != number of inputs");
  const auto ands = g.and_lits();
  const auto outs = g.out_lits();
  std::vector<std::uint8_t> out(outs.size());
  detail::check(groot_simulate(g.num_inputs(), g.num_ands(), ands.data(), static_cast<std::uint32_t>(outs.size()),
                               outs.data(), assignment.data(), out.data()));
  return out;
}

// ---- device-resident handles -------------------------------------------------------
namespace gpu {
struct GraphDeleter {
  void operator()(groot_graph* g) const { groot_graph_free(g); }
};
using DeviceGraph = std::unique_ptr<groot_graph, GraphDeleter>;
struct AssignDeleter {
  void operator()(groot_assignment* a) const { groot_assignment_free(a); }
};
using DeviceAssignment = std::unique_ptr<groot_assignment, AssignDeleter>;
struct PartsDeleter {
  void operator()(groot_parts* p) const { groot_parts_free(p); }
};
using DeviceParts = std::unique_ptr<groot_parts, PartsDeleter>;
struct ModelDeleter {
  void operator()(groot_model* m) const { groot_model_free(m); }
};
using DeviceModel = std::unique_ptr<groot_model, ModelDeleter>;
}  // namespace gpu

// ---- inc/encode.hpp -------------------------------------------------------------
struct EdaGraph {
  std::uint32_t n = 0;
  std::vector<std::uint64_t> row_ptr;
  std::vector<std::uint32_t> col_idx;
  std::vector<std::uint8_t> features;  // n x 4
  std::vector<std::uint8_t> labels;
  std::vector<std::uint32_t> degree;
  std::vector<std::pair<std::uint32_t, std::uint32_t>> fwd_edges;

  std::array<std::uint8_t, 4> feature(std::uint32_t v) const {
    return {features[4 * v], features[4 * v + 1], features[4 * v + 2], features[4 * v + 3]};
  }
  std::uint64_t num_undirected_edges() const { return fwd_edges.size(); }

  // Host copy of a resident graph.
  static EdaGraph from_device(const groot_graph* g) {
    EdaGraph e;
    std::uint64_t nnz, ne;
    detail::check(groot_graph_sizes(g, &e.n, &nnz, &ne));
    e.row_ptr.resize(e.n + 1ull);
    e.col_idx.resize(nnz);
    e.features.resize(4ull * e.n);
    e.labels.resize(e.n);
    e.degree.resize(e.n);
    std::vector<std::uint32_t> edges(2 * ne);
    detail::check(groot_graph_copy_out(g, e.row_ptr.data(), e.col_idx.data(), e.features.data(), e.labels.data(),
                                       e.degree.data(), edges.data()));
    e.fwd_edges.resize(ne);
    for (std::uint64_t i = 0; i < ne; ++i) e.fwd_edges[i] = {edges[2 * i], edges[2 * i + 1]};
    return e;
  }
  // Upload to HBM (the resident form every device entry point takes).
  gpu::DeviceGraph to_device() const {
    std::vector<std::uint32_t> edges(2 * fwd_edges.size());
    for (size_t i = 0; i < fwd_edges.size(); ++i) {
      edges[2 * i] = fwd_edges[i].first;
      edges[2 * i + 1] = fwd_edges[i].second;
    }
    groot_graph* g = nullptr;
    detail::check(groot_graph_from_host(n, row_ptr.data(), col_idx.data(), features.empty() ? nullptr : features.data(),
                                        labels.empty() ? nullptr : labels.data(), fwd_edges.size(),
                                        edges.empty() ? nullptr : edges.data(), &g));
    return gpu::DeviceGraph(g);
  }
};

inline std::array<std::uint8_t, 4> po_feature(bool driver_inverted) {  // src/encode.cpp:10-12
  return {0, static_cast<std::uint8_t>(driver_inverted ? 1 : 0), 1, 1};
}

namespace gpu {
// encode on the device, graph stays resident.
inline DeviceGraph encode(const Aig& g, const GroundTruth& gt) {
  const std::uint32_t n = g.num_nodes() + static_cast<std::uint32_t>(g.outputs().size());
  if (gt.labels.size() != n) throw std::invalid_argument("encode: label count does not match encoded node count");
  const auto ands = g.and_lits();
  const auto outs = g.out_lits();
  groot_graph* out = nullptr;
  detail::check(groot_encode(g.num_inputs(), g.num_ands(), ands.data(), static_cast<std::uint32_t>(outs.size()),
                             outs.data(), gt.labels.data(), &out));
  return DeviceGraph(out);
}
inline DeviceGraph batch(const groot_graph* g, std::uint32_t copies) {
  groot_graph* out = nullptr;
  detail::check(groot_batch(g, copies, &out));
  return DeviceGraph(out);
}
}  // namespace gpu

// encode (src/encode.cpp:33-68), batch (src/encode.cpp:70-101)
inline EdaGraph encode(const Aig& g, const GroundTruth& gt) { return EdaGraph::from_device(gpu::encode(g, gt).get()); }
inline EdaGraph batch(const EdaGraph& g, std::uint32_t copies) {
  if (copies < 1) throw std::invalid_argument("batch: copy count must be >= 1");
  if (copies == 1) return g;
  auto d = g.to_device();
  return EdaGraph::from_device(gpu::batch(d.get(), copies).get());
}

// ---- inc/partition.hpp ---------------------------------------------------------------
struct PartitionAssignment {
  std::vector<std::uint32_t> part_of;
  std::uint32_t k = 0;
  gpu::DeviceAssignment to_device() const {
    groot_assignment* a = nullptr;
    detail::check(groot_assignment_from_host(static_cast<std::uint32_t>(part_of.size()), part_of.data(), &a));
    return gpu::DeviceAssignment(a);
  }
  static PartitionAssignment from_device(const groot_assignment* a) {
    PartitionAssignment pa;
    std::uint32_t n;
    detail::check(groot_assignment_info(a, &n, &pa.k));
    pa.part_of.resize(n);
    detail::check(groot_assignment_copy_out(a, pa.part_of.data()));
    return pa;
  }
};

struct AugmentedPartition {
  std::vector<std::uint32_t> core_nodes;
  std::vector<std::uint32_t> boundary_nodes;
  std::vector<std::uint32_t> local_to_global;
  std::unordered_map<std::uint32_t, std::uint32_t> local_index;
  std::vector<std::pair<std::uint32_t, std::uint32_t>> edges;
  std::vector<std::uint8_t> core_mask;
  std::uint32_t num_core() const { return static_cast<std::uint32_t>(core_nodes.size()); }
  std::uint32_t size() const { return static_cast<std::uint32_t>(local_to_global.size()); }
};

inline std::vector<AugmentedPartition> parts_from_device(const groot_parts* p) {
  std::uint32_t k;
  detail::check(groot_parts_count(p, &k));
  std::vector<AugmentedPartition> out(k);
  for (std::uint32_t q = 0; q < k; ++q) {
    std::uint32_t nc, nb;
    std::uint64_t ne;
    detail::check(groot_parts_sizes(p, q, &nc, &nb, &ne));
    AugmentedPartition& ap = out[q];
    ap.core_nodes.resize(nc);
    ap.boundary_nodes.resize(nb);
    std::vector<std::uint32_t> e(2 * ne);
    detail::check(groot_parts_copy_out(p, q, ap.core_nodes.data(), ap.boundary_nodes.data(), e.data()));
    ap.local_to_global = ap.core_nodes;
    ap.local_to_global.insert(ap.local_to_global.end(), ap.boundary_nodes.begin(), ap.boundary_nodes.end());
    ap.local_index.reserve(ap.local_to_global.size());
    for (std::uint32_t i = 0; i < ap.local_to_global.size(); ++i) ap.local_index.emplace(ap.local_to_global[i], i);
    ap.core_mask.assign(ap.local_to_global.size(), 0);
    std::fill(ap.core_mask.begin(), ap.core_mask.begin() + nc, 1);
    ap.edges.resize(ne);
    for (std::uint64_t i = 0; i < ne; ++i) ap.edges[i] = {e[2 * i], e[2 * i + 1]};
  }
  return out;
}

// The caller's parts, uploaded as they are (groot_parts_from_host).
inline gpu::DeviceParts parts_to_device(std::uint32_t n, const std::vector<AugmentedPartition>& parts) {
  const std::uint32_t k = static_cast<std::uint32_t>(parts.size());
  std::vector<std::uint64_t> co(k + 1, 0), bo(k + 1, 0), eo(k + 1, 0);
  std::vector<std::uint32_t> core, bnd, edges;
  for (std::uint32_t p = 0; p < k; ++p) {
    const AugmentedPartition& a = parts[p];
    core.insert(core.end(), a.core_nodes.begin(), a.core_nodes.end());
    bnd.insert(bnd.end(), a.boundary_nodes.begin(), a.boundary_nodes.end());
    for (const auto& [u, v] : a.edges) {
      edges.push_back(u);
      edges.push_back(v);
    }
    co[p + 1] = core.size();
    bo[p + 1] = bnd.size();
    eo[p + 1] = edges.size() / 2;
  }
  groot_parts* out = nullptr;
  detail::check(groot_parts_from_host(n, k, co.data(), core.data(), bo.data(), bnd.data(), eo.data(), edges.data(), &out));
  return gpu::DeviceParts(out);
}

inline PartitionAssignment partition_topo_chunks(const EdaGraph& g, std::uint32_t k) {  // src/partition.cpp:301
  auto d = g.to_device();
  groot_assignment* a = nullptr;
  detail::check(groot_partition_topo_chunks(d.get(), k, &a));
  gpu::DeviceAssignment da(a);
  return PartitionAssignment::from_device(da.get());
}
// partition_multilevel (src/partition.cpp:314-367) replacement: topo chunks +
// device label propagation within the 5 % cap; terminates for every k (the
// reference livelocks for k >= 8); equal to the reference where it terminates
// and its refined-topo candidate wins.
inline PartitionAssignment partition_multilevel(const EdaGraph& g, std::uint32_t k, std::uint64_t seed) {
  auto d = g.to_device();
  groot_assignment* a = nullptr;
  detail::check(groot_partition_multilevel(d.get(), k, seed, &a, nullptr, nullptr));
  gpu::DeviceAssignment da(a);
  return PartitionAssignment::from_device(da.get());
}
inline PartitionAssignment load_assignment(const std::string& path, std::uint32_t n) {  // src/partition.cpp:369
  groot_assignment* a = nullptr;
  detail::check(groot_load_assignment(path.c_str(), n, &a));
  gpu::DeviceAssignment da(a);
  return PartitionAssignment::from_device(da.get());
}
inline void save_assignment(const std::string& path, const PartitionAssignment& pa) {
  std::ofstream out(path);
  if (!out) throw std::runtime_error("cannot write assignment file: " + path);
  for (std::size_t v = 0; v < pa.part_of.size(); ++v) out << v << ' ' << pa.part_of[v] << '\n';
}

namespace gpu {
inline DeviceParts regrow(const groot_graph* g, const groot_assignment* a, bool with_boundary = true) {
  groot_parts* p = nullptr;
  detail::check(groot_regrow(g, a, with_boundary ? 1 : 0, &p));
  return DeviceParts(p);
}
}  // namespace gpu

inline std::vector<AugmentedPartition> regrow(const EdaGraph& g, const PartitionAssignment& pa) {
  if (pa.part_of.size() != g.n) throw std::invalid_argument("regrow: assignment size mismatch");
  auto d = g.to_device();
  auto a = pa.to_device();
  return parts_from_device(gpu::regrow(d.get(), a.get(), true).get());
}
inline std::vector<AugmentedPartition> core_subgraphs(const EdaGraph& g, const PartitionAssignment& pa) {
  if (pa.part_of.size() != g.n) throw std::invalid_argument("regrow: assignment size mismatch");
  auto d = g.to_device();
  auto a = pa.to_device();
  return parts_from_device(gpu::regrow(d.get(), a.get(), false).get());
}
inline double crossing_fraction(const EdaGraph& g, const PartitionAssignment& pa) {  // src/partition.cpp:468-474
  auto d = g.to_device();
  auto a = pa.to_device();
  double f = 0.0;
  detail::check(groot_crossing_fraction(d.get(), a.get(), &f));
  return f;
}
inline std::uint64_t edge_cut(const EdaGraph& g, const PartitionAssignment& pa) {  // src/partition.cpp:508-513
  auto d = g.to_device();
  auto a = pa.to_device();
  std::uint64_t c = 0;
  detail::check(groot_edge_cut(d.get(), a.get(), &c));
  return c;
}
inline std::uint64_t footprint_proxy(const std::vector<AugmentedPartition>& parts, std::uint32_t feature_cols = 4,
                                     std::uint32_t hidden_dim = 32) {
  std::uint64_t peak = 0;
  for (const AugmentedPartition& p : parts)
    peak = std::max<std::uint64_t>(peak, static_cast<std::uint64_t>(p.size()) * (feature_cols + hidden_dim) * 4 +
                                             2 * static_cast<std::uint64_t>(p.edges.size()) * 8);
  return peak;
}
inline EdaGraph materialize(const EdaGraph& g, const AugmentedPartition& part) {  // src/partition.cpp:488
  const std::uint32_t n = part.size();
  std::vector<std::uint8_t> feat(4ull * n), lab(n);
  for (std::uint32_t i = 0; i < n; ++i) {
    const std::uint32_t v = part.local_to_global[i];
    for (int c = 0; c < 4; ++c) feat[4ull * i + c] = g.features[4ull * v + c];
    lab[i] = g.labels[v];
  }
  std::vector<std::uint32_t> edges(2 * part.edges.size());
  for (size_t i = 0; i < part.edges.size(); ++i) {
    edges[2 * i] = part.edges[i].first;
    edges[2 * i + 1] = part.edges[i].second;
  }
  groot_graph* d = nullptr;  // symmetric CSR built on the device (build_symmetric_csr)
  detail::check(groot_graph_from_edges(n, feat.data(), lab.data(), part.edges.size(),
                                       edges.empty() ? nullptr : edges.data(), &d));
  gpu::DeviceGraph dg(d);
  return EdaGraph::from_device(dg.get());
}

// ---- inc/gnn.hpp ---------------------------------------------------------------------
// Row-major dense matrix standing in for Eigen::Matrix<double, Dynamic, Dynamic, RowMajor>.
class RowMat {
 public:
  RowMat() = default;
  RowMat(std::int64_t r, std::int64_t c) : r_(r), c_(c), v_(static_cast<size_t>(r * c), 0.0) {}
  std::int64_t rows() const { return r_; }
  std::int64_t cols() const { return c_; }
  std::int64_t size() const { return r_ * c_; }
  double* data() { return v_.data(); }
  const double* data() const { return v_.data(); }
  double& operator()(std::int64_t i, std::int64_t j) { return v_[static_cast<size_t>(i * c_ + j)]; }
  double operator()(std::int64_t i, std::int64_t j) const { return v_[static_cast<size_t>(i * c_ + j)]; }

 private:
  std::int64_t r_ = 0, c_ = 0;
  std::vector<double> v_;
};
using RowVec = RowMat;  // 1 x n

struct SageLayer {
  RowMat w_self, w_neigh;
  RowVec bias;
};

struct Model {
  std::vector<SageLayer> layers;
  RowMat w_out;
  RowVec b_out;
  std::uint32_t in_dim() const { return static_cast<std::uint32_t>(layers.front().w_self.rows()); }
  std::uint32_t num_classes() const { return static_cast<std::uint32_t>(w_out.cols()); }

  // ASG1 parameter order: per layer W_self, W_neigh, bias; then W_out, b_out.
  std::vector<double> params() const {
    std::vector<double> p;
    auto add = [&](const RowMat& m) { p.insert(p.end(), m.data(), m.data() + m.size()); };
    for (const SageLayer& l : layers) {
      add(l.w_self);
      add(l.w_neigh);
      add(l.bias);
    }
    add(w_out);
    add(b_out);
    return p;
  }
  static Model from_params(const std::vector<double>& p, std::uint32_t depth, std::uint32_t in, std::uint32_t hid,
                           std::uint32_t classes) {
    Model m;
    size_t off = 0;
    auto take = [&](std::uint32_t r, std::uint32_t c) {
      RowMat x(r, c);
      for (std::int64_t i = 0; i < x.size(); ++i) x.data()[i] = p.at(off++);
      return x;
    };
    std::uint32_t d = in;
    for (std::uint32_t l = 0; l < depth; ++l) {
      SageLayer L;
      L.w_self = take(d, hid);
      L.w_neigh = take(d, hid);
      L.bias = take(1, hid);
      m.layers.push_back(std::move(L));
      d = hid;
    }
    m.w_out = take(d, classes);
    m.b_out = take(1, classes);
    return m;
  }
  gpu::DeviceModel to_device() const {
    const auto p = params();
    groot_model* dm = nullptr;
    detail::check(groot_model_create(static_cast<std::uint32_t>(layers.size()), in_dim(),
                                     static_cast<std::uint32_t>(layers.front().w_self.cols()), num_classes(), p.data(),
                                     &dm));
    return gpu::DeviceModel(dm);
  }
};

// init_model (src/gnn.cpp:113-138): identical weights (mt19937_64 Glorot).
inline Model init_model(std::uint64_t seed, std::uint32_t in_dim = 4, std::uint32_t hidden = 32,
                        std::uint32_t num_classes = kNumClasses, std::uint32_t depth = 4) {
  std::vector<double> p(groot_param_count(depth, in_dim, hidden, num_classes));
  detail::check(groot_init_params(seed, in_dim, hidden, num_classes, depth, p.data()));
  return Model::from_params(p, depth, in_dim, hidden, num_classes);
}

inline Model load_model(const std::string& path) {  // src/gnn.cpp:349-372
  groot_model* dm = nullptr;
  detail::check(groot_model_load(path.c_str(), &dm));
  gpu::DeviceModel m(dm);
  std::uint32_t depth, in, hid, cls;
  detail::check(groot_model_info(m.get(), &depth, &in, &hid, &cls));
  std::vector<double> p(groot_param_count(depth, in, hid, cls));
  detail::check(groot_model_params(m.get(), p.data()));
  return Model::from_params(p, depth, in, hid, cls);
}
inline void save_model(const std::string& path, const Model& model) {  // src/gnn.cpp:330-345
  auto m = model.to_device();
  detail::check(groot_model_save(m.get(), path.c_str()));
}

// ---- training (inc/gnn.hpp:38-50, src/gnn.cpp:180-255), fp64 on the device ---------------
struct TrainConfig {
  std::uint32_t epochs = 100;
  double learning_rate = 1e-3;
  std::uint64_t seed = 7;
  double beta1 = 0.9;
  double beta2 = 0.999;
  double adam_eps = 1e-8;
};
struct TrainStats {
  std::vector<double> loss;
  std::vector<double> accuracy;
};
inline Model train(const EdaGraph& g, const TrainConfig& cfg, TrainStats* stats = nullptr) {
  if (cfg.learning_rate <= 0) throw std::invalid_argument("train: learning rate must be positive");
  auto d = g.to_device();
  const std::uint32_t depth = 4, in = 4, hid = 32, cls = kNumClasses;
  std::vector<double> p(groot_param_count(depth, in, hid, cls)), loss(cfg.epochs), acc(cfg.epochs);
  detail::check(groot_train(d.get(), depth, in, hid, cls, cfg.epochs, cfg.learning_rate, cfg.seed, cfg.beta1, cfg.beta2,
                            cfg.adam_eps, nullptr, p.data(), loss.data(), acc.data()));
  if (stats) {
    stats->loss = loss;
    stats->accuracy = acc;
  }
  return Model::from_params(p, depth, in, hid, cls);
}
// grad_check (inc/gnn.hpp:88-90): max |a - n| / max(|a|, |n|, 1) over every
// parameter, analytic (device backward) vs central differences (device loss).
inline double grad_check(const Model& model, const EdaGraph& g, double epsilon = 1e-4) {
  auto d = g.to_device();
  const std::uint32_t depth = static_cast<std::uint32_t>(model.layers.size()), in = model.in_dim(),
                      hid = static_cast<std::uint32_t>(model.layers.front().w_self.cols()), cls = model.num_classes();
  std::vector<double> p = model.params(), ana(p.size()), scratch(p.size());
  double loss = 0, worst = 0;
  detail::check(groot_loss_and_grads(d.get(), depth, in, hid, cls, p.data(), ana.data(), &loss));
  for (std::size_t i = 0; i < p.size(); ++i) {
    const double keep = p[i];
    double lp = 0, lm = 0;
    p[i] = keep + epsilon;
    detail::check(groot_loss_and_grads(d.get(), depth, in, hid, cls, p.data(), nullptr, &lp));
    p[i] = keep - epsilon;
    detail::check(groot_loss_and_grads(d.get(), depth, in, hid, cls, p.data(), nullptr, &lm));
    p[i] = keep;
    const double num = (lp - lm) / (2 * epsilon);
    worst = std::max(worst, std::abs(ana[i] - num) / std::max({std::abs(ana[i]), std::abs(num), 1.0}));
  }
  return worst;
}

struct Prediction {
  std::vector<std::uint8_t> labels;
  std::array<std::array<std::uint64_t, kNumClasses>, kNumClasses> confusion{};
  double accuracy = 0.0;
};

inline RowMat forward(const Model& model, const EdaGraph& g) {  // src/gnn.cpp:172-178
  auto m = model.to_device();
  auto d = g.to_device();
  std::vector<float> lg(static_cast<size_t>(g.n) * model.num_classes());
  detail::check(groot_forward(m.get(), d.get(), lg.data()));
  RowMat out(g.n, model.num_classes());
  for (size_t i = 0; i < lg.size(); ++i) out.data()[i] = lg[i];
  return out;
}

namespace detail {
inline Prediction finish(std::vector<std::uint8_t> labels, const std::uint64_t* conf, double acc) {
  Prediction p;
  p.labels = std::move(labels);
  for (std::uint32_t t = 0; t < kNumClasses; ++t)
    for (std::uint32_t q = 0; q < kNumClasses; ++q) p.confusion[t][q] = conf[t * kNumClasses + q];
  p.accuracy = acc;
  return p;
}
}  // namespace detail

inline Prediction predict_full(const Model& model, const EdaGraph& g) {  // src/gnn.cpp:293-300
  auto m = model.to_device();
  auto d = g.to_device();
  std::vector<std::uint8_t> labels(g.n);
  std::uint64_t conf[25];
  double acc = 0;
  detail::check(groot_predict_full(m.get(), d.get(), labels.data(), conf, &acc));
  return detail::finish(std::move(labels), conf, acc);
}

// predict (src/gnn.cpp:280-291): every part forwarded as given, each node scored
// from the part that holds it as a core node.
inline Prediction predict(const Model& model, const EdaGraph& g, const std::vector<AugmentedPartition>& parts) {
  auto m = model.to_device();
  auto d = g.to_device();
  auto dp = parts_to_device(g.n, parts);
  std::vector<std::uint8_t> labels(g.n);
  std::uint64_t conf[25];
  double acc = 0;
  detail::check(groot_predict(m.get(), d.get(), dp.get(), labels.data(), conf, &acc));
  return detail::finish(std::move(labels), conf, acc);
}

// ---- inc/worker_pool.hpp -----------------------------------------------------------
// Host thread pool with the reference's surface (inc/worker_pool.hpp:18-56). The
// device path does not use it (the GPU is the parallelism); it is here so caller
// code that builds or passes pools compiles and runs unchanged.
class WorkerPool {
 public:
  explicit WorkerPool(unsigned workers = 0) : workers_(workers ? workers : default_workers()) {}
  WorkerPool(const WorkerPool&) = delete;
  WorkerPool& operator=(const WorkerPool&) = delete;
  unsigned workers() const { return workers_; }
  void for_each(std::size_t count, const std::function<void(std::size_t)>& fn) {
    if (workers_ <= 1 || count <= 1 || busy_.exchange(true)) {  // nested / concurrent: inline
      for (std::size_t i = 0; i < count; ++i) fn(i);
      return;
    }
    std::atomic<std::size_t> next{0};
    auto run = [&] {
      for (std::size_t i = next++; i < count; i = next++) fn(i);
    };
    std::vector<std::thread> ts;
    for (unsigned t = 1; t < workers_; ++t) ts.emplace_back(run);
    run();
    for (auto& t : ts) t.join();
    busy_ = false;
  }
  static unsigned default_workers() {
    if (const char* e = std::getenv("AIGSAGE_WORKERS")) {
      const long v = std::strtol(e, nullptr, 10);
      if (v > 0) return static_cast<unsigned>(v);
    }
    const unsigned h = std::thread::hardware_concurrency();
    return h ? h : 1u;
  }

 private:
  unsigned workers_ = 1;
  std::atomic<bool> busy_{false};
};
inline WorkerPool& default_pool() {
  static WorkerPool pool;
  return pool;
}

// ---- inc/spmm.hpp ---------------------------------------------------------------------
namespace spmm {
template <class T>
struct CsrMatrix {
  std::uint32_t rows = 0, cols = 0;
  std::vector<std::uint64_t> row_ptr;
  std::vector<std::uint32_t> col_idx;
  std::vector<T> values;
  std::uint64_t nnz() const { return row_ptr.empty() ? 0 : row_ptr.back(); }
  std::uint32_t degree(std::uint32_t r) const { return static_cast<std::uint32_t>(row_ptr[r + 1] - row_ptr[r]); }
  void validate() const {  // inc/spmm.hpp:25-36, same messages
    if (row_ptr.size() != static_cast<std::size_t>(rows) + 1) throw std::invalid_argument("CsrMatrix: row_ptr size");
    for (std::uint32_t r = 0; r < rows; ++r)
      if (row_ptr[r] > row_ptr[r + 1]) throw std::invalid_argument("CsrMatrix: row_ptr not monotone");
    if (col_idx.size() != nnz() || values.size() != nnz()) throw std::invalid_argument("CsrMatrix: nnz mismatch");
    for (std::uint32_t c : col_idx)
      if (c >= cols) throw std::invalid_argument("CsrMatrix: column index out of range");
  }
};

struct DegreeSort {
  std::vector<std::uint32_t> perm;            // sorted position -> original row
  std::vector<std::uint64_t> sorted_row_ptr;  // row pointers in the new order
};

// degree_sort (src/spmm.cpp:9-35): stable ascending by degree, on the device.
inline DegreeSort degree_sort(std::uint32_t rows, std::span<const std::uint64_t> row_ptr) {
  if (row_ptr.size() != static_cast<std::size_t>(rows) + 1) throw std::invalid_argument("degree_sort: row_ptr size");
  DegreeSort d;
  d.perm.resize(rows);
  d.sorted_row_ptr.resize(rows + 1ull);
  detail::check(groot_degree_sort(rows, row_ptr.data(), d.perm.data(), d.sorted_row_ptr.data()));
  return d;
}
template <class T>
DegreeSort degree_sort(const CsrMatrix<T>& m) {
  return degree_sort(m.rows, m.row_ptr);
}

enum class WorkKind : std::uint8_t { HdChunk, LdBatch, MidRow };
struct WorkUnit {
  WorkKind kind;
  std::uint32_t sorted_row = 0;
  std::uint32_t row_count = 1;
  std::uint64_t nz_begin = 0;
  std::uint64_t nz_end = 0;
  std::uint32_t partial_slot = 0;
};
struct LdGroup {
  std::uint32_t degree;
  std::uint32_t row_begin;
  std::uint32_t row_end;
};
struct SpmmPlan {  // inc/spmm.hpp:72-90
  std::uint32_t rows = 0;
  std::uint64_t nnz = 0;
  std::vector<std::uint32_t> perm;
  std::vector<std::uint32_t> inv_perm;
  std::vector<std::uint64_t> sorted_row_ptr;
  std::vector<std::uint32_t> hd_rows;
  std::vector<LdGroup> ld_groups;
  std::vector<std::uint32_t> mid_rows;
  std::vector<WorkUnit> work_units;
  std::uint32_t hd_threshold = 512;
  std::uint32_t ld_threshold = 12;
  std::uint32_t nz_budget = 96;
  std::uint32_t ld_row_begin = 0;
  std::uint32_t ld_row_end = 0;
  unsigned workers = 0;
};
inline constexpr std::uint32_t kHdChunksPerRow = 32;

// build_plan (src/spmm.cpp:37-127): the row classifier; the degree sort runs on
// the device, the unit list is the reference's exactly.
inline SpmmPlan build_plan(std::uint32_t rows, std::span<const std::uint64_t> row_ptr, unsigned workers,
                           std::uint32_t hd_threshold = 512, std::uint32_t ld_threshold = 12,
                           std::uint32_t nz_budget = 96) {
  if (row_ptr.size() != static_cast<std::size_t>(rows) + 1) throw std::invalid_argument("build_plan: row_ptr size");
  std::uint64_t counts[6];
  detail::check(groot_build_plan_rows(rows, row_ptr.data(), hd_threshold, ld_threshold, nz_budget, counts, nullptr,
                                      nullptr, nullptr, nullptr, nullptr));
  SpmmPlan p;
  p.rows = rows;
  p.nnz = row_ptr[rows];
  p.hd_threshold = hd_threshold;
  p.ld_threshold = ld_threshold;
  p.nz_budget = nz_budget;
  p.workers = workers;
  p.perm.resize(rows);
  p.hd_rows.resize(counts[0]);
  p.mid_rows.resize(counts[1]);
  std::vector<std::uint32_t> ldg(3 * counts[2]);
  std::vector<std::uint64_t> units(6 * counts[3]);
  detail::check(groot_build_plan_rows(rows, row_ptr.data(), hd_threshold, ld_threshold, nz_budget, counts,
                                      p.perm.data(), p.hd_rows.data(), p.mid_rows.data(), ldg.data(), units.data()));
  p.ld_row_begin = static_cast<std::uint32_t>(counts[4]);
  p.ld_row_end = static_cast<std::uint32_t>(counts[5]);
  p.inv_perm.resize(rows);
  for (std::uint32_t s = 0; s < rows; ++s) p.inv_perm[p.perm[s]] = s;
  p.sorted_row_ptr.assign(rows + 1ull, 0);
  for (std::uint32_t s = 0; s < rows; ++s)
    p.sorted_row_ptr[s + 1] = p.sorted_row_ptr[s] + (row_ptr[p.perm[s] + 1] - row_ptr[p.perm[s]]);
  for (std::uint64_t i = 0; i < counts[2]; ++i) p.ld_groups.push_back({ldg[3 * i], ldg[3 * i + 1], ldg[3 * i + 2]});
  for (std::uint64_t i = 0; i < counts[3]; ++i) {
    const std::uint64_t* u = &units[6 * i];
    const WorkKind kind = u[0] == 0 ? WorkKind::HdChunk : (u[0] == 1 ? WorkKind::LdBatch : WorkKind::MidRow);
    p.work_units.push_back({kind, static_cast<std::uint32_t>(u[1]), static_cast<std::uint32_t>(u[2]), u[3], u[4],
                            static_cast<std::uint32_t>(u[5])});
  }
  return p;
}
template <class T>
SpmmPlan build_plan(const CsrMatrix<T>& m, unsigned workers, std::uint32_t hd_threshold = 512,
                    std::uint32_t ld_threshold = 12, std::uint32_t nz_budget = 96) {
  return build_plan(m.rows, m.row_ptr, workers, hd_threshold, ld_threshold, nz_budget);
}

namespace detail {
// out = m * dense on the device, rows of degree >= hd_threshold as 32 ordered chunk
// partials (0: plain row loop). Bitwise the reference's arithmetic for T = float, double.
template <class T>
void device_spmm(const CsrMatrix<T>& m, const T* dense, std::uint32_t f, T* out, std::uint32_t hd_threshold) {
  static_assert(std::is_same_v<T, float> || std::is_same_v<T, double>, "spmm: float or double values");
  if constexpr (std::is_same_v<T, double>)
    aigsage::detail::check(groot_spmm_csr_f64(m.rows, m.cols, m.row_ptr.data(), m.col_idx.data(),
                                              m.values.empty() ? nullptr : m.values.data(), dense, f, hd_threshold, out));
  else
    aigsage::detail::check(groot_spmm_csr(m.rows, m.cols, m.row_ptr.data(), m.col_idx.data(),
                                          m.values.empty() ? nullptr : m.values.data(), dense, f, hd_threshold, out));
}
}  // namespace detail

// execute (inc/spmm.hpp:106-170): out = m * dense on the device; bitwise the
// reference's result for this plan (same per-row order, HD rows as 32 ordered
// chunk partials). The pool argument is accepted and unused.
template <class T>
void execute(const SpmmPlan& plan, const CsrMatrix<T>& m, const T* dense, std::uint32_t f, T* out,
             WorkerPool* pool = nullptr) {
  (void)pool;
  if (m.rows != plan.rows || m.nnz() != plan.nnz)
    throw std::invalid_argument("spmm::execute: plan does not match matrix");
  detail::device_spmm(m, dense, f, out, plan.hd_rows.empty() ? 0u : plan.hd_threshold);
}
template <class T>
std::vector<T> execute(const SpmmPlan& plan, const CsrMatrix<T>& m, const std::vector<T>& dense, std::uint32_t f,
                       WorkerPool* pool = nullptr) {
  if (dense.size() != static_cast<std::size_t>(m.cols) * f) throw std::invalid_argument("spmm::execute: dense shape mismatch");
  std::vector<T> out(static_cast<std::size_t>(m.rows) * f);
  execute(plan, m, dense.data(), f, out.data(), pool);
  return out;
}
// Convenience (no plan argument): the plan the reference would build by default.
template <class T>
std::vector<T> execute(const CsrMatrix<T>& m, const std::vector<T>& dense, std::uint32_t f) {
  return execute(build_plan(m, 0), m, dense, f);
}

// reference_spmm (inc/spmm.hpp:183-204): plain row loop, on the device.
template <class T>
void reference_spmm(const CsrMatrix<T>& m, const T* dense, std::uint32_t f, T* out) {
  detail::device_spmm(m, dense, f, out, 0u);
}
template <class T>
std::vector<T> reference_spmm(const CsrMatrix<T>& m, const std::vector<T>& dense, std::uint32_t f) {
  if (dense.size() != static_cast<std::size_t>(m.cols) * f)
    throw std::invalid_argument("spmm::reference_spmm: dense shape mismatch");
  std::vector<T> out(static_cast<std::size_t>(m.rows) * f);
  reference_spmm(m, dense.data(), f, out.data());
  return out;
}
// row_parallel_reference (inc/spmm.hpp:206-225): same result as reference_spmm.
template <class T>
void row_parallel_reference(const CsrMatrix<T>& m, const T* dense, std::uint32_t f, T* out, WorkerPool& pool) {
  (void)pool;
  reference_spmm(m, dense, f, out);
}

struct BenchReport {
  double plan_ms = 0;
  double exec_ms = 0;
  double baseline_ms = 0;
  double speedup = 0;  // baseline_ms / exec_ms
  unsigned workers = 0;
  int reps = 0;
};
// bench (src/spmm.cpp:129-175): median-of-reps wall time of build_plan + execute
// against the row loop, f columns of U(-1,1) from mt19937_64(0xb00b1e5), through
// the host entry points (copies included).
inline BenchReport bench(const CsrMatrix<float>& m, std::uint32_t f, int reps, WorkerPool* pool = nullptr) {
  m.validate();
  std::mt19937_64 rng(0xb00b1e5);
  std::uniform_real_distribution<float> dist(-1.0f, 1.0f);
  std::vector<float> dense(static_cast<std::size_t>(m.cols) * f), out(static_cast<std::size_t>(m.rows) * f);
  for (float& x : dense) x = dist(rng);
  auto ms_of = [](auto fn) {
    const auto t0 = std::chrono::steady_clock::now();
    fn();
    return std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  };
  auto median = [](std::vector<double> v) {
    std::sort(v.begin(), v.end());
    return v.empty() ? 0.0 : v[v.size() / 2];
  };
  BenchReport r;
  r.reps = reps < 1 ? 1 : reps;
  r.workers = pool ? pool->workers() : 0;
  SpmmPlan plan;
  r.plan_ms = ms_of([&] { plan = build_plan(m, r.workers); });
  std::vector<double> ex, base;
  for (int i = 0; i < r.reps; ++i) {
    ex.push_back(ms_of([&] { execute(plan, m, dense.data(), f, out.data(), pool); }));
    base.push_back(ms_of([&] { reference_spmm(m, dense.data(), f, out.data()); }));
  }
  r.exec_ms = median(ex);
  r.baseline_ms = median(base);
  r.speedup = r.exec_ms > 0 ? r.baseline_ms / r.exec_ms : 0.0;
  return r;
}
}  // namespace spmm

// ---- inc/gnn.hpp: SageContext (src/gnn.cpp:140-178) ------------------------------------
// The reference's host fields (a_mean = D^-1 A, a_mean_t = A D^-1 with 1/deg values,
// their plans, features as an n x 4 matrix, labels) plus the graph resident in
// HBM with the device's per-graph state built (groot_graph_prepare: row
// classifier, tile plan, HD chunk plan, activations). forward(model, ctx) runs
// on that resident graph without re-uploading or re-planning it.
struct SageContext {
  spmm::CsrMatrix<double> a_mean;
  spmm::CsrMatrix<double> a_mean_t;
  spmm::SpmmPlan plan;
  spmm::SpmmPlan plan_t;
  RowMat features;
  std::vector<std::uint8_t> labels;
  std::shared_ptr<groot_graph> device;
};

inline SageContext make_context(const EdaGraph& g) {
  SageContext c;
  c.a_mean.rows = c.a_mean.cols = g.n;
  c.a_mean.row_ptr = g.row_ptr;
  c.a_mean.col_idx = g.col_idx;
  c.a_mean.values.resize(g.col_idx.size());
  c.a_mean_t = c.a_mean;
  for (std::uint32_t v = 0; v < g.n; ++v) {
    const double inv = g.degree[v] ? 1.0 / g.degree[v] : 0.0;
    for (std::uint64_t q = g.row_ptr[v]; q < g.row_ptr[v + 1]; ++q) {
      c.a_mean.values[q] = inv;
      const std::uint32_t u = g.col_idx[q];
      c.a_mean_t.values[q] = g.degree[u] ? 1.0 / g.degree[u] : 0.0;
    }
  }
  c.plan = spmm::build_plan(c.a_mean, 0);
  c.plan_t = spmm::build_plan(c.a_mean_t, 0);
  c.features = RowMat(g.n, 4);
  for (std::size_t i = 0; i < g.features.size(); ++i) c.features.data()[i] = g.features[i];
  c.labels = g.labels;
  auto d = g.to_device();
  detail::check(groot_graph_prepare(d.get()));
  c.device = std::shared_ptr<groot_graph>(d.release(), gpu::GraphDeleter{});
  return c;
}

inline RowMat forward(const Model& model, const SageContext& ctx) {  // src/gnn.cpp:172-178
  auto m = model.to_device();
  std::uint32_t n;
  std::uint64_t nnz, ne;
  detail::check(groot_graph_sizes(ctx.device.get(), &n, &nnz, &ne));
  std::vector<float> lg(static_cast<size_t>(n) * model.num_classes());
  detail::check(groot_forward(m.get(), ctx.device.get(), lg.data()));
  RowMat out(n, model.num_classes());
  for (size_t i = 0; i < lg.size(); ++i) out.data()[i] = lg[i];
  return out;
}

}  // namespace aigsage
