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
//  * GroundTruth::supports is not populated by gen_csa_multiplier (it only
//    feeds the verifier, which is outside the hot path).
//  * aigsage::gpu::DeviceGraph keeps a graph resident in HBM across calls;
//    the value-returning functions copy to the host like the reference does.
//
// Link: -I include -L paper_2511_18297_b200 -lgroot_b200
#pragma once

#include <array>
#include <cstdint>
#include <fstream>
#include <iterator>
#include <map>
#include <memory>
#include <sstream>
#include <stdexcept>
#include <string>
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

// ---- inc/circuitgen.hpp ---------------------------------------------------------
enum class NodeClass : std::uint8_t { Po = 0, Maj = 1, Xor = 2, And = 3, Pi = 4 };
inline constexpr std::uint32_t kNumClasses = 5;

struct GroundTruth {
  std::vector<std::uint8_t> labels;
  std::vector<std::uint32_t> po_nodes;
  std::map<std::uint32_t, std::vector<Literal>> supports;  // not populated (verifier input only)
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

inline PartitionAssignment partition_topo_chunks(const EdaGraph& g, std::uint32_t k) {  // src/partition.cpp:301
  auto d = g.to_device();
  groot_assignment* a = nullptr;
  detail::check(groot_partition_topo_chunks(d.get(), k, &a));
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
inline double crossing_fraction(const EdaGraph& g, const PartitionAssignment& pa) {
  if (g.fwd_edges.empty()) return 0.0;
  std::uint64_t c = 0;
  for (const auto& [u, v] : g.fwd_edges) c += pa.part_of[u] != pa.part_of[v];
  return static_cast<double>(c) / static_cast<double>(g.fwd_edges.size());
}
inline std::uint64_t edge_cut(const EdaGraph& g, const PartitionAssignment& pa) {
  std::uint64_t c = 0;
  for (const auto& [u, v] : g.fwd_edges) c += pa.part_of[u] != pa.part_of[v];
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

inline Prediction predict(const Model& model, const EdaGraph& g, const std::vector<AugmentedPartition>& parts) {
  // src/gnn.cpp:280-291: the parts are re-derived on the device from their core sets.
  PartitionAssignment pa;
  pa.part_of.assign(g.n, 0);
  pa.k = static_cast<std::uint32_t>(parts.size());
  bool regrown = false;
  for (std::uint32_t p = 0; p < parts.size(); ++p) {
    for (std::uint32_t v : parts[p].core_nodes) pa.part_of[v] = p;
    regrown = regrown || !parts[p].boundary_nodes.empty();
  }
  auto m = model.to_device();
  auto d = g.to_device();
  auto a = pa.to_device();
  auto dp = gpu::regrow(d.get(), a.get(), regrown);
  std::vector<std::uint8_t> labels(g.n);
  std::uint64_t conf[25];
  double acc = 0;
  detail::check(groot_predict(m.get(), d.get(), dp.get(), labels.data(), conf, &acc));
  return detail::finish(std::move(labels), conf, acc);
}

// ---- inc/spmm.hpp (API parity) -----------------------------------------------------------
namespace spmm {
template <class T>
struct CsrMatrix {
  std::uint32_t rows = 0, cols = 0;
  std::vector<std::uint64_t> row_ptr;
  std::vector<std::uint32_t> col_idx;
  std::vector<T> values;
  std::uint64_t nnz() const { return row_ptr.empty() ? 0 : row_ptr.back(); }
  std::uint32_t degree(std::uint32_t r) const { return static_cast<std::uint32_t>(row_ptr[r + 1] - row_ptr[r]); }
};

// out = m * dense (spmm::execute, inc/spmm.hpp:106-181) on the device, fp32.
template <class T>
std::vector<T> execute(const CsrMatrix<T>& m, const std::vector<T>& dense, std::uint32_t f) {
  if (dense.size() != static_cast<size_t>(m.cols) * f) throw std::invalid_argument("spmm::execute: dense shape mismatch");
  std::vector<float> v(m.values.begin(), m.values.end()), d(dense.begin(), dense.end()),
      o(static_cast<size_t>(m.rows) * f);
  detail::check(groot_spmm_csr(m.rows, m.cols, m.row_ptr.data(), m.col_idx.data(), v.data(), d.data(), f, o.data()));
  return std::vector<T>(o.begin(), o.end());
}
}  // namespace spmm

}  // namespace aigsage
