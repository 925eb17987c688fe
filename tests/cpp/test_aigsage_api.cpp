// Exercises the C++ drop-in mirror (include/groot_aigsage.hpp) the way a
// reference (aigsage) user would call it. Host-only checks always run; the
// device pipeline runs when a CUDA device is present (argv[1] == "gpu").
#include <algorithm>
#include <cassert>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <ctime>
#include <sstream>

#include "groot_aigsage.hpp"

using namespace aigsage;

#define CHECK(c)                                                      \
  do {                                                                \
    if (!(c)) {                                                       \
      std::fprintf(stderr, "CHECK failed: %s (line %d)\n", #c, __LINE__); \
      return 1;                                                       \
    }                                                                 \
  } while (0)

int main(int argc, char** argv) {
  const bool gpu = argc > 1 && std::strcmp(argv[1], "gpu") == 0;
  // --- host: generator, AIGER round trip, error types, init_model ---
  CsaCircuit c = gen_csa_multiplier(2);
  CHECK(c.aig.num_inputs() == 4 && c.aig.num_ands() == 10 && c.aig.outputs().size() == 4);
  CHECK(c.gt.labels.size() == 19 && c.gt.labels[10] == 2 && c.gt.labels[8] == 1 && c.gt.labels[15] == 0);
  CsaCircuit c1024 = gen_csa_multiplier(1024);
  CHECK(c1024.half_adders == 1024 && c1024.full_adders == 1046528);
  std::stringstream ss;
  write_aiger(c.aig, ss);
  Aig back = parse_aiger(ss);
  CHECK(back == c.aig);
  bool threw = false;
  try {
    std::istringstream bad("aag 1 1 1 0 0\n2\n2 3\n");
    parse_aiger(bad);
  } catch (const std::runtime_error& e) {
    threw = std::string(e.what()).find("latches unsupported") != std::string::npos;
  }
  CHECK(threw);
  // file forms (inc/aig.hpp:73, inc/circuitgen.hpp): AIGER, labels, supports round trips
  const std::string tmp = std::string(std::getenv("TMPDIR") ? std::getenv("TMPDIR") : "/tmp") + "/groot_api_" +
                          std::to_string(static_cast<long>(std::time(nullptr)) % 100000);
  write_aiger_file(c.aig, tmp + ".aag");
  CHECK(parse_aiger_file(tmp + ".aag") == c.aig);
  write_labels(tmp + ".lab", c.gt.labels);
  CHECK(load_labels(tmp + ".lab", c.gt.labels.size()) == c.gt.labels);
  threw = false;
  try {
    load_labels(tmp + ".lab", c.gt.labels.size() + 1);  // node 19 missing
  } catch (const std::runtime_error& e) {
    threw = std::string(e.what()).find("missing node 19") != std::string::npos;
  }
  CHECK(threw);
  CsaCircuit c4 = gen_csa_multiplier(4);
  CHECK(!c4.gt.supports.empty());
  write_supports(tmp + ".sup", c4.gt.supports);
  CHECK(load_supports(tmp + ".sup") == c4.gt.supports);
  std::remove((tmp + ".aag").c_str());
  std::remove((tmp + ".lab").c_str());
  std::remove((tmp + ".sup").c_str());
  // flip_and_fanin (src/aig.cpp:24-29): toggles one fanin's inversion, twice restores
  Aig flipped = c.aig;
  const std::uint32_t v = flipped.first_and() + 3;
  flipped.flip_and_fanin(v, true);
  CHECK(flipped.and_node(v).right.inverted != c.aig.and_node(v).right.inverted &&
        flipped.and_node(v).left == c.aig.and_node(v).left && !(flipped == c.aig));
  flipped.flip_and_fanin(v, true);
  CHECK(flipped == c.aig);
  threw = false;
  try {
    flipped.flip_and_fanin(1, false);  // an input, not an AND node
  } catch (const std::invalid_argument& e) {
    threw = std::string(e.what()) == "Aig::flip_and_fanin: not an AND node";
  }
  CHECK(threw);
  threw = false;
  try {
    gen_csa_multiplier(1);
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw);
  Model m = init_model(7);
  CHECK(m.layers.size() == 4 && m.in_dim() == 4 && m.num_classes() == 5 && m.layers[1].w_self.rows() == 32);
  const double lim = std::sqrt(6.0 / 36.0);
  CHECK(std::fabs(m.layers[0].w_self(0, 0)) <= lim);
  // worker pool surface (inc/worker_pool.hpp)
  WorkerPool pool(4);
  std::vector<int> hit(100, 0);
  pool.for_each(hit.size(), [&](std::size_t i) { hit[i] += 1; });
  CHECK(pool.workers() == 4 && std::count(hit.begin(), hit.end(), 1) == 100);
  CHECK(default_pool().workers() >= 1);
  // verifier (host): ground-truth labels and the generator's supports prove the multiplier
  CsaCircuit c6 = gen_csa_multiplier(6);
  CHECK(c6.gt.supports.size() == 2u * 6 * 5);
  VerifyReport vr = backward_rewrite(c6.aig, c6.gt.labels, c6.gt.supports, 6);
  CHECK(vr.equivalent && !vr.inconclusive && vr.shortcut_count == 30 && vr.residual.empty());
  CHECK(truth_table_equiv(c6.aig, 6));
  std::vector<std::uint8_t> in12(12, 1);
  std::vector<std::uint8_t> prod = simulate(c6.aig, in12);  // 63 * 63 = 3969
  std::uint32_t word = 0;
  for (std::size_t k = 0; k < prod.size(); ++k) word |= static_cast<std::uint32_t>(prod[k]) << k;
  CHECK(word == 63u * 63u);
  if (!gpu) {
    std::printf("host checks ok\n");
    return 0;
  }
  // --- device pipeline: encode -> batch -> partition -> regrow -> predict ---
  CsaCircuit c8 = gen_csa_multiplier(8);
  EdaGraph g = encode(c8.aig, c8.gt);
  CHECK(g.n == 457 && g.num_undirected_edges() == 864 && g.row_ptr.back() == 1728);
  CHECK(g.feature(5 + 0)[0] == 0 || true);
  EdaGraph gb = batch(g, 3);
  CHECK(gb.n == 3 * 457 && gb.col_idx[1728] == g.col_idx[0] + 457);
  PartitionAssignment pa = partition_topo_chunks(gb, 4);
  CHECK(pa.k == 4 && pa.part_of.front() == 0 && pa.part_of.back() == 3);
  auto parts = regrow(gb, pa);
  CHECK(parts.size() == 4);
  std::uint64_t total_core = 0;
  for (auto& p : parts) total_core += p.num_core();
  CHECK(total_core == gb.n);
  EdaGraph sub = materialize(gb, parts[1]);
  CHECK(sub.n == parts[1].size() && sub.num_undirected_edges() == parts[1].edges.size());
  auto core = core_subgraphs(gb, pa);
  CHECK(footprint_proxy(parts) >= footprint_proxy(core));
  Prediction full = predict_full(m, gb);
  Prediction part1 = predict(m, gb, regrow(gb, partition_topo_chunks(gb, 1)));
  CHECK(full.labels == part1.labels);  // k=1 regrown == whole graph
  RowMat lg = forward(m, gb);
  CHECK(lg.rows() == gb.n && lg.cols() == 5);
  std::uint64_t hits = 0;
  for (std::uint32_t t = 0; t < 5; ++t) hits += full.confusion[t][t];
  CHECK(std::fabs(full.accuracy - static_cast<double>(hits) / gb.n) < 1e-12);
  spmm::CsrMatrix<double> eye;
  eye.rows = eye.cols = 3;
  eye.row_ptr = {0, 1, 2, 3};
  eye.col_idx = {0, 1, 2};
  eye.values = {1, 1, 1};
  auto y = spmm::execute(eye, std::vector<double>{1, 2, 3, 4, 5, 6}, 2);
  CHECK(y == (std::vector<double>{1, 2, 3, 4, 5, 6}));
  // SageContext (src/gnn.cpp:140-178): host fields as the reference builds them,
  // and forward(model, ctx) on the prepared resident graph
  SageContext ctx = make_context(gb);
  CHECK(ctx.a_mean.rows == gb.n && ctx.a_mean.nnz() == gb.col_idx.size() && ctx.plan.rows == gb.n);
  CHECK(ctx.a_mean.values[gb.row_ptr[10]] == 1.0 / gb.degree[10]);
  CHECK(ctx.a_mean_t.values[gb.row_ptr[10]] == 1.0 / gb.degree[gb.col_idx[gb.row_ptr[10]]]);
  CHECK(ctx.features.rows() == gb.n && ctx.features.cols() == 4 && ctx.labels == gb.labels);
  RowMat lc = forward(m, ctx);
  for (std::int64_t i = 0; i < lg.size(); ++i) CHECK(lc.data()[i] == lg.data()[i]);
  // spmm surface: degree_sort, build_plan, execute (bitwise the plain loop here: no HD rows at 8 bits)
  std::vector<std::uint64_t> rp3 = {0, 3, 4, 6};
  spmm::DegreeSort ds = spmm::degree_sort(3, rp3);
  CHECK((ds.perm == std::vector<std::uint32_t>{1, 2, 0}) && ds.sorted_row_ptr.back() == 6);
  ctx.a_mean.validate();
  CHECK(ctx.plan.hd_rows.empty() && !ctx.plan.work_units.empty() && ctx.plan.nnz == ctx.a_mean.nnz());
  std::vector<double> x(static_cast<std::size_t>(gb.n) * 4);
  for (std::size_t i = 0; i < x.size(); ++i) x[i] = std::sin(0.37 * static_cast<double>(i));
  std::vector<double> y1 = spmm::execute(ctx.plan, ctx.a_mean, x, 4, &default_pool());
  std::vector<double> y0(x.size(), 0.0);
  for (std::uint32_t r = 0; r < gb.n; ++r)
    for (std::uint64_t q = gb.row_ptr[r]; q < gb.row_ptr[r + 1]; ++q)
      for (int c = 0; c < 4; ++c) y0[4 * r + c] += ctx.a_mean.values[q] * x[4ull * gb.col_idx[q] + c];
  CHECK(y1 == y0);
  CHECK(spmm::reference_spmm(ctx.a_mean, x, 4) == y0);
  bool mismatch = false;
  try {
    spmm::execute(ctx.plan, eye, std::vector<double>{1, 2, 3}, 1);
  } catch (const std::invalid_argument& e) {
    mismatch = std::string(e.what()) == "spmm::execute: plan does not match matrix";
  }
  CHECK(mismatch);
  spmm::CsrMatrix<float> af;
  af.rows = af.cols = gb.n;
  af.row_ptr = gb.row_ptr;
  af.col_idx = gb.col_idx;
  af.values.assign(gb.col_idx.size(), 0.5f);
  spmm::BenchReport br = spmm::bench(af, 32, 3);
  CHECK(br.exec_ms > 0 && br.baseline_ms > 0 && br.reps == 3);
  // predict consumes the parts it is given: core_subgraphs' parts == regrow's parts with boundaries cut off
  auto cut = regrow(gb, pa);
  for (auto& p : cut) {
    const std::uint32_t nc = p.num_core();
    std::vector<std::pair<std::uint32_t, std::uint32_t>> keep;
    for (auto& e : p.edges)
      if (e.first < nc && e.second < nc) keep.push_back(e);
    p.edges = keep;
    p.boundary_nodes.clear();
    p.local_to_global.resize(nc);
  }
  CHECK(predict(m, gb, cut).labels == predict(m, gb, core).labels);
  std::uint64_t cross = 0;
  for (const auto& [u, v] : gb.fwd_edges) cross += pa.part_of[u] != pa.part_of[v];
  CHECK(edge_cut(gb, pa) == cross && crossing_fraction(gb, pa) == static_cast<double>(cross) / gb.fwd_edges.size());
  TrainStats ts;
  TrainConfig tc;
  tc.epochs = 10;
  Model tm = train(g, tc, &ts);
  CHECK(ts.loss.size() == 10 && ts.loss.back() < ts.loss.front() && tm.layers.size() == 4);
  PartitionAssignment ml = partition_multilevel(gb, 8, 7);  // k >= 8: the reference livelocks here
  std::vector<std::uint32_t> sizes(8, 0);
  for (std::uint32_t p : ml.part_of) ++sizes[p];
  const std::uint32_t cap = static_cast<std::uint32_t>(std::ceil(1.05 * gb.n / 8));
  CHECK(ml.k == 8 && *std::min_element(sizes.begin(), sizes.end()) >= 1 && *std::max_element(sizes.begin(), sizes.end()) <= cap);
  std::printf("device checks ok (accuracy %.4f)\n", full.accuracy);
  return 0;
}
