// capi.cpp — the extern "C" boundary (include/groot.h) over the device path.
//
// Host-side pieces that are inherently sequential live here: the CSA
// multiplier generator (input source, src/circuitgen.cpp:66-133), the ASCII
// AIGER parser (src/aig.cpp:47-88), Glorot init (src/gnn.cpp:113-138) and the
// ASG1 model format (src/gnn.cpp:330-372). Everything on the data path —
// features, CSR, batch, partition, regrow, materialize, forward, classify —
// runs in the CUDA kernels of graph_build.cu / forward.cu.
#include <chrono>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <fstream>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "common.cuh"

namespace groot {

std::atomic<uint64_t> g_launches{0};
static thread_local std::string g_error;

// One session per device: every device has its own library
// stream and cached attributes; the calling thread's current device selects
// them, and the handle-taking entry points make the handle's device current.
static std::atomic<cudaStream_t> g_stream[kMaxDevices];
static std::atomic<int> g_sms[kMaxDevices];

int current_device() {
  int dev = 0;
  GROOT_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= kMaxDevices) fail(GROOT_ECUDA, "device ordinal beyond the library's session table");
  return dev;
}

cudaStream_t stream() { return g_stream[current_device()].load(std::memory_order_relaxed); }

int num_sms() {
  const int dev = current_device();
  int sms = g_sms[dev].load(std::memory_order_relaxed);
  if (!sms) {
    GROOT_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    g_sms[dev].store(sms, std::memory_order_relaxed);
  }
  return sms;
}

// graph_build.cu / forward.cu
groot_graph* encode(uint32_t, uint32_t, const uint32_t*, uint32_t, const uint32_t*, const uint8_t*);
groot_graph* batch(const groot_graph*, uint32_t);
groot_graph* graph_from_edges(uint32_t, const uint8_t*, const uint8_t*, uint64_t, const uint32_t*);
groot_graph* graph_from_host(uint32_t, const uint64_t*, const uint32_t*, const uint8_t*, const uint8_t*, uint64_t,
                             const uint32_t*);
void graph_copy_out(const groot_graph*, uint64_t*, uint32_t*, uint8_t*, uint8_t*, uint32_t*, uint32_t*);
groot_assignment* topo_chunks(const groot_graph*, uint32_t);
groot_assignment* partition_lp(const groot_graph*, uint32_t, uint64_t, uint32_t, uint32_t*, uint64_t*);
groot_assignment* assignment_from_host(uint32_t, const uint32_t*);
groot_assignment* load_assignment(const char*, uint32_t);
uint64_t edge_cut(const groot_graph*, const groot_assignment*);
groot_parts* regrow(const groot_graph*, const groot_assignment*, int);
groot_graph* materialize(const groot_graph*, const groot_parts*, uint32_t);
groot_parts* parts_from_host(uint32_t, uint32_t, const uint64_t*, const uint32_t*, const uint64_t*, const uint32_t*,
                             const uint64_t*, const uint32_t*);
groot_graph* union_of_parts(const groot_graph*, const groot_parts*, std::vector<uint64_t>&,
                            const std::vector<uint32_t>*);
void scatter_core_labels(const groot_parts*, const std::vector<uint64_t>&, const uint8_t*, uint8_t*);
void forward_device(const groot_model*, groot_graph*, uint8_t*, float*, unsigned long long*);
void layer_device(const groot_model*, groot_graph*, uint32_t, const float*, float*, uint8_t*, float*, uint32_t, uint32_t,
                  bool, bool keyed_in = false);
void forward_classify_to_host(const groot_model*, groot_graph*, uint8_t*, unsigned long long*, uint32_t, uint32_t,
                              uint32_t, uint8_t*);
void layer_prepare(const groot_model*, groot_graph*);
groot_graph* batch_padded(const groot_graph*, uint32_t, uint32_t);
bool replicate_forward_plan(groot_graph*, groot_graph*, uint32_t, uint32_t);
void forward_naive_device(const groot_model*, groot_graph*, uint8_t*, float*, unsigned long long*);
void spmm_mean_device(groot_graph*, const float*, uint32_t, float*);
void spmm_csr_device(uint32_t, const uint32_t*, const uint32_t*, const float*, const float*, uint32_t, float*, uint32_t);
void model_upload(groot_model*);
void classify_rows(groot_graph*, uint32_t);
uint32_t hd_threshold();
void confusion_device(uint32_t, const uint8_t*, const uint8_t*, unsigned long long*);
void spmm_csr_device_f64(uint32_t, const uint32_t*, const uint32_t*, const double*, const double*, uint32_t, double*,
                         uint32_t);
void graph_prepare(groot_graph*);
void graph_release_context(groot_graph*);

// ---------------------------------------------------------------------------
// CSA multiplier generator (src/circuitgen.cpp:13-133). Nodes are created in
// the reference's order so every downstream array is bit-identical.
// ---------------------------------------------------------------------------
namespace {

enum : uint8_t { kPo = 0, kMaj = 1, kXor = 2, kAnd = 3, kPi = 4 };
constexpr uint32_t kNone = 0xFFFFFFFFu;  // "no literal" in a column slot

struct Csa {
  uint32_t w;
  uint32_t inputs;
  std::vector<uint32_t> ands;    // (left, right) literal pairs
  std::vector<uint8_t> labels;   // const + PIs + ANDs (+ POs at the end)
  std::vector<uint32_t> outs;
  // GroundTruth::supports (src/circuitgen.cpp:30-32, 50-62): root node, arity,
  // 3 support literals (the third unused for a half adder)
  std::vector<uint32_t> sup;

  explicit Csa(uint32_t width) : w(width), inputs(2 * width) {
    labels.assign(1 + inputs, kAnd);
    std::fill(labels.begin() + 1, labels.end(), kPi);
  }
  uint32_t node(uint32_t l, uint32_t r, uint8_t cls) {
    const uint32_t v = 1 + inputs + static_cast<uint32_t>(ands.size() >> 1);
    ands.push_back(l);
    ands.push_back(r);
    labels.push_back(cls);
    return v << 1;
  }
  // Column reduction: 1 input passes, 2 -> half adder, 3 -> full adder.
  // Returns sum; carry written to *carry (kNone when none).
  uint32_t reduce(const uint32_t* in, int cnt, uint32_t* carry) {
    if (cnt == 1) { *carry = kNone; return in[0]; }
    const uint32_t a = in[0], b = in[1];
    if (cnt == 2) {  // gen_half_adder
      const uint32_t c = node(a, b, kMaj);
      const uint32_t nr = node(a ^ 1, b ^ 1, kAnd);
      *carry = c;
      const uint32_t sum = node(c ^ 1, nr ^ 1, kXor);
      sup.insert(sup.end(), {sum >> 1, 2u, a, b, 0u, c >> 1, 2u, a, b, 0u});
      return sum;
    }
    const uint32_t cin = in[2];  // gen_full_adder
    const uint32_t c1 = node(a, b, kAnd);
    const uint32_t n1 = node(a ^ 1, b ^ 1, kAnd);
    const uint32_t x1 = node(c1 ^ 1, n1 ^ 1, kAnd);
    const uint32_t c2 = node(x1, cin, kAnd);
    const uint32_t n2 = node(x1 ^ 1, cin ^ 1, kAnd);
    const uint32_t s = node(c2 ^ 1, n2 ^ 1, kXor);
    const uint32_t mj = node(c1 ^ 1, c2 ^ 1, kMaj);
    *carry = mj ^ 1;
    sup.insert(sup.end(), {s >> 1, 3u, a, b, cin, mj >> 1, 3u, a, b, cin});
    return s;
  }
  void build() {
    auto pp = [&](uint32_t i, uint32_t j) { return node(2 * (i + 1), 2 * (w + j + 1), kAnd); };
    std::vector<uint32_t> sums(2 * w, kNone), carries(2 * w, kNone), m(2 * w, 0);
    m[0] = pp(0, 0);
    for (uint32_t j = 1; j < w; ++j) sums[j] = pp(0, j);
    std::vector<uint32_t> ns(2 * w), nc(2 * w);
    for (uint32_t i = 1; i < w; ++i) {
      std::fill(ns.begin(), ns.end(), kNone);
      std::fill(nc.begin(), nc.end(), kNone);
      for (uint32_t j = 0; j < w; ++j) {
        const uint32_t c = i + j;
        uint32_t in[3];
        int cnt = 0;
        if (sums[c] != kNone) in[cnt++] = sums[c];
        in[cnt++] = pp(i, j);
        if (carries[c] != kNone) in[cnt++] = carries[c];
        uint32_t carry;
        const uint32_t s = reduce(in, cnt, &carry);
        (j == 0 ? m[i] : ns[c]) = s;
        if (carry != kNone) nc[c + 1] = carry;
      }
      sums.swap(ns);
      carries.swap(nc);
    }
    uint32_t ripple = kNone;
    for (uint32_t c = w; c < 2 * w; ++c) {
      uint32_t in[3];
      int cnt = 0;
      if (sums[c] != kNone) in[cnt++] = sums[c];
      if (carries[c] != kNone) in[cnt++] = carries[c];
      if (ripple != kNone) in[cnt++] = ripple;
      if (cnt == 0) fail(GROOT_ERUNTIME, "gen_csa_multiplier: empty column");
      m[c] = reduce(in, cnt, &ripple);
    }
    outs = m;
    labels.insert(labels.end(), outs.size(), kPo);
  }
};

// Closed-form sizes: w^2 partial products; rows 1..w-1 reduce w columns each
// (column j=0 of row i and the top column are half adders when the carry or
// sum slot is empty). Counting by construction keeps it exact.
void csa_counts(uint32_t w, uint32_t* na) {
  Csa c(w);
  c.build();
  *na = static_cast<uint32_t>(c.ands.size() / 2);
}

// ---------------------------------------------------------------------------
// Radix-4 Booth multiplier generator (BASELINE config 3; the reference has no
// Booth generator, SPEC.md:18,163 — GROOT's paper evaluates Booth AIGs from ABC,
// PAPER.md:297). Unsigned w x w -> 2w bits, inputs a = PIs 1..w, b = w+1..2w
// (the CSA generator's order). Structure:
//   * Booth encoder per digit i = 0..floor(w/2) over (b[2i+1], b[2i], b[2i-1])
//     (b[-1] = b[w] = b[w+1] = 0): one = b[2i] ^ b[2i-1],
//     two = b[2i+1] ? ~b[2i] & ~b[2i-1] : b[2i] & b[2i-1], neg = b[2i+1];
//   * selector per partial-product bit j = 0..w: pp = ((a[j] & one) |
//     (a[j-1] & two)) ^ neg;
//   * row i contributes pp bits at columns 2i+j, its two's-complement +1 (neg)
//     at column 2i and ~sign at column 2i+w+1; the sign extensions are folded
//     into one constant, -sum_i 2^(2i+w+1) mod 2^(2w), added as constant-true
//     bits (sign-extension prevention);
//   * Wallace-style column compression (full adders on bit triples, half
//     adders on a leftover pair when a column still holds more than two bits),
//     then a ripple-carry adder over the final two rows.
// Full/half adders are the reference's gen_full_adder / gen_half_adder (same
// 7 / 3 AND gates, XOR and MAJ roots labelled as in src/circuitgen.cpp:44-64);
// the encoder and selector logic is labelled AND. Node creation folds
// constants (an AND with a constant input or with its own complement is not
// materialised), so the AIG has no constant fanins.
// ---------------------------------------------------------------------------
struct Booth {
  uint32_t w;
  uint32_t inputs;
  std::vector<uint32_t> ands;
  std::vector<uint8_t> labels;
  std::vector<uint32_t> outs;

  explicit Booth(uint32_t width) : w(width), inputs(2 * width) {
    labels.assign(1 + inputs, kAnd);
    std::fill(labels.begin() + 1, labels.end(), kPi);
  }
  uint32_t node(uint32_t l, uint32_t r, uint8_t cls) {
    if (l == 0 || r == 0 || l == (r ^ 1)) return 0;  // constant false
    if (l == 1) return r;
    if (r == 1 || l == r) return l;
    const uint32_t v = 1 + inputs + static_cast<uint32_t>(ands.size() >> 1);
    ands.push_back(l);
    ands.push_back(r);
    labels.push_back(cls);
    return v << 1;
  }
  uint32_t or2(uint32_t x, uint32_t y) { return node(x ^ 1, y ^ 1, kAnd) ^ 1; }
  uint32_t xor2(uint32_t x, uint32_t y) {
    const uint32_t c = node(x, y, kAnd), n = node(x ^ 1, y ^ 1, kAnd);
    return node(c ^ 1, n ^ 1, kAnd);
  }
  uint32_t a(int64_t j) const { return (j < 0 || j >= static_cast<int64_t>(w)) ? 0u : 2u * static_cast<uint32_t>(j + 1); }
  uint32_t b(int64_t j) const { return (j < 0 || j >= static_cast<int64_t>(w)) ? 0u : 2u * static_cast<uint32_t>(w + j + 1); }
  // gen_half_adder / gen_full_adder (src/circuitgen.cpp:44-64)
  void half(uint32_t x, uint32_t y, uint32_t* s, uint32_t* c) {
    *c = node(x, y, kMaj);
    const uint32_t nr = node(x ^ 1, y ^ 1, kAnd);
    *s = node(*c ^ 1, nr ^ 1, kXor);
  }
  void full(uint32_t x, uint32_t y, uint32_t cin, uint32_t* s, uint32_t* c) {
    const uint32_t c1 = node(x, y, kAnd);
    const uint32_t n1 = node(x ^ 1, y ^ 1, kAnd);
    const uint32_t x1 = node(c1 ^ 1, n1 ^ 1, kAnd);
    const uint32_t c2 = node(x1, cin, kAnd);
    const uint32_t n2 = node(x1 ^ 1, cin ^ 1, kAnd);
    *s = node(c2 ^ 1, n2 ^ 1, kXor);
    *c = node(c1 ^ 1, c2 ^ 1, kMaj) ^ 1;
  }
  void build() {
    const uint32_t W = 2 * w;
    std::vector<std::vector<uint32_t>> col(W);
    auto put = [&](uint64_t c, uint32_t lit) {
      if (c < W && lit != 0) col[c].push_back(lit);
    };
    const uint32_t digits = w / 2 + 1;
    std::vector<uint64_t> konst(W, 0);  // -sum_i 2^(2i+w+1) mod 2^W, as bits
    {
      std::vector<uint32_t> acc(W + 1, 0);  // subtract each term from 0 in binary
      for (uint32_t i = 0; i < digits; ++i) {
        const uint64_t p = 2ull * i + w + 1;
        if (p >= W) continue;
        // acc -= 2^p  (mod 2^W): borrow propagation
        uint64_t q = p;
        while (q < W) {
          if (acc[q]) { acc[q] = 0; break; }
          acc[q] = 1;
          ++q;
        }
      }
      for (uint32_t c = 0; c < W; ++c) konst[c] = acc[c];
    }
    for (uint32_t i = 0; i < digits; ++i) {
      const int64_t k = 2 * static_cast<int64_t>(i);
      const uint32_t b0 = b(k - 1), b1 = b(k), b2 = b(k + 1);
      const uint32_t one = xor2(b1, b0);
      const uint32_t two = or2(node(b2, node(b1 ^ 1, b0 ^ 1, kAnd), kAnd), node(b2 ^ 1, node(b1, b0, kAnd), kAnd));
      const uint32_t neg = b2;
      for (uint32_t j = 0; j <= w; ++j) {
        const uint32_t sel = or2(node(a(j), one, kAnd), node(a(static_cast<int64_t>(j) - 1), two, kAnd));
        put(static_cast<uint64_t>(k) + j, xor2(sel, neg));
      }
      put(static_cast<uint64_t>(k), neg);
      put(static_cast<uint64_t>(k) + w + 1, neg ^ 1);
    }
    for (uint32_t c = 0; c < W; ++c)
      if (konst[c]) col[c].push_back(1);
    // constant-true bits: fold pairs (1 + 1 = carry 1, sum 0) so at most one remains per column
    for (uint32_t c = 0; c < W; ++c) {
      uint32_t ones = 0;
      std::vector<uint32_t> keep;
      for (uint32_t l : col[c]) {
        if (l == 1) ++ones;
        else keep.push_back(l);
      }
      col[c] = keep;
      if (ones & 1) col[c].push_back(1);
      if (ones >> 1 && c + 1 < W)
        for (uint32_t t = 0; t < (ones >> 1); ++t) col[c + 1].push_back(1);
    }
    // Wallace layers
    while (true) {
      bool done = true;
      for (uint32_t c = 0; c < W; ++c) done &= col[c].size() <= 2;
      if (done) break;
      std::vector<std::vector<uint32_t>> nxt(W);
      for (uint32_t c = 0; c < W; ++c) {
        const std::vector<uint32_t>& v = col[c];
        size_t i = 0;
        for (; i + 3 <= v.size(); i += 3) {
          uint32_t sm, cy;
          full(v[i], v[i + 1], v[i + 2], &sm, &cy);
          nxt[c].push_back(sm);
          if (c + 1 < W) nxt[c + 1].push_back(cy);
        }
        const size_t left = v.size() - i;
        if (left == 2 && v.size() > 3) {
          uint32_t sm, cy;
          half(v[i], v[i + 1], &sm, &cy);
          nxt[c].push_back(sm);
          if (c + 1 < W) nxt[c + 1].push_back(cy);
        } else {
          for (; i < v.size(); ++i) nxt[c].push_back(v[i]);
        }
      }
      col.swap(nxt);
    }
    // ripple-carry adder over the last two rows
    outs.assign(W, 0);
    uint32_t carry = 0;
    for (uint32_t c = 0; c < W; ++c) {
      std::vector<uint32_t> v = col[c];
      if (carry) v.push_back(carry);
      carry = 0;
      if (v.empty()) { outs[c] = 0; continue; }
      if (v.size() == 1) { outs[c] = v[0]; continue; }
      uint32_t sm, cy;
      if (v.size() == 2) half(v[0], v[1], &sm, &cy);
      else full(v[0], v[1], v[2], &sm, &cy);
      outs[c] = sm;
      carry = cy;
    }
    labels.insert(labels.end(), outs.size(), kPo);
  }
};

// ---------------------------------------------------------------------------
// ASCII AIGER (src/aig.cpp:47-88) — same validation order and messages.
// ---------------------------------------------------------------------------
struct ParsedAig {
  uint32_t inputs = 0;
  std::vector<uint32_t> ands, outs;
};

ParsedAig parse_aiger_text(const char* text, size_t len) {
  std::istringstream in(std::string(text, len));
  auto num = [&](const char* what) {
    uint64_t v;
    if (!(in >> v)) fail(GROOT_ERUNTIME, std::string("AIGER: missing or bad ") + what);
    return v;
  };
  std::string magic;
  if (!(in >> magic)) fail(GROOT_ERUNTIME, "AIGER: empty input");
  if (magic != "aag") fail(GROOT_ERUNTIME, "AIGER: expected ASCII header 'aag', got '" + magic + "'");
  const uint64_t M = num("M"), I = num("I"), L = num("L"), O = num("O"), A = num("A");
  if (L != 0) fail(GROOT_ERUNTIME, "AIGER: latches unsupported (sequential circuit)");
  if (M != I + A) fail(GROOT_ERUNTIME, "AIGER: non-contiguous variable numbering (M != I + A)");
  if (1 + M + O >= 0xFFFFFFFFull) fail(GROOT_ERUNTIME, "AIGER: too many nodes");
  ParsedAig p;
  p.inputs = static_cast<uint32_t>(I);
  for (uint64_t k = 0; k < I; ++k)
    if (num("input literal") != 2 * (k + 1)) fail(GROOT_ERUNTIME, "AIGER: inputs must be the literals 2..2I in order");
  auto lit = [&](uint64_t l, const char* what) {
    if (l > 2 * M + 1) fail(GROOT_ERUNTIME, std::string("AIGER: ") + what + " literal out of range");
    return static_cast<uint32_t>(l);
  };
  std::vector<uint64_t> olits(O);
  for (uint64_t k = 0; k < O; ++k) olits[k] = num("output literal");
  p.ands.reserve(2 * A);
  for (uint64_t k = 0; k < A; ++k) {
    const uint64_t lhs = num("AND lhs");
    if (lhs != 2 * (I + 1 + k)) fail(GROOT_ERUNTIME, "AIGER: AND definitions must appear in ascending index order");
    const uint32_t l = lit(num("AND rhs0"), "AND rhs0");
    const uint32_t r = lit(num("AND rhs1"), "AND rhs1");
    const uint64_t own = lhs >> 1;
    if ((l >> 1) >= own || (r >> 1) >= own) fail(GROOT_ERUNTIME, "AIGER: fanin index >= own index (cycle)");
    p.ands.push_back(l);
    p.ands.push_back(r);
  }
  for (uint64_t v : olits) p.outs.push_back(lit(v, "output"));
  return p;
}

// ---------------------------------------------------------------------------
// Model: init_model (src/gnn.cpp:113-138), ASG1 I/O (src/gnn.cpp:330-372)
// ---------------------------------------------------------------------------
uint64_t param_count(uint32_t depth, uint32_t in_dim, uint32_t hidden, uint32_t classes) {
  uint64_t c = 0;
  uint32_t in = in_dim;
  for (uint32_t l = 0; l < depth; ++l) {
    c += 2ull * in * hidden + hidden;
    in = hidden;
  }
  return c + static_cast<uint64_t>(in) * classes + classes;
}

void init_params(uint64_t seed, uint32_t in_dim, uint32_t hidden, uint32_t classes, uint32_t depth, double* out) {
  if (depth < 1) fail(GROOT_EINVAL, "init_model: depth must be >= 1");
  std::mt19937_64 rng(seed);
  double* q = out;
  auto glorot = [&](uint32_t rows, uint32_t cols) {
    const double lim = std::sqrt(6.0 / (rows + cols));
    std::uniform_real_distribution<double> dist(-lim, lim);
    for (uint64_t i = 0; i < static_cast<uint64_t>(rows) * cols; ++i) *q++ = dist(rng);
  };
  uint32_t in = in_dim;
  for (uint32_t l = 0; l < depth; ++l) {
    glorot(in, hidden);
    glorot(in, hidden);
    for (uint32_t o = 0; o < hidden; ++o) *q++ = 0.0;
    in = hidden;
  }
  glorot(in, classes);
  for (uint32_t o = 0; o < classes; ++o) *q++ = 0.0;
}

groot_model* model_create(uint32_t depth, uint32_t in_dim, uint32_t hidden, uint32_t classes, const double* prm) {
  if (depth < 1 || depth > 64) fail(GROOT_EINVAL, "model: depth must be in 1..64");
  if (in_dim != 4 || hidden != 32) fail(GROOT_EINVAL, "model: the device path supports in_dim 4 and hidden 32");
  if (classes < 1 || classes > 8) fail(GROOT_EINVAL, "model: classes must be in 1..8");
  auto* m = new groot_model;
  m->device = current_device();
  m->depth = depth;
  m->in_dim = in_dim;
  m->hidden = hidden;
  m->classes = classes;
  m->params.assign(prm, prm + param_count(depth, in_dim, hidden, classes));
  try {
    model_upload(m);
  } catch (...) {
    delete m;
    throw;
  }
  return m;
}

}  // namespace

void init_model_params(uint64_t seed, uint32_t in_dim, uint32_t hidden, uint32_t classes, uint32_t depth, double* prm) {
  init_params(seed, in_dim, hidden, classes, depth, prm);
}
void train_device(const groot_graph*, uint32_t, uint32_t, uint32_t, uint32_t, uint32_t, double, uint64_t, double, double,
                  double, const double*, double*, double*, double*);
double loss_and_grads_device(const groot_graph*, uint32_t, uint32_t, uint32_t, uint32_t, const double*, double*);

void set_last_error(const std::string& msg) { g_error = msg; }

static void need(const void* p, const char* what) {
  if (!p) fail(GROOT_EINVAL, std::string(what) + ": null argument");
}

// spmm::execute over a host CsrMatrix<T> (validate() checks, inc/spmm.hpp:25-36)
template <class T, class Dev>
static void spmm_csr_host(uint32_t rows, uint32_t cols, const uint64_t* rp, const uint32_t* col, const T* vals,
                          const T* dense, uint32_t f, uint32_t hd_threshold, T* out, Dev device_fn) {
  need(rp, "groot_spmm_csr");
  const uint64_t nnz = rp[rows];
  if (nnz >= 0xFFFFFFFFull) fail(GROOT_EINVAL, "spmm: nnz must be < 2^32");
  std::vector<uint32_t> rp32(rows + 1ull);
  for (uint32_t r = 0; r <= rows; ++r) {
    if (r && rp[r] < rp[r - 1]) fail(GROOT_EINVAL, "CsrMatrix: row_ptr not monotone");
    rp32[r] = static_cast<uint32_t>(rp[r]);
  }
  for (uint64_t q = 0; q < nnz; ++q)
    if (col[q] >= cols) fail(GROOT_EINVAL, "CsrMatrix: column index out of range");
  DevBuf<uint32_t> drp(rows + 1ull), dcol(nnz);
  DevBuf<T> dval(nnz), dd(static_cast<size_t>(cols) * f), dout(static_cast<size_t>(rows) * f);
  drp.upload(rp32.data(), rows + 1ull);
  dcol.upload(col, nnz);
  if (vals) dval.upload(vals, nnz);
  dd.upload(dense, static_cast<size_t>(cols) * f);
  device_fn(rows, drp.p, dcol.p, vals ? dval.p : nullptr, dd.p, f, dout.p, hd_threshold);
  dout.download(out, static_cast<size_t>(rows) * f);
  stream_sync();
}

static void same_device(const groot_model* m, const groot_graph* g) {
  if (m->device != g->device) fail(GROOT_EINVAL, "model and graph live on different devices");
}

}  // namespace groot

using namespace groot;

extern "C" {

const char* groot_last_error(void) { return g_error.c_str(); }
int groot_version(void) { return 1; }

int groot_set_stream(void* s) {
  return guarded([&] { g_stream[current_device()].store(static_cast<cudaStream_t>(s)); });
}
void* groot_get_stream(void) {
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= kMaxDevices) return nullptr;
  return g_stream[dev].load();
}
int groot_device_synchronize(void) {
  return guarded([] { GROOT_CUDA(cudaStreamSynchronize(stream())); });
}
uint64_t groot_kernel_launches(void) { return g_launches.load(); }
void groot_reset_kernel_launches(void) { g_launches.store(0); }

// ---- AIG sources ------------------------------------------------------------
int groot_csa_sizes(uint32_t width, uint32_t* ni, uint32_t* na, uint32_t* no) {
  return guarded([&] {
    if (width < 2) fail(GROOT_EINVAL, "gen_csa_multiplier: width must be >= 2");
    need(ni, "groot_csa_sizes");
    csa_counts(width, na);
    *ni = 2 * width;
    *no = 2 * width;
  });
}

int groot_gen_csa(uint32_t width, uint32_t* and_lits, uint32_t* out_lits, uint8_t* labels) {
  return guarded([&] {
    if (width < 2) fail(GROOT_EINVAL, "gen_csa_multiplier: width must be >= 2");
    Csa c(width);
    c.build();
    if (and_lits) std::copy(c.ands.begin(), c.ands.end(), and_lits);
    if (out_lits) std::copy(c.outs.begin(), c.outs.end(), out_lits);
    if (labels) std::copy(c.labels.begin(), c.labels.end(), labels);
  });
}

int groot_csa_supports(uint32_t width, uint32_t* count, uint32_t* records) {
  return guarded([&] {
    if (width < 2) fail(GROOT_EINVAL, "gen_csa_multiplier: width must be >= 2");
    need(count, "groot_csa_supports");
    Csa c(width);
    c.build();
    *count = static_cast<uint32_t>(c.sup.size() / 5);
    if (records) std::copy(c.sup.begin(), c.sup.end(), records);
  });
}

int groot_booth_sizes(uint32_t width, uint32_t* ni, uint32_t* na, uint32_t* no) {
  return guarded([&] {
    if (width < 2) fail(GROOT_EINVAL, "gen_booth_multiplier: width must be >= 2");
    need(ni, "groot_booth_sizes");
    Booth bt(width);
    bt.build();
    *ni = 2 * width;
    *na = static_cast<uint32_t>(bt.ands.size() / 2);
    *no = 2 * width;
  });
}

int groot_gen_booth(uint32_t width, uint32_t* and_lits, uint32_t* out_lits, uint8_t* labels) {
  return guarded([&] {
    if (width < 2) fail(GROOT_EINVAL, "gen_booth_multiplier: width must be >= 2");
    Booth bt(width);
    bt.build();
    if (and_lits) std::copy(bt.ands.begin(), bt.ands.end(), and_lits);
    if (out_lits) std::copy(bt.outs.begin(), bt.outs.end(), out_lits);
    if (labels) std::copy(bt.labels.begin(), bt.labels.end(), labels);
  });
}

int groot_aiger_sizes(const char* text, size_t len, uint32_t* ni, uint32_t* na, uint32_t* no) {
  return guarded([&] {
    need(text, "groot_aiger_sizes");
    const ParsedAig p = parse_aiger_text(text, len);
    *ni = p.inputs;
    *na = static_cast<uint32_t>(p.ands.size() / 2);
    *no = static_cast<uint32_t>(p.outs.size());
  });
}

int groot_aiger_fill(const char* text, size_t len, uint32_t* and_lits, uint32_t* out_lits) {
  return guarded([&] {
    need(text, "groot_aiger_fill");
    const ParsedAig p = parse_aiger_text(text, len);
    if (and_lits) std::copy(p.ands.begin(), p.ands.end(), and_lits);
    if (out_lits) std::copy(p.outs.begin(), p.outs.end(), out_lits);
  });
}

// ---- graphs -----------------------------------------------------------------
int groot_encode(uint32_t ni, uint32_t na, const uint32_t* ands, uint32_t no, const uint32_t* outs,
                 const uint8_t* labels, groot_graph** out) {
  return guarded([&] {
    need(out, "groot_encode");
    if (na) need(ands, "groot_encode");
    if (no) need(outs, "groot_encode");
    *out = encode(ni, na, ands, no, outs, labels);
  });
}

int groot_batch(const groot_graph* g, uint32_t copies, groot_graph** out) {
  return guarded([&] {
    need(g, "groot_batch");
    DeviceScope ds_g(g->device);
    *out = batch(g, copies);
  });
}

int groot_graph_from_host(uint32_t n, const uint64_t* rp, const uint32_t* col, const uint8_t* feat,
                          const uint8_t* lab, uint64_t ne, const uint32_t* edges, groot_graph** out) {
  return guarded([&] {
    need(rp, "groot_graph_from_host");
    if (rp[n]) need(col, "groot_graph_from_host");
    *out = graph_from_host(n, rp, col, feat, lab, ne, edges);
  });
}

int groot_graph_from_edges(uint32_t n, const uint8_t* feat, const uint8_t* lab, uint64_t ne, const uint32_t* edges,
                           groot_graph** out) {
  return guarded([&] {
    need(out, "groot_graph_from_edges");
    if (ne) need(edges, "groot_graph_from_edges");
    *out = graph_from_edges(n, feat, lab, ne, edges);
  });
}

int groot_graph_sizes(const groot_graph* g, uint32_t* n, uint64_t* nnz, uint64_t* ne) {
  return guarded([&] {
    need(g, "groot_graph_sizes");
    DeviceScope ds_g(g->device);
    if (n) *n = g->n;
    if (nnz) *nnz = g->nnz;
    if (ne) *ne = g->ne;
  });
}

int groot_graph_copy_out(const groot_graph* g, uint64_t* rp, uint32_t* col, uint8_t* feat, uint8_t* lab,
                         uint32_t* deg, uint32_t* edges) {
  return guarded([&] {
    need(g, "groot_graph_copy_out");
    DeviceScope ds_g(g->device);
    graph_copy_out(g, rp, col, feat, lab, deg, edges);
  });
}

int groot_graph_device_ptrs(const groot_graph* g, const uint32_t** rp, const uint32_t** col, const uint8_t** feat,
                            const uint8_t** lab, const uint32_t** edges) {
  return guarded([&] {
    need(g, "groot_graph_device_ptrs");
    DeviceScope ds_g(g->device);
    if (rp) *rp = g->rp.p;
    if (col) *col = g->col.p;
    if (feat) *feat = g->feat.p;
    if (lab) *lab = g->labels.p;
    if (edges) *edges = g->edges.p;
  });
}

void groot_graph_free(groot_graph* g) { delete g; }

// ---- partition ----------------------------------------------------------------
int groot_partition_topo_chunks(const groot_graph* g, uint32_t k, groot_assignment** out) {
  return guarded([&] {
    need(g, "groot_partition_topo_chunks");
    DeviceScope ds_g(g->device);
    *out = topo_chunks(g, k);
  });
}

int groot_load_assignment(const char* path, uint32_t n, groot_assignment** out) {
  return guarded([&] {
    need(path, "groot_load_assignment");
    *out = load_assignment(path, n);
  });
}

int groot_assignment_from_host(uint32_t n, const uint32_t* part_of, groot_assignment** out) {
  return guarded([&] {
    need(part_of, "groot_assignment_from_host");
    *out = assignment_from_host(n, part_of);
  });
}

int groot_assignment_info(const groot_assignment* a, uint32_t* n, uint32_t* k) {
  return guarded([&] {
    need(a, "groot_assignment_info");
    DeviceScope ds_a(a->device);
    if (n) *n = a->n;
    if (k) *k = a->k;
  });
}

int groot_assignment_copy_out(const groot_assignment* a, uint32_t* part_of) {
  return guarded([&] {
    need(a, "groot_assignment_copy_out");
    DeviceScope ds_a(a->device);
    a->part_of.download(part_of, a->n);
    stream_sync();
  });
}

int groot_partition_multilevel(const groot_graph* g, uint32_t k, uint64_t seed, groot_assignment** out,
                               uint32_t* rounds, uint64_t* moves) {
  return guarded([&] {
    need(g, "groot_partition_multilevel");
    DeviceScope ds_g(g->device);
    need(out, "groot_partition_multilevel");
    const char* e = std::getenv("GROOT_LP_ROUNDS");
    const uint32_t max_rounds = e ? static_cast<uint32_t>(std::strtoul(e, nullptr, 10)) : 32u;
    *out = partition_lp(g, k, seed, max_rounds, rounds, moves);
  });
}

void groot_assignment_free(groot_assignment* a) { delete a; }

int groot_crossing_fraction(const groot_graph* g, const groot_assignment* a, double* fraction) {
  return guarded([&] {
    need(g, "groot_crossing_fraction");
    DeviceScope ds_g(g->device);
    need(a, "groot_crossing_fraction");
    const uint64_t cut = edge_cut(g, a);
    *fraction = g->ne ? static_cast<double>(cut) / static_cast<double>(g->ne) : 0.0;
  });
}

int groot_edge_cut(const groot_graph* g, const groot_assignment* a, uint64_t* cut) {
  return guarded([&] {
    need(g, "groot_edge_cut");
    DeviceScope ds_g(g->device);
    need(a, "groot_edge_cut");
    *cut = edge_cut(g, a);
  });
}

// ---- regrow -----------------------------------------------------------------------
int groot_regrow(const groot_graph* g, const groot_assignment* a, int with_b, groot_parts** out) {
  return guarded([&] {
    need(g, "groot_regrow");
    DeviceScope ds_g(g->device);
    need(a, "groot_regrow");
    *out = regrow(g, a, with_b);
  });
}

int groot_parts_count(const groot_parts* p, uint32_t* k) {
  return guarded([&] {
    need(p, "groot_parts_count");
    DeviceScope ds_p(p->device);
    *k = p->k;
  });
}

int groot_parts_sizes(const groot_parts* p, uint32_t part, uint32_t* nc, uint32_t* nb, uint64_t* ne) {
  return guarded([&] {
    need(p, "groot_parts_sizes");
    DeviceScope ds_p(p->device);
    if (part >= p->k) fail(GROOT_EINVAL, "parts: index out of range");
    if (nc) *nc = static_cast<uint32_t>(p->core_off[part + 1] - p->core_off[part]);
    if (nb) *nb = static_cast<uint32_t>(p->bnd_off[part + 1] - p->bnd_off[part]);
    if (ne) *ne = p->edge_off[part + 1] - p->edge_off[part];
  });
}

int groot_parts_copy_out(const groot_parts* p, uint32_t part, uint32_t* core, uint32_t* bnd, uint32_t* edges) {
  return guarded([&] {
    need(p, "groot_parts_copy_out");
    DeviceScope ds_p(p->device);
    if (part >= p->k) fail(GROOT_EINVAL, "parts: index out of range");
    const uint64_t c0 = p->core_off[part], c1 = p->core_off[part + 1];
    const uint64_t b0 = p->bnd_off[part], b1 = p->bnd_off[part + 1];
    const uint64_t e0 = p->edge_off[part], e1 = p->edge_off[part + 1];
    if (core && c1 > c0)
      GROOT_CUDA(cudaMemcpyAsync(core, p->core.p + c0, (c1 - c0) * 4, cudaMemcpyDeviceToHost, stream()));
    if (bnd && b1 > b0)
      GROOT_CUDA(cudaMemcpyAsync(bnd, p->bnd.p + b0, (b1 - b0) * 4, cudaMemcpyDeviceToHost, stream()));
    if (edges && e1 > e0)
      GROOT_CUDA(cudaMemcpyAsync(edges, p->edges.p + 2 * e0, (e1 - e0) * 8, cudaMemcpyDeviceToHost, stream()));
    stream_sync();
  });
}

int groot_footprint_proxy(const groot_parts* p, uint32_t feature_cols, uint32_t hidden_dim, uint64_t* bytes) {
  return guarded([&] {
    need(p, "groot_footprint_proxy");
    DeviceScope ds_p(p->device);
    uint64_t best = 0;
    for (uint32_t q = 0; q < p->k; ++q) {
      const uint64_t size = (p->core_off[q + 1] - p->core_off[q]) + (p->bnd_off[q + 1] - p->bnd_off[q]);
      const uint64_t ne = p->edge_off[q + 1] - p->edge_off[q];
      best = std::max(best, size * (feature_cols + hidden_dim) * 4 + 2 * ne * 8);
    }
    *bytes = best;
  });
}

int groot_materialize(const groot_graph* g, const groot_parts* p, uint32_t part, groot_graph** out) {
  return guarded([&] {
    need(g, "groot_materialize");
    DeviceScope ds_g(g->device);
    need(p, "groot_materialize");
    *out = materialize(g, p, part);
  });
}

int groot_parts_from_host(uint32_t n, uint32_t k, const uint64_t* core_off, const uint32_t* core_nodes,
                          const uint64_t* bnd_off, const uint32_t* boundary_nodes, const uint64_t* edge_off,
                          const uint32_t* edges, groot_parts** out) {
  return guarded([&] {
    need(out, "groot_parts_from_host");
    *out = parts_from_host(n, k, core_off, core_nodes, bnd_off, boundary_nodes, edge_off, edges);
  });
}

void groot_parts_free(groot_parts* p) { delete p; }

// ---- model --------------------------------------------------------------------------
uint64_t groot_param_count(uint32_t depth, uint32_t in_dim, uint32_t hidden, uint32_t classes) {
  return param_count(depth, in_dim, hidden, classes);
}

int groot_init_params(uint64_t seed, uint32_t in_dim, uint32_t hidden, uint32_t classes, uint32_t depth,
                      double* params) {
  return guarded([&] {
    need(params, "groot_init_params");
    init_params(seed, in_dim, hidden, classes, depth, params);
  });
}

int groot_model_create(uint32_t depth, uint32_t in_dim, uint32_t hidden, uint32_t classes, const double* params,
                       groot_model** out) {
  return guarded([&] {
    need(params, "groot_model_create");
    *out = model_create(depth, in_dim, hidden, classes, params);
  });
}

int groot_model_load(const char* path, groot_model** out) {
  return guarded([&] {
    need(path, "groot_model_load");
    std::ifstream in(path, std::ios::binary);
    if (!in) fail(GROOT_ERUNTIME, std::string("cannot open model file: ") + path);
    char magic[4];
    in.read(magic, 4);
    if (!in || std::string(magic, 4) != "ASG1") fail(GROOT_ERUNTIME, "model file: bad magic or version");
    uint32_t hdr[4];
    in.read(reinterpret_cast<char*>(hdr), 16);
    if (!in || hdr[0] == 0 || hdr[0] > 64) fail(GROOT_ERUNTIME, "model file: bad header");
    std::vector<double> prm(param_count(hdr[0], hdr[1], hdr[2], hdr[3]));
    in.read(reinterpret_cast<char*>(prm.data()), static_cast<std::streamsize>(prm.size() * 8));
    if (!in) fail(GROOT_ERUNTIME, "model file: truncated");
    *out = model_create(hdr[0], hdr[1], hdr[2], hdr[3], prm.data());
  });
}

int groot_model_save(const groot_model* m, const char* path) {
  return guarded([&] {
    need(m, "groot_model_save");
    std::ofstream out(path, std::ios::binary);
    if (!out) fail(GROOT_ERUNTIME, std::string("cannot write model file: ") + path);
    out.write("ASG1", 4);
    const uint32_t hdr[4] = {m->depth, m->in_dim, m->hidden, m->classes};
    out.write(reinterpret_cast<const char*>(hdr), 16);
    out.write(reinterpret_cast<const char*>(m->params.data()), static_cast<std::streamsize>(m->params.size() * 8));
  });
}

int groot_model_info(const groot_model* m, uint32_t* depth, uint32_t* in_dim, uint32_t* hidden, uint32_t* classes) {
  return guarded([&] {
    need(m, "groot_model_info");
    if (depth) *depth = m->depth;
    if (in_dim) *in_dim = m->in_dim;
    if (hidden) *hidden = m->hidden;
    if (classes) *classes = m->classes;
  });
}

int groot_model_params(const groot_model* m, double* params) {
  return guarded([&] {
    need(m, "groot_model_params");
    std::copy(m->params.begin(), m->params.end(), params);
  });
}

void groot_model_free(groot_model* m) { delete m; }

// ---- training (src/gnn.cpp:180-255) --------------------------------------------------
int groot_train(const groot_graph* g, uint32_t depth, uint32_t in_dim, uint32_t hidden, uint32_t classes,
                uint32_t epochs, double learning_rate, uint64_t seed, double beta1, double beta2, double adam_eps,
                const double* init_params, double* params_out, double* loss_out, double* accuracy_out) {
  return guarded([&] {
    need(g, "groot_train");
    DeviceScope ds_g(g->device);
    need(params_out, "groot_train");
    train_device(g, depth, in_dim, hidden, classes, epochs, learning_rate, seed, beta1, beta2, adam_eps, init_params,
                 params_out, loss_out, accuracy_out);
  });
}

int groot_loss_and_grads(const groot_graph* g, uint32_t depth, uint32_t in_dim, uint32_t hidden, uint32_t classes,
                         const double* params, double* grads_out, double* loss) {
  return guarded([&] {
    need(g, "groot_loss_and_grads");
    DeviceScope ds_g(g->device);
    need(params, "groot_loss_and_grads");
    const double l = loss_and_grads_device(g, depth, in_dim, hidden, classes, params, grads_out);
    if (loss) *loss = l;
  });
}

// ---- forward / predict -------------------------------------------------------------
static void finish_confusion(const uint64_t* conf, uint32_t n, uint64_t* confusion, double* accuracy) {
  if (confusion) std::copy(conf, conf + 25, confusion);
  if (accuracy) {
    uint64_t hit = 0;
    for (int c = 0; c < 5; ++c) hit += conf[c * 5 + c];
    *accuracy = n ? static_cast<double>(hit) / static_cast<double>(n) : 0.0;
  }
}

int groot_forward(const groot_model* m, const groot_graph* g, float* logits_host) {
  return guarded([&] {
    need(m, "groot_forward");
    need(g, "groot_forward");
    DeviceScope ds_g(g->device);
    same_device(m, g);
    auto* gg = const_cast<groot_graph*>(g);
    DevBuf<uint8_t> cls(g->n);
    DevBuf<float> lg(static_cast<size_t>(g->n) * m->classes);
    forward_device(m, gg, cls.p, lg.p, nullptr);
    if (logits_host) lg.download(logits_host, static_cast<size_t>(g->n) * m->classes);
    stream_sync();
  });
}

// Debug/differential path: thread-per-row kernels (tests only).
int groot_debug_forward_naive(const groot_model* m, const groot_graph* g, float* logits_host, uint8_t* labels_host) {
  return guarded([&] {
    need(m, "groot_debug_forward_naive");
    need(g, "groot_debug_forward_naive");
    DeviceScope ds_g(g->device);
    same_device(m, g);
    auto* gg = const_cast<groot_graph*>(g);
    DevBuf<uint8_t> cls(g->n);
    DevBuf<float> lg(static_cast<size_t>(g->n) * m->classes);
    forward_naive_device(m, gg, cls.p, lg.p, nullptr);
    if (logits_host) lg.download(logits_host, static_cast<size_t>(g->n) * m->classes);
    if (labels_host) cls.download(labels_host, g->n);
    stream_sync();
  });
}

int groot_predict_full(const groot_model* m, const groot_graph* g, uint8_t* labels_host, uint64_t* confusion,
                       double* accuracy) {
  return guarded([&] {
    need(m, "groot_predict_full");
    need(g, "groot_predict_full");
    DeviceScope ds_g(g->device);
    same_device(m, g);
    auto* gg = const_cast<groot_graph*>(g);
    DevBuf<uint8_t> cls(g->n);
    DevBuf<unsigned long long> conf(25);
    conf.zero();
    forward_device(m, gg, cls.p, nullptr, conf.p);
    uint64_t h[25];
    conf.download(reinterpret_cast<unsigned long long*>(h), 25);
    if (labels_host) cls.download(labels_host, g->n);
    stream_sync();
    finish_confusion(h, g->n, confusion, accuracy);
  });
}

int groot_predict_full_dev(const groot_model* m, const groot_graph* g, uint8_t* labels_dev, float* logits_dev,
                           uint64_t* confusion_dev) {
  return guarded([&] {
    need(m, "groot_predict_full_dev");
    need(g, "groot_predict_full_dev");
    DeviceScope ds_g(g->device);
    same_device(m, g);
    need(labels_dev, "groot_predict_full_dev");
    forward_device(m, const_cast<groot_graph*>(g), labels_dev, logits_dev,
                   reinterpret_cast<unsigned long long*>(confusion_dev));
  });
}

int groot_layer_dev(const groot_model* m, const groot_graph* g, uint32_t layer, const float* hin_dev, float* hout_dev,
                    uint8_t* labels_dev, float* logits_dev) {
  return guarded([&] {
    need(m, "groot_layer_dev");
    need(g, "groot_layer_dev");
    DeviceScope ds_g(g->device);
    same_device(m, g);
    if (layer >= m->depth) fail(GROOT_EINVAL, "layer: index out of range");
    const bool last = layer + 1 == m->depth;
    if (layer > 0 && !hin_dev) fail(GROOT_EINVAL, "layer: input activations required for layer >= 1");
    if ((!last || m->depth == 1) && !hout_dev) fail(GROOT_EINVAL, "layer: output activations required");
    if (last && !labels_dev) fail(GROOT_EINVAL, "layer: class output required for the last layer");
    groot_graph* gg = const_cast<groot_graph*>(g);
    layer_prepare(m, gg);
    layer_device(m, gg, layer, hin_dev, hout_dev, labels_dev, logits_dev, 0, ~0u, true);
  });
}

int groot_predict(const groot_model* m, const groot_graph* g, const groot_parts* p, uint8_t* labels_host,
                  uint64_t* confusion, double* accuracy) {
  return guarded([&] {
    need(m, "groot_predict");
    need(g, "groot_predict");
    DeviceScope ds_g(g->device);
    same_device(m, g);
    need(p, "groot_predict");
    std::vector<uint64_t> node_off;
    groot_graph* u = union_of_parts(g, p, node_off, nullptr);
    try {
      DevBuf<uint8_t> cls(u->n), out(g->n);
      DevBuf<unsigned long long> dconf(25);
      out.zero();
      dconf.zero();
      if (u->n) forward_device(m, u, cls.p, nullptr, nullptr);
      scatter_core_labels(p, node_off, cls.p, out.p);
      confusion_device(g->n, out.p, g->labels.p, dconf.p);  // over all n nodes (src/gnn.cpp:265-276)
      uint64_t conf[25];
      dconf.download(reinterpret_cast<unsigned long long*>(conf), 25);
      if (labels_host) out.download(labels_host, g->n);
      stream_sync();
      finish_confusion(conf, g->n, confusion, accuracy);
    } catch (...) {
      delete u;
      throw;
    }
    delete u;
  });
}

int groot_predict_parts(const groot_model* m, const groot_graph* g, const groot_parts* p, const uint32_t* part_ids,
                        uint32_t count, uint8_t* labels_host) {
  return guarded([&] {
    need(m, "groot_predict_parts");
    need(g, "groot_predict_parts");
    DeviceScope ds_g(g->device);
    same_device(m, g);
    need(p, "groot_predict_parts");
    need(labels_host, "groot_predict_parts");
    std::vector<uint32_t> ids(part_ids, part_ids + count);
    std::vector<uint64_t> node_off;
    groot_graph* u = union_of_parts(g, p, node_off, &ids);
    try {
      DevBuf<uint8_t> cls(u->n), out(g->n);
      out.upload(labels_host, g->n);
      if (u->n) forward_device(m, u, cls.p, nullptr, nullptr);
      scatter_core_labels(p, node_off, cls.p, out.p);
      out.download(labels_host, g->n);
      stream_sync();
    } catch (...) {
      delete u;
      throw;
    }
    delete u;
  });
}

int groot_classify_aig(const groot_model* m, uint32_t ni, uint32_t na, const uint32_t* ands, uint32_t no,
                       const uint32_t* outs, const uint8_t* labels, uint32_t copies, uint8_t* labels_out,
                       uint64_t* confusion, double* accuracy) {
  return guarded([&] {
    need(m, "groot_classify_aig");
    static const bool host_timing = std::getenv("GROOT_HOST_TIMING") != nullptr;
    auto now = [] { return std::chrono::steady_clock::now(); };
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    const auto t0 = now();
    groot_graph* g1 = encode(ni, na, ands, no, outs, labels);
    groot_graph* g = g1;
    try {
      if (host_timing) stream_sync();
      const auto t1 = now();
      if (copies < 1) fail(GROOT_EINVAL, "batch: copy count must be >= 1");
      // Batch copies on tile-aligned row strides (padding rows in between), so the
      // row classifier and tile plan of one copy are replicated rather than
      // rebuilt over the whole batch; the classes are read back per copy in the
      // reference's numbering (node v of copy k = k*n1 + v).
      const uint32_t n1 = g1->n;
      uint32_t P = n1;
      if (copies > 1) {
        const uint32_t Pa = (n1 + 127u) / 128u * 128u;
        groot_graph* gp = batch_padded(g1, copies, Pa);
        static const bool periodic = std::getenv("GROOT_E2E_PERIODIC") == nullptr ||
                                     std::atoi(std::getenv("GROOT_E2E_PERIODIC")) != 0;  // experiment knob
        if (periodic && m->depth > 1 && replicate_forward_plan(g1, gp, copies, Pa)) {
          g = gp;
          P = Pa;
        } else {
          delete gp;
          g = batch(g1, copies);
        }
        delete g1;
        g1 = nullptr;
      }
      if (host_timing) stream_sync();
      const auto t2 = now();
      DevBuf<uint8_t> cls(g->n);
      DevBuf<unsigned long long> conf(25);
      conf.zero();
      forward_classify_to_host(m, g, cls.p, conf.p, copies, n1, P, labels_out);
      const auto t3 = now();
      uint64_t h[25];
      conf.download(reinterpret_cast<unsigned long long*>(h), 25);
      stream_sync();
      const auto t4 = now();
      if (host_timing)
        std::fprintf(stderr, "[classify_aig] encode %.2f ms, batch %.2f ms, forward (enqueue) %.2f ms, forward+download %.2f ms\n",
                     ms(t0, t1), ms(t1, t2), ms(t2, t3), ms(t3, t4));
      finish_confusion(h, n1 * copies, confusion, accuracy);
    } catch (...) {
      delete g1;
      if (g != g1) delete g;
      throw;
    }
    const auto t5 = now();
    if (g != g1) delete g;
    delete g1;
    if (host_timing) std::fprintf(stderr, "[classify_aig] total %.2f ms, release %.2f ms\n", ms(t0, now()), ms(t5, now()));
  });
}

// ---- SpMM ------------------------------------------------------------------------------
int groot_spmm_mean(const groot_graph* g, const float* dense, uint32_t f, float* out) {
  return guarded([&] {
    need(g, "groot_spmm_mean");
    DeviceScope ds_g(g->device);
    need(dense, "groot_spmm_mean");
    need(out, "groot_spmm_mean");
    if (f == 0) fail(GROOT_EINVAL, "spmm: f must be >= 1");
    DevBuf<float> d(static_cast<size_t>(g->n) * f), o(static_cast<size_t>(g->n) * f);
    d.upload(dense, static_cast<size_t>(g->n) * f);
    spmm_mean_device(const_cast<groot_graph*>(g), d.p, f, o.p);
    o.download(out, static_cast<size_t>(g->n) * f);
    stream_sync();
  });
}

int groot_spmm_mean_dev(const groot_graph* g, const float* dense_dev, uint32_t f, float* out_dev) {
  return guarded([&] {
    need(g, "groot_spmm_mean_dev");
    DeviceScope ds_g(g->device);
    if (f == 0) fail(GROOT_EINVAL, "spmm: f must be >= 1");
    spmm_mean_device(const_cast<groot_graph*>(g), dense_dev, f, out_dev);
  });
}

int groot_graph_prepare(const groot_graph* g) {
  return guarded([&] {
    need(g, "groot_graph_prepare");
    DeviceScope ds(g->device);
    graph_prepare(const_cast<groot_graph*>(g));
  });
}

int groot_graph_release_context(const groot_graph* g) {
  return guarded([&] {
    need(g, "groot_graph_release_context");
    DeviceScope ds(g->device);
    graph_release_context(const_cast<groot_graph*>(g));
  });
}

int groot_spmm_csr(uint32_t rows, uint32_t cols, const uint64_t* rp, const uint32_t* col, const float* vals,
                   const float* dense, uint32_t f, uint32_t hd_threshold, float* out) {
  return guarded([&] { spmm_csr_host(rows, cols, rp, col, vals, dense, f, hd_threshold, out, spmm_csr_device); });
}

int groot_spmm_csr_f64(uint32_t rows, uint32_t cols, const uint64_t* rp, const uint32_t* col, const double* vals,
                       const double* dense, uint32_t f, uint32_t hd_threshold, double* out) {
  return guarded([&] { spmm_csr_host(rows, cols, rp, col, vals, dense, f, hd_threshold, out, spmm_csr_device_f64); });
}

}  // extern "C"
