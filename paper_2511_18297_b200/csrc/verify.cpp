// verify.cpp — the consumer of the predicted classes: label-guided
// backward rewriting of a multiplier's output word polynomial.
//
// Reference: backward_rewrite / multiplier_spec_poly / truth_table_equiv
// (src/verify.cpp:220-418) over the multilinear BigInt polynomials of
// src/polynomial.cpp. The reference needs Boost.Multiprecision (absent here, so
// it cannot be compiled); this is a Boost-free restatement with its own
// arbitrary-precision integer. The algorithm is the reference's:
//   * the word polynomial sum_k 2^k out_k is rewritten from the last AND node
//     down to the inputs; each node still present is replaced by a model;
//   * a node labelled XOR (class 2) or MAJ (class 1) is replaced in one step by
//     an XOR2/XOR3 or MAJ/AND model over a 2- or 3-node support (the
//     generator's support when given, else the structural XOR2 / full-adder
//     shapes) -- but only after the cone's truth table over that support
//     confirms the model, so wrong labels cost time, never soundness;
//   * an XOR root and a MAJ root over the same support, both present only
//     linearly with coefficients c and 2c, collapse to c (a + b + c_in)
//     (fa_reduce, the x1 + 2 x2 rule) without any nonlinear term;
//   * every other node expands as the AND of its fan-ins;
//   * more than `monomial_cap` terms ends the run as inconclusive.
// The result is the residual word - spec (zero iff equivalent).
#include <algorithm>
#include <array>
#include <cstdint>
#include <cstring>
#include <map>
#include <optional>
#include <string>
#include <vector>

#include "common.cuh"

namespace groot {
namespace {

// ---------------------------------------------------------------------------
// Signed arbitrary-precision integer: sign + magnitude in 32-bit limbs
// (little-endian, no leading zero limbs; zero = empty, non-negative).
// ---------------------------------------------------------------------------
class BigInt {
 public:
  BigInt() = default;
  BigInt(int64_t v) {  // NOLINT(google-explicit-constructor)
    neg_ = v < 0;
    uint64_t m = neg_ ? 0ull - static_cast<uint64_t>(v) : static_cast<uint64_t>(v);
    while (m) {
      mag_.push_back(static_cast<uint32_t>(m));
      m >>= 32;
    }
  }
  static BigInt pow2(uint32_t e) {
    BigInt r;
    r.mag_.assign(e / 32 + 1, 0);
    r.mag_.back() = 1u << (e % 32);
    return r;
  }
  bool is_zero() const { return mag_.empty(); }
  bool negative() const { return neg_; }
  BigInt operator-() const {
    BigInt r = *this;
    if (!r.is_zero()) r.neg_ = !r.neg_;
    return r;
  }
  BigInt& operator+=(const BigInt& o) {
    if (neg_ == o.neg_) {
      add_mag(mag_, o.mag_);
    } else if (cmp_mag(mag_, o.mag_) >= 0) {
      sub_mag(mag_, o.mag_);
    } else {
      std::vector<uint32_t> t = o.mag_;
      sub_mag(t, mag_);
      mag_.swap(t);
      neg_ = o.neg_;
    }
    if (mag_.empty()) neg_ = false;
    return *this;
  }
  BigInt& operator-=(const BigInt& o) { return *this += -o; }
  friend BigInt operator+(BigInt a, const BigInt& b) { return a += b; }
  friend BigInt operator-(BigInt a, const BigInt& b) { return a -= b; }
  friend BigInt operator*(const BigInt& a, const BigInt& b) {
    BigInt r;
    if (a.is_zero() || b.is_zero()) return r;
    r.mag_.assign(a.mag_.size() + b.mag_.size(), 0);
    for (size_t i = 0; i < a.mag_.size(); ++i) {
      uint64_t carry = 0;
      for (size_t j = 0; j < b.mag_.size(); ++j) {
        const uint64_t t = static_cast<uint64_t>(a.mag_[i]) * b.mag_[j] + r.mag_[i + j] + carry;
        r.mag_[i + j] = static_cast<uint32_t>(t);
        carry = t >> 32;
      }
      r.mag_[i + b.mag_.size()] = static_cast<uint32_t>(carry);
    }
    trim(r.mag_);
    r.neg_ = a.neg_ != b.neg_;
    return r;
  }
  friend bool operator==(const BigInt& a, const BigInt& b) { return a.neg_ == b.neg_ && a.mag_ == b.mag_; }
  friend bool operator!=(const BigInt& a, const BigInt& b) { return !(a == b); }
  std::string str() const {
    if (is_zero()) return "0";
    std::vector<uint32_t> m = mag_;
    std::string digits;
    while (!m.empty()) {  // divide by 10^9, collect remainders
      uint64_t rem = 0;
      for (size_t i = m.size(); i-- > 0;) {
        const uint64_t cur = (rem << 32) | m[i];
        m[i] = static_cast<uint32_t>(cur / 1000000000u);
        rem = cur % 1000000000u;
      }
      trim(m);
      char buf[16];
      std::snprintf(buf, sizeof buf, m.empty() ? "%u" : "%09u", static_cast<unsigned>(rem));
      digits.insert(0, buf);
    }
    return (neg_ ? "-" : "") + digits;
  }

 private:
  static void trim(std::vector<uint32_t>& m) {
    while (!m.empty() && m.back() == 0) m.pop_back();
  }
  static int cmp_mag(const std::vector<uint32_t>& a, const std::vector<uint32_t>& b) {
    if (a.size() != b.size()) return a.size() < b.size() ? -1 : 1;
    for (size_t i = a.size(); i-- > 0;)
      if (a[i] != b[i]) return a[i] < b[i] ? -1 : 1;
    return 0;
  }
  static void add_mag(std::vector<uint32_t>& a, const std::vector<uint32_t>& b) {
    if (a.size() < b.size()) a.resize(b.size(), 0);
    uint64_t carry = 0;
    for (size_t i = 0; i < a.size(); ++i) {
      const uint64_t t = static_cast<uint64_t>(a[i]) + (i < b.size() ? b[i] : 0u) + carry;
      a[i] = static_cast<uint32_t>(t);
      carry = t >> 32;
      if (!carry && i >= b.size()) break;
    }
    if (carry) a.push_back(static_cast<uint32_t>(carry));
  }
  static void sub_mag(std::vector<uint32_t>& a, const std::vector<uint32_t>& b) {  // |a| >= |b|
    int64_t borrow = 0;
    for (size_t i = 0; i < a.size(); ++i) {
      int64_t t = static_cast<int64_t>(a[i]) - (i < b.size() ? b[i] : 0u) - borrow;
      borrow = t < 0;
      if (t < 0) t += (1ll << 32);
      a[i] = static_cast<uint32_t>(t);
      if (!borrow && i >= b.size()) break;
    }
    trim(a);
  }
  bool neg_ = false;
  std::vector<uint32_t> mag_;
};

// ---------------------------------------------------------------------------
// Multilinear polynomials over 0/1 variables (node ids; x^2 = x).
// ---------------------------------------------------------------------------
using Monomial = std::vector<uint32_t>;  // sorted, unique; {} = constant term
using Terms = std::map<Monomial, BigInt>;

Monomial mono_mul(const Monomial& a, const Monomial& b) {
  Monomial m;
  m.reserve(a.size() + b.size());
  std::set_union(a.begin(), a.end(), b.begin(), b.end(), std::back_inserter(m));
  return m;
}

void add_term(Terms& t, const Monomial& m, const BigInt& c) {
  if (c.is_zero()) return;
  auto [it, fresh] = t.try_emplace(m, c);
  if (!fresh) {
    it->second += c;
    if (it->second.is_zero()) t.erase(it);
  }
}

Terms poly_mul(const Terms& a, const Terms& b) {
  Terms r;
  for (const auto& [ma, ca] : a)
    for (const auto& [mb, cb] : b) add_term(r, mono_mul(ma, mb), ca * cb);
  return r;
}
Terms poly_add(Terms a, const Terms& b, const BigInt& scale = 1) {
  for (const auto& [m, c] : b) add_term(a, m, c * scale);
  return a;
}
Terms poly_const(const BigInt& c) {
  Terms t;
  add_term(t, {}, c);
  return t;
}
// literal of node v: x_v, or 1 - x_v when inverted; node 0 is constant false
Terms poly_lit(uint32_t node, bool inv) {
  if (node == 0) return poly_const(inv ? 1 : 0);
  Terms t;
  if (inv) add_term(t, {}, 1);
  add_term(t, {node}, inv ? -1 : 1);
  return t;
}

// Operator models (src/polynomial.cpp:122-156):
//   XOR2 a+b-2ab, XOR3 a+b+c-2(ab+ac+bc)+4abc, MAJ ab+ac+bc-2abc, AND ab.
Terms model_xor(const std::vector<Terms>& x) {
  const Terms ab = poly_mul(x[0], x[1]);
  Terms r = poly_add(poly_add(x[0], x[1]), ab, -2);
  if (x.size() == 3) {
    const Terms ac = poly_mul(x[0], x[2]), bc = poly_mul(x[1], x[2]);
    r = poly_add(r, x[2]);
    r = poly_add(poly_add(r, ac, -2), bc, -2);
    r = poly_add(r, poly_mul(ab, x[2]), 4);
  }
  return r;
}
Terms model_maj(const std::vector<Terms>& x) {
  const Terms ab = poly_mul(x[0], x[1]), ac = poly_mul(x[0], x[2]), bc = poly_mul(x[1], x[2]);
  return poly_add(poly_add(poly_add(ab, ac), bc), poly_mul(ab, x[2]), -2);
}

// ---------------------------------------------------------------------------
// AIG view over the C-ABI literal arrays.
// ---------------------------------------------------------------------------
struct AigView {
  uint32_t ni = 0, na = 0;
  const uint32_t* ands = nullptr;  // 2 literals per AND
  uint32_t num_nodes() const { return 1 + ni + na; }
  uint32_t first_and() const { return 1 + ni; }
  bool is_input(uint32_t v) const { return v >= 1 && v <= ni; }
  bool is_and(uint32_t v) const { return v >= first_and() && v < num_nodes(); }
  uint32_t lit(uint32_t v, int side) const { return ands[2 * (v - first_and()) + side]; }
};

enum class Fn : uint8_t { Xor, Maj, And };

struct RootModel {  // base function over (support[i] ^ pin[i]), complemented when out_inv
  Fn fn;
  std::vector<uint32_t> support;  // sorted node ids
  std::vector<uint8_t> pin;
  bool out_inv = false;
  uint8_t tt = 0;
};

// Truth table of v over the support nodes (bit i of the row index drives
// support[i]); none when the cone reaches another input or passes 64 nodes.
std::optional<uint8_t> cone_truth_table(const AigView& g, uint32_t v, const std::vector<uint32_t>& sup) {
  constexpr int kBudget = 64;
  uint8_t tt = 0;
  std::vector<std::pair<uint32_t, uint8_t>> memo;
  for (uint32_t row = 0; row < (1u << sup.size()); ++row) {
    memo.clear();
    int budget = kBudget;
    bool ok = true;
    auto eval = [&](auto&& self, uint32_t node) -> uint8_t {
      for (size_t i = 0; i < sup.size(); ++i)
        if (sup[i] == node) return (row >> i) & 1u;
      if (node == 0) return 0;
      if (g.is_input(node) || !ok) {
        ok = false;
        return 0;
      }
      for (const auto& [n, bit] : memo)
        if (n == node) return bit;
      if (--budget < 0) {
        ok = false;
        return 0;
      }
      const uint32_t l = g.lit(node, 0), r = g.lit(node, 1);
      const uint8_t lb = self(self, l >> 1) ^ (l & 1u);
      if (!ok) return 0;
      const uint8_t rb = self(self, r >> 1) ^ (r & 1u);
      if (!ok) return 0;
      const uint8_t bit = lb & rb;
      memo.emplace_back(node, bit);
      return bit;
    };
    const uint8_t bit = eval(eval, v);
    if (!ok) return std::nullopt;
    tt |= static_cast<uint8_t>(bit << row);
  }
  return tt;
}

uint8_t fn_table(Fn fn, size_t arity, uint32_t pin_mask, bool out_inv) {
  uint8_t tt = 0;
  for (uint32_t row = 0; row < (1u << arity); ++row) {
    const uint32_t x = row ^ pin_mask, a = x & 1u, b = (x >> 1) & 1u, c = (x >> 2) & 1u;
    uint32_t bit = fn == Fn::Xor ? (arity == 2 ? a ^ b : a ^ b ^ c) : fn == Fn::Maj ? ((a & b) | (a & c) | (b & c)) : (a & b);
    tt |= static_cast<uint8_t>((bit ^ (out_inv ? 1u : 0u)) << row);
  }
  return tt;
}

// input / output polarities under which fn over the support gives tt
std::optional<RootModel> fit_polarity(Fn fn, uint8_t tt, const std::vector<uint32_t>& sup) {
  for (uint32_t pin = 0; pin < (1u << sup.size()); ++pin)
    for (int out = 0; out < 2; ++out)
      if (fn_table(fn, sup.size(), pin, out != 0) == tt) {
        RootModel m{fn, sup, std::vector<uint8_t>(sup.size()), out != 0, tt};
        for (size_t i = 0; i < sup.size(); ++i) m.pin[i] = (pin >> i) & 1u;
        return m;
      }
  return std::nullopt;
}

// v = AND(~AND(x,y), ~AND(~x,~y)) style: both fan-ins are ANDs over the same two nodes
std::optional<std::array<uint32_t, 2>> xor2_pair(const AigView& g, uint32_t v) {
  if (!g.is_and(v)) return std::nullopt;
  const uint32_t p = g.lit(v, 0) >> 1, q = g.lit(v, 1) >> 1;
  if (!g.is_and(p) || !g.is_and(q)) return std::nullopt;
  std::array<uint32_t, 2> a{g.lit(p, 0) >> 1, g.lit(p, 1) >> 1}, b{g.lit(q, 0) >> 1, g.lit(q, 1) >> 1};
  std::sort(a.begin(), a.end());
  std::sort(b.begin(), b.end());
  if (a != b || a[0] == a[1]) return std::nullopt;
  return a;
}

// Structural support candidates of a labelled root (src/verify.cpp:136-180).
std::vector<std::vector<uint32_t>> structural_supports(const AigView& g, uint32_t v, uint8_t label) {
  std::vector<std::vector<uint32_t>> out;
  auto add = [&](std::vector<uint32_t> s) {
    std::sort(s.begin(), s.end());
    if (std::adjacent_find(s.begin(), s.end()) != s.end()) return;
    for (uint32_t x : s)
      if (x == 0 || x >= v) return;
    if (std::find(out.begin(), out.end(), s) == out.end()) out.push_back(std::move(s));
  };
  if (label == 2) {  // XOR: XOR3 through an inner XOR2 on either side, then XOR2
    if (auto s = xor2_pair(g, v)) {
      const uint32_t x = (*s)[0], y = (*s)[1];
      if (auto sx = xor2_pair(g, x)) add({(*sx)[0], (*sx)[1], y});
      if (auto sy = xor2_pair(g, y)) add({x, (*sy)[0], (*sy)[1]});
      add({x, y});
    }
  } else if (label == 1) {  // MAJ: full-adder carry over (a, b, cin), else a 2-input AND
    const uint32_t p = g.lit(v, 0) >> 1, q = g.lit(v, 1) >> 1;
    if (g.is_and(p) && g.is_and(q)) {
      for (const auto& [c1, c2] : {std::pair{p, q}, std::pair{q, p}}) {
        std::array<uint32_t, 2> base{g.lit(c1, 0) >> 1, g.lit(c1, 1) >> 1};
        std::sort(base.begin(), base.end());
        const uint32_t f0 = g.lit(c2, 0) >> 1, f1 = g.lit(c2, 1) >> 1;
        for (const auto& [inner, other] : {std::pair{f0, f1}, std::pair{f1, f0}}) {
          const auto sx = xor2_pair(g, inner);
          if (sx && *sx == base) add({base[0], base[1], other});
        }
      }
    }
    add({p, q});
  }
  return out;
}

Terms root_poly(const RootModel& m) {
  std::vector<Terms> x;
  for (size_t i = 0; i < m.support.size(); ++i) x.push_back(poly_lit(m.support[i], m.pin[i] != 0));
  Terms base = m.fn == Fn::Xor ? model_xor(x) : m.fn == Fn::Maj ? model_maj(x) : poly_mul(x[0], x[1]);
  return m.out_inv ? poly_add(poly_const(1), base, -1) : base;
}

// Word polynomial with a per-variable count of the terms holding it.
struct Word {
  Terms t;
  std::vector<uint32_t> occ;
  explicit Word(uint32_t nvars) : occ(nvars, 0) {}
  void add(const Monomial& m, const BigInt& c) {
    if (c.is_zero()) return;
    auto [it, fresh] = t.try_emplace(m, c);
    if (fresh) {
      for (uint32_t x : m) ++occ[x];
      return;
    }
    it->second += c;
    if (it->second.is_zero()) {
      for (uint32_t x : m) --occ[x];
      t.erase(it);
    }
  }
  void add(const Terms& p, const BigInt& scale) {
    for (const auto& [m, c] : p) add(m, c * scale);
  }
  BigInt coeff(const Monomial& m) const {
    auto it = t.find(m);
    return it == t.end() ? BigInt() : it->second;
  }
};

Terms spec_poly(uint32_t w) {  // (sum 2^i a_i)(sum 2^j b_j), a_i = node 1+i, b_j = node 1+w+j
  Terms s;
  for (uint32_t i = 0; i < w; ++i)
    for (uint32_t j = 0; j < w; ++j) add_term(s, {1 + i, 1 + w + j}, BigInt::pow2(i + j));
  return s;
}

struct Report {
  bool equivalent = false, inconclusive = false;
  Terms residual;
  uint64_t substitutions = 0, shortcuts = 0, fallbacks = 0;
};

// supports: for node v, sup_off[v]..sup_off[v+1] index sup_nodes (may be empty)
Report rewrite(const AigView& g, const std::vector<uint32_t>& outs, const uint8_t* labels,
               const std::vector<std::vector<uint32_t>>& given, uint32_t w, uint64_t cap) {
  Report rep;
  const uint32_t N = g.num_nodes();
  Word word(N);
  for (size_t k = 0; k < outs.size(); ++k) word.add(poly_lit(outs[k] >> 1, outs[k] & 1u), BigInt::pow2(static_cast<uint32_t>(k)));

  std::vector<std::optional<RootModel>> models(N);
  std::vector<uint8_t> resolved(N, 0);
  auto model_of = [&](uint32_t v) -> const std::optional<RootModel>& {
    if (resolved[v]) return models[v];
    resolved[v] = 1;
    const uint8_t label = labels[v];
    if (label != 2 && label != 1) return models[v];
    std::vector<std::vector<uint32_t>> cands;
    if (v < given.size() && (given[v].size() == 2 || given[v].size() == 3)) {
      std::vector<uint32_t> s = given[v];
      std::sort(s.begin(), s.end());
      bool ok = std::adjacent_find(s.begin(), s.end()) == s.end();
      for (uint32_t x : s) ok = ok && x != 0 && x < v;
      if (ok) cands.push_back(std::move(s));
    }
    for (auto& s : structural_supports(g, v, label))
      if (std::find(cands.begin(), cands.end(), s) == cands.end()) cands.push_back(std::move(s));
    for (const auto& s : cands) {
      const auto tt = cone_truth_table(g, v, s);
      if (!tt) continue;
      const Fn fn = label == 2 ? Fn::Xor : s.size() == 3 ? Fn::Maj : Fn::And;
      if (auto m = fit_polarity(fn, *tt, s)) {
        models[v] = std::move(m);
        break;
      }
    }
    return models[v];
  };
  // an XOR model re-fitted to prescribed input polarities (XOR absorbs them in the output)
  auto xor_with_pins = [&](const RootModel& x, const std::vector<uint8_t>& pin) -> std::optional<RootModel> {
    uint32_t mask = 0;
    for (size_t i = 0; i < pin.size(); ++i) mask |= static_cast<uint32_t>(pin[i]) << i;
    for (int out = 0; out < 2; ++out)
      if (fn_table(Fn::Xor, x.support.size(), mask, out != 0) == x.tt) {
        RootModel m = x;
        m.pin = pin;
        m.out_inv = out != 0;
        return m;
      }
    return std::nullopt;
  };

  for (uint32_t v = N - 1; v >= g.first_and() && v < N; --v) {
    if (word.occ[v] == 0) continue;
    const uint8_t label = labels[v];
    const std::optional<RootModel>& root = model_of(v);
    if ((label == 2 || label == 1) && !root) ++rep.fallbacks;

    // full-adder shortcut: linear XOR / MAJ pair over one support, coefficients c and 2c
    if (root && word.occ[v] == 1) {
      const BigInt cv = word.coeff({v});
      if (!cv.is_zero()) {
        const bool v_xor = root->fn == Fn::Xor;
        uint32_t partner = 0;
        std::optional<RootModel> xm, um;
        BigInt cx, cu;
        for (const auto& [m, c] : word.t) {
          if (m.size() != 1 || m[0] == v) continue;
          const uint32_t u = m[0];
          if (!g.is_and(u) || word.occ[u] != 1) continue;
          if (labels[u] != (v_xor ? 1 : 2)) continue;
          const auto& other = model_of(u);
          if (!other || other->support != root->support) continue;
          auto rx = v_xor ? xor_with_pins(*root, other->pin) : xor_with_pins(*other, root->pin);
          if (!rx) continue;
          xm = rx;
          um = v_xor ? *other : *root;
          cx = v_xor ? cv : c;
          cu = v_xor ? c : cv;
          partner = u;
          break;
        }
        if (partner) {
          const BigInt sx = xm->out_inv ? -1 : 1, su = um->out_inv ? -1 : 1;
          if (cu * su == BigInt(2) * cx * sx) {
            word.add(Monomial{v}, -cv);
            word.add(Monomial{partner}, v_xor ? -cu : -cx);
            BigInt k0;
            if (xm->out_inv) k0 += cx;
            if (um->out_inv) k0 += cu;
            word.add(Monomial{}, k0);
            for (size_t i = 0; i < xm->support.size(); ++i)
              word.add(poly_lit(xm->support[i], xm->pin[i] != 0), cx * sx);
            rep.shortcuts += 1;
            rep.substitutions += 2;
            continue;
          }
        }
      }
    }

    // substitute v by its model, or by the AND of its fan-ins
    const Terms model = root ? root_poly(*root)
                             : poly_mul(poly_lit(g.lit(v, 0) >> 1, g.lit(v, 0) & 1u), poly_lit(g.lit(v, 1) >> 1, g.lit(v, 1) & 1u));
    std::vector<std::pair<Monomial, BigInt>> hit;
    for (const auto& [m, c] : word.t)
      if (std::binary_search(m.begin(), m.end(), v)) hit.emplace_back(m, c);
    if (word.t.size() + hit.size() * model.size() > cap) {
      rep.inconclusive = true;
      return rep;
    }
    for (const auto& [m, c] : hit) {
      word.add(m, -c);
      Monomial rest;
      for (uint32_t x : m)
        if (x != v) rest.push_back(x);
      for (const auto& [pm, pc] : model) word.add(mono_mul(rest, pm), c * pc);
    }
    ++rep.substitutions;
  }
  rep.residual = poly_add(word.t, spec_poly(w), -1);
  rep.equivalent = rep.residual.empty();
  return rep;
}

// simulate (src/aig.cpp:115-138): output bits for one input assignment
void simulate_outputs(const AigView& g, const std::vector<uint32_t>& outs, const uint8_t* in, uint8_t* out) {
  std::vector<uint8_t> val(g.num_nodes(), 0);
  for (uint32_t i = 0; i < g.ni; ++i) val[1 + i] = in[i] ? 1 : 0;
  for (uint32_t a = 0; a < g.na; ++a) {
    const uint32_t l = g.ands[2 * a], r = g.ands[2 * a + 1];
    val[g.first_and() + a] = (val[l >> 1] ^ (l & 1u)) & (val[r >> 1] ^ (r & 1u));
  }
  for (size_t k = 0; k < outs.size(); ++k) out[k] = val[outs[k] >> 1] ^ (outs[k] & 1u);
}

void check_aig(uint32_t ni, uint32_t na, const uint32_t* ands, uint32_t no, const uint32_t* outs) {
  if (na && !ands) fail(GROOT_EINVAL, "verify: null AND literals");
  if (no && !outs) fail(GROOT_EINVAL, "verify: null output literals");
  for (uint32_t a = 0; a < na; ++a)
    for (int s = 0; s < 2; ++s)
      if ((ands[2 * a + s] >> 1) >= 1 + ni + a)
        fail(GROOT_EINVAL, "Aig::add_and: fanin index must be strictly below the new node");
  for (uint32_t k = 0; k < no; ++k)
    if ((outs[k] >> 1) >= 1 + ni + na) fail(GROOT_EINVAL, "Aig::add_output: driver references unknown node");
}

thread_local std::string g_residual_text;

}  // namespace
}  // namespace groot

using namespace groot;

extern "C" {

int groot_backward_rewrite(uint32_t ni, uint32_t na, const uint32_t* ands, uint32_t no, const uint32_t* outs,
                           const uint8_t* labels, uint32_t num_labels, const uint32_t* support_off,
                           const uint32_t* support_nodes, uint32_t width, uint64_t monomial_cap, int32_t* equivalent,
                           int32_t* inconclusive, uint64_t* residual_terms, uint64_t* counts) {
  return guarded([&] {
    check_aig(ni, na, ands, no, outs);
    const AigView g{ni, na, ands};
    if (!labels || num_labels < g.num_nodes())
      fail(GROOT_EINVAL, "backward_rewrite: labels do not cover the graph");
    if (ni != 2 * width || no != 2 * width)
      fail(GROOT_EINVAL, "backward_rewrite: not a width-bit multiplier candidate");
    std::vector<std::vector<uint32_t>> given;
    if (support_off && support_nodes) {
      given.resize(g.num_nodes());
      for (uint32_t v = 0; v < g.num_nodes(); ++v)
        given[v].assign(support_nodes + support_off[v], support_nodes + support_off[v + 1]);
    }
    const std::vector<uint32_t> o(outs, outs + no);
    const Report r = rewrite(g, o, labels, given, width, monomial_cap ? monomial_cap : 2000000ull);
    if (equivalent) *equivalent = r.equivalent ? 1 : 0;
    if (inconclusive) *inconclusive = r.inconclusive ? 1 : 0;
    if (residual_terms) *residual_terms = r.residual.size();
    if (counts) {
      counts[0] = r.substitutions;
      counts[1] = r.shortcuts;
      counts[2] = r.fallbacks;
    }
    // the residual as text (first 64 terms): "coeff*x1*x5 + ..."
    std::string s;
    size_t shown = 0;
    for (const auto& [m, c] : r.residual) {
      if (shown++ == 64) {
        s += " + ...";
        break;
      }
      if (!s.empty()) s += " + ";
      s += c.str();
      for (uint32_t x : m) s += "*x" + std::to_string(x);
    }
    g_residual_text = s;
  });
}

const char* groot_backward_rewrite_residual(void) { return g_residual_text.c_str(); }

int groot_truth_table_equiv(uint32_t ni, uint32_t na, const uint32_t* ands, uint32_t no, const uint32_t* outs,
                            uint32_t width, int32_t* equivalent) {
  return guarded([&] {
    if (2 * width > 20) fail(GROOT_EINVAL, "truth_table_equiv: width too large");
    check_aig(ni, na, ands, no, outs);
    if (ni != 2 * width || no != 2 * width)
      fail(GROOT_EINVAL, "truth_table_equiv: not a width-bit multiplier candidate");
    const AigView g{ni, na, ands};
    const std::vector<uint32_t> o(outs, outs + no);
    std::vector<uint8_t> in(ni), out(no);
    bool eq = true;
    for (uint64_t a = 0; a < (1ull << width) && eq; ++a)
      for (uint64_t b = 0; b < (1ull << width) && eq; ++b) {
        for (uint32_t i = 0; i < width; ++i) {
          in[i] = (a >> i) & 1u;
          in[width + i] = (b >> i) & 1u;
        }
        simulate_outputs(g, o, in.data(), out.data());
        uint64_t got = 0;
        for (uint32_t k = 0; k < no; ++k) got |= static_cast<uint64_t>(out[k]) << k;
        eq = got == a * b;
      }
    *equivalent = eq ? 1 : 0;
  });
}

int groot_simulate(uint32_t ni, uint32_t na, const uint32_t* ands, uint32_t no, const uint32_t* outs,
                   const uint8_t* inputs, uint8_t* outputs) {
  return guarded([&] {
    check_aig(ni, na, ands, no, outs);
    const std::vector<uint32_t> o(outs, outs + no);
    simulate_outputs(AigView{ni, na, ands}, o, inputs, outputs);
  });
}

}  // extern "C"
