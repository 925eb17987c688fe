// train.cu — full-batch GraphSAGE training on the device.
//
// Reference: loss_and_grads + train (src/gnn.cpp:180-255): forward with the
// whole cache (h, m, z per layer), softmax cross entropy averaged over nodes
// (:56-68), backward through the head and the layers with the transposed mean
// aggregation a_mean_t (values 1/deg(u) on row v's neighbour u, :158-166), and
// Adam with bias correction (:236-250). Everything runs in fp64 like the
// reference, with deterministic orders: every sum runs over its index in
// ascending order with separately rounded multiply and add, except the
// weight-gradient reductions over nodes, which sum fixed 256-row blocks and
// add the block sums in block order. The training graphs are small (an 8-bit CSA
// has 457 nodes), so these kernels favour a fixed order over throughput;
// the inference path is forward.cu.
#include <cmath>
#include <vector>

#include "common.cuh"

namespace groot {
namespace {

__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }

constexpr uint32_t kHdAgg = 512;   // rows of at least this degree: 32 ordered chunk partials (execute's HD band)
constexpr uint32_t kRowBlock = 256;  // rows per partial of a reduction over nodes

__global__ void tr_features_kernel(uint32_t n, const uint8_t* __restrict__ feat, double* __restrict__ h) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < 4 * n; i += gridDim.x * blockDim.x) h[i] = feat[i];
}

// out[r][c] = sum_k val_k x[col_k][c]; val = 1/deg(r) (a_mean) or 1/deg(col_k) (a_mean_t)
__global__ void tr_agg_kernel(uint32_t n, const uint32_t* __restrict__ rp, const uint32_t* __restrict__ col,
                              const double* __restrict__ x, uint32_t f, int transpose, double* __restrict__ out) {
  const uint64_t total = static_cast<uint64_t>(n) * f;
  for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t r = static_cast<uint32_t>(t / f), c = static_cast<uint32_t>(t % f);
    const uint32_t b = rp[r], e = rp[r + 1], d = e - b;
    const double vr = d ? 1.0 / static_cast<double>(d) : 0.0;
    auto sum = [&](uint32_t q0, uint32_t q1) {
      double acc = 0.0;
      for (uint32_t q = q0; q < q1; ++q) {
        const uint32_t u = col[q];
        double v = vr;
        if (transpose) {
          const uint32_t du = rp[u + 1] - rp[u];
          v = du ? 1.0 / static_cast<double>(du) : 0.0;
        }
        acc = dadd(acc, dmul(v, x[static_cast<size_t>(u) * f + c]));
      }
      return acc;
    };
    double acc = 0.0;
    if (d >= kHdAgg) {
      const uint32_t qd = d / 32, rem = d % 32;
      uint32_t nz = b;
      for (uint32_t k = 0; k < 32; ++k) {
        const uint32_t len = qd + (k >= 32 - rem ? 1u : 0u);
        acc = dadd(acc, sum(nz, nz + len));
        nz += len;
      }
    } else {
      acc = sum(b, e);
    }
    out[t] = acc;
  }
}

// z = (h Ws + m Wn) + b, hn = max(z, 0): thread per (row, output)
__global__ void tr_dense_kernel(uint32_t n, const double* __restrict__ h, const double* __restrict__ m,
                                uint32_t in, uint32_t out, const double* __restrict__ ws,
                                const double* __restrict__ wn, const double* __restrict__ bias,
                                double* __restrict__ z, double* __restrict__ hn) {
  const uint64_t total = static_cast<uint64_t>(n) * out;
  for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t r = static_cast<uint32_t>(t / out), j = static_cast<uint32_t>(t % out);
    double s1 = 0.0, s2 = 0.0;
    for (uint32_t k = 0; k < in; ++k) {
      s1 = dadd(s1, dmul(h[static_cast<size_t>(r) * in + k], ws[k * out + j]));
      s2 = dadd(s2, dmul(m[static_cast<size_t>(r) * in + k], wn[k * out + j]));
    }
    const double zz = dadd(dadd(s1, s2), bias[j]);
    z[t] = zz;
    hn[t] = zz > 0.0 ? zz : 0.0;
  }
}

// logits = h Wout + bout
__global__ void tr_head_kernel(uint32_t n, const double* __restrict__ h, uint32_t hid, uint32_t classes,
                               const double* __restrict__ wo, const double* __restrict__ bo,
                               double* __restrict__ logits) {
  const uint64_t total = static_cast<uint64_t>(n) * classes;
  for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t r = static_cast<uint32_t>(t / classes), j = static_cast<uint32_t>(t % classes);
    double s = 0.0;
    for (uint32_t k = 0; k < hid; ++k) s = dadd(s, dmul(h[static_cast<size_t>(r) * hid + k], wo[k * classes + j]));
    logits[t] = dadd(s, bo[j]);
  }
}

// softmax cross entropy (src/gnn.cpp:56-68): per row the loss term, the hit
// (first maximum), and dlogits = (prob - onehot) / n
__global__ void tr_softmax_kernel(uint32_t n, uint32_t classes, const double* __restrict__ logits,
                                  const uint8_t* __restrict__ labels, double* __restrict__ row_loss,
                                  uint32_t* __restrict__ row_hit, double* __restrict__ dl) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const double* lg = logits + static_cast<size_t>(i) * classes;
    double mx = lg[0];
    uint32_t arg = 0;
    for (uint32_t j = 1; j < classes; ++j)
      if (lg[j] > mx) {
        mx = lg[j];
        arg = j;
      }
    double e[8], den = 0.0;
    for (uint32_t j = 0; j < classes; ++j) {
      e[j] = exp(lg[j] - mx);
      den = dadd(den, e[j]);
    }
    const uint32_t y = labels[i];
    row_loss[i] = -log(e[y] / den);
    row_hit[i] = arg == y;
    const double inv_n = static_cast<double>(n);
    for (uint32_t j = 0; j < classes; ++j) {
      double p = e[j] / den;
      if (j == y) p -= 1.0;
      dl[static_cast<size_t>(i) * classes + j] = p / inv_n;
    }
  }
}

// partial[blk][a][j] = sum over rows of block blk of A[i][a] * B[i][j]
// (A == nullptr: ones, i.e. column sums of B)
__global__ void tr_outer_partial_kernel(uint32_t n, const double* __restrict__ A, uint32_t p,
                                        const double* __restrict__ B, uint32_t q, double* __restrict__ partial) {
  const uint32_t blocks = (n + kRowBlock - 1) / kRowBlock;
  const uint64_t total = static_cast<uint64_t>(blocks) * p * q;
  for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t blk = static_cast<uint32_t>(t / (static_cast<uint64_t>(p) * q));
    const uint32_t a = static_cast<uint32_t>((t / q) % p), j = static_cast<uint32_t>(t % q);
    const uint32_t i0 = blk * kRowBlock, i1 = min(n, i0 + kRowBlock);
    double s = 0.0;
    for (uint32_t i = i0; i < i1; ++i) {
      const double av = A ? A[static_cast<size_t>(i) * p + a] : 1.0;
      s = dadd(s, A ? dmul(av, B[static_cast<size_t>(i) * q + j]) : B[static_cast<size_t>(i) * q + j]);
    }
    partial[t] = s;
  }
}

__global__ void tr_reduce_partials_kernel(uint32_t blocks, uint32_t count, const double* __restrict__ partial,
                                          double* __restrict__ out) {
  for (uint32_t t = blockIdx.x * blockDim.x + threadIdx.x; t < count; t += gridDim.x * blockDim.x) {
    double s = 0.0;
    for (uint32_t b = 0; b < blocks; ++b) s = dadd(s, partial[static_cast<size_t>(b) * count + t]);
    out[t] = s;
  }
}

// dh = dl Wout^T (rows x hid)
__global__ void tr_back_head_kernel(uint32_t n, const double* __restrict__ dl, uint32_t classes, uint32_t hid,
                                    const double* __restrict__ wo, double* __restrict__ dh) {
  const uint64_t total = static_cast<uint64_t>(n) * hid;
  for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t i = static_cast<uint32_t>(t / hid), a = static_cast<uint32_t>(t % hid);
    double s = 0.0;
    for (uint32_t j = 0; j < classes; ++j) s = dadd(s, dmul(dl[static_cast<size_t>(i) * classes + j], wo[a * classes + j]));
    dh[t] = s;
  }
}

__global__ void tr_relu_mask_kernel(uint64_t count, const double* __restrict__ z, const double* __restrict__ dh,
                                    double* __restrict__ dz) {
  for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < count;
       t += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    dz[t] = z[t] > 0.0 ? dh[t] : 0.0;
}

// a1 = dz Ws^T, a2 = dz Wn^T (rows x in)
__global__ void tr_back_layer_kernel(uint32_t n, const double* __restrict__ dz, uint32_t out, uint32_t in,
                                     const double* __restrict__ ws, const double* __restrict__ wn,
                                     double* __restrict__ a1, double* __restrict__ a2) {
  const uint64_t total = static_cast<uint64_t>(n) * in;
  for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < total;
       t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const uint32_t i = static_cast<uint32_t>(t / in), a = static_cast<uint32_t>(t % in);
    double s1 = 0.0, s2 = 0.0;
    for (uint32_t j = 0; j < out; ++j) {
      const double g = dz[static_cast<size_t>(i) * out + j];
      s1 = dadd(s1, dmul(g, ws[a * out + j]));
      s2 = dadd(s2, dmul(g, wn[a * out + j]));
    }
    a1[t] = s1;
    a2[t] = s2;
  }
}

__global__ void tr_add_kernel(uint64_t count, const double* __restrict__ a, const double* __restrict__ b,
                              double* __restrict__ out) {
  for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < count;
       t += static_cast<uint64_t>(gridDim.x) * blockDim.x)
    out[t] = dadd(a[t], b[t]);
}

// Adam with bias correction (src/gnn.cpp:236-250)
__global__ void tr_adam_kernel(uint64_t count, double* __restrict__ prm, const double* __restrict__ grad,
                               double* __restrict__ m1, double* __restrict__ m2, double lr, double b1, double b2,
                               double eps, double bc1, double bc2) {
  for (uint64_t t = blockIdx.x * static_cast<uint64_t>(blockDim.x) + threadIdx.x; t < count;
       t += static_cast<uint64_t>(gridDim.x) * blockDim.x) {
    const double g = grad[t];
    m1[t] = dadd(dmul(b1, m1[t]), dmul(1.0 - b1, g));
    m2[t] = dadd(dmul(b2, m2[t]), dmul(dmul(1.0 - b2, g), g));
    prm[t] = prm[t] - dmul(lr, m1[t] / bc1) / (sqrt(m2[t] / bc2) + eps);
  }
}

// loss = (row terms summed in row order) / n, accuracy = hits / n (one thread)
__global__ void tr_loss_kernel(uint32_t n, const double* __restrict__ row_loss, const uint32_t* __restrict__ row_hit,
                               double* __restrict__ loss, double* __restrict__ acc) {
  if (blockIdx.x != 0 || threadIdx.x != 0) return;
  double s = 0.0;
  uint64_t hits = 0;
  for (uint32_t i = 0; i < n; ++i) {
    s = dadd(s, row_loss[i]);
    hits += row_hit[i];
  }
  *loss = s / static_cast<double>(n);
  *acc = n ? static_cast<double>(hits) / static_cast<double>(n) : 0.0;
}

struct Shape {
  uint32_t depth, in_dim, hidden, classes;
  uint64_t count() const {
    uint64_t c = 0;
    uint32_t in = in_dim;
    for (uint32_t l = 0; l < depth; ++l) {
      c += 2ull * in * hidden + hidden;
      in = hidden;
    }
    return c + static_cast<uint64_t>(in) * classes + classes;
  }
  uint64_t layer_off(uint32_t l) const {
    uint64_t o = 0;
    uint32_t in = in_dim;
    for (uint32_t k = 0; k < l; ++k) {
      o += 2ull * in * hidden + hidden;
      in = hidden;
    }
    return o;
  }
  uint32_t in_of(uint32_t l) const { return l ? hidden : in_dim; }
};

unsigned grid_for(uint64_t items) { return blocks_for(items, 256, static_cast<unsigned>(num_sms()) * 8); }

// One loss_and_grads (src/gnn.cpp:180-209) on device buffers; loss/acc are device scalars.
struct Trainer {
  const groot_graph* g;
  Shape s;
  uint32_t n;
  DevBuf<double> x0, logits, dl, rloss, dh, dz, a1, a2, t, partial;
  DevBuf<uint32_t> rhit;
  std::vector<DevBuf<double>> h, m, z;

  Trainer(const groot_graph* graph, Shape shape) : g(graph), s(shape), n(graph->n) {
    const size_t H = shape.hidden;
    x0.alloc(4ull * n);
    GROOT_LAUNCH(tr_features_kernel, grid_for(4ull * n), 256, 0, n, g->feat.p, x0.p);
    h.resize(s.depth + 1);
    m.resize(s.depth);
    z.resize(s.depth);
    for (uint32_t l = 0; l < s.depth; ++l) {
      m[l].alloc(static_cast<size_t>(n) * s.in_of(l));
      z[l].alloc(static_cast<size_t>(n) * H);
      h[l + 1].alloc(static_cast<size_t>(n) * H);
    }
    logits.alloc(static_cast<size_t>(n) * s.classes);
    dl.alloc(static_cast<size_t>(n) * s.classes);
    rloss.alloc(n);
    rhit.alloc(n);
    dh.alloc(static_cast<size_t>(n) * H);
    dz.alloc(static_cast<size_t>(n) * H);
    a1.alloc(static_cast<size_t>(n) * H);
    a2.alloc(static_cast<size_t>(n) * H);
    t.alloc(static_cast<size_t>(n) * H);
    const uint32_t blocks = (n + kRowBlock - 1) / kRowBlock;
    partial.alloc(static_cast<size_t>(blocks) * H * H);
  }
  const double* hl(uint32_t l) const { return l ? h[l].p : x0.p; }

  void outer(const double* A, uint32_t p, const double* B, uint32_t q, double* out) {
    const uint32_t blocks = (n + kRowBlock - 1) / kRowBlock;
    GROOT_LAUNCH(tr_outer_partial_kernel, grid_for(static_cast<uint64_t>(blocks) * p * q), 256, 0, n, A, p, B, q,
                 partial.p);
    GROOT_LAUNCH(tr_reduce_partials_kernel, grid_for(p * q), 256, 0, blocks, p * q, partial.p, out);
  }

  void forward(const double* prm) {
    const uint32_t H = s.hidden;
    for (uint32_t l = 0; l < s.depth; ++l) {
      const uint32_t in = s.in_of(l);
      const double* ws = prm + s.layer_off(l);
      GROOT_LAUNCH(tr_agg_kernel, grid_for(static_cast<uint64_t>(n) * in), 256, 0, n, g->rp.p, g->col.p, hl(l), in, 0,
                   m[l].p);
      GROOT_LAUNCH(tr_dense_kernel, grid_for(static_cast<uint64_t>(n) * H), 256, 0, n, hl(l), m[l].p, in, H, ws,
                   ws + in * H, ws + 2 * in * H, z[l].p, h[l + 1].p);
    }
    const double* wo = prm + s.layer_off(s.depth);
    GROOT_LAUNCH(tr_head_kernel, grid_for(static_cast<uint64_t>(n) * s.classes), 256, 0, n, h[s.depth].p, H,
                 s.classes, wo, wo + H * s.classes, logits.p);
  }

  void loss_and_grads(const double* prm, double* grad, double* loss, double* acc) {
    const uint32_t H = s.hidden, C = s.classes;
    forward(prm);
    GROOT_LAUNCH(tr_softmax_kernel, grid_for(n), 256, 0, n, C, logits.p, g->labels.p, rloss.p, rhit.p, dl.p);
    GROOT_LAUNCH(tr_loss_kernel, 1, 32, 0, n, rloss.p, rhit.p, loss, acc);
    const uint64_t oo = s.layer_off(s.depth);
    outer(h[s.depth].p, H, dl.p, C, grad + oo);             // W_out = h_L^T dl
    outer(nullptr, 1, dl.p, C, grad + oo + H * C);          // b_out = column sums
    const double* wo = prm + oo;
    GROOT_LAUNCH(tr_back_head_kernel, grid_for(static_cast<uint64_t>(n) * H), 256, 0, n, dl.p, C, H, wo, dh.p);
    for (uint32_t l = s.depth; l-- > 0;) {
      const uint32_t in = s.in_of(l);
      const uint64_t off = s.layer_off(l);
      GROOT_LAUNCH(tr_relu_mask_kernel, grid_for(static_cast<uint64_t>(n) * H), 256, 0, static_cast<uint64_t>(n) * H,
                   z[l].p, dh.p, dz.p);
      outer(hl(l), in, dz.p, H, grad + off);                // W_self = h_l^T dz
      outer(m[l].p, in, dz.p, H, grad + off + in * H);      // W_neigh = m_l^T dz
      outer(nullptr, 1, dz.p, H, grad + off + 2 * in * H);  // bias = column sums
      if (l > 0) {
        const double* ws = prm + off;
        GROOT_LAUNCH(tr_back_layer_kernel, grid_for(static_cast<uint64_t>(n) * in), 256, 0, n, dz.p, H, in, ws,
                     ws + in * H, a1.p, a2.p);
        GROOT_LAUNCH(tr_agg_kernel, grid_for(static_cast<uint64_t>(n) * in), 256, 0, n, g->rp.p, g->col.p, a2.p, in, 1,
                     t.p);
        GROOT_LAUNCH(tr_add_kernel, grid_for(static_cast<uint64_t>(n) * in), 256, 0, static_cast<uint64_t>(n) * in, a1.p,
                     t.p, dh.p);
      }
    }
  }
};

}  // namespace

void init_model_params(uint64_t seed, uint32_t in_dim, uint32_t hidden, uint32_t classes, uint32_t depth, double* prm);

// train (src/gnn.cpp:211-255). init: NULL -> init_model(seed) (src/gnn.cpp:113-138).
void train_device(const groot_graph* g, uint32_t depth, uint32_t in_dim, uint32_t hidden, uint32_t classes,
                  uint32_t epochs, double lr, uint64_t seed, double b1, double b2, double eps, const double* init,
                  double* params_out, double* loss_out, double* acc_out) {
  require(lr > 0, "train: learning rate must be positive");
  require(in_dim == 4, "train: the device path supports in_dim 4");
  require(depth >= 1 && hidden >= 1 && hidden <= 64 && classes >= 1 && classes <= 8, "train: model shape unsupported");
  const Shape s{depth, in_dim, hidden, classes};
  const uint64_t np = s.count();
  std::vector<double> p0(np);
  if (init) std::copy(init, init + np, p0.begin());
  else init_model_params(seed, in_dim, hidden, classes, depth, p0.data());
  DevBuf<double> prm(np), grad(np), m1(np), m2(np), ld(2 * static_cast<size_t>(epochs ? epochs : 1));
  prm.upload(p0.data(), np);
  m1.zero();
  m2.zero();
  if (g->n == 0) fail(GROOT_EINVAL, "train: empty graph");
  Trainer tr(g, s);
  for (uint32_t ep = 1; ep <= epochs; ++ep) {
    tr.loss_and_grads(prm.p, grad.p, ld.p + 2 * (ep - 1), ld.p + 2 * (ep - 1) + 1);
    const double bc1 = 1.0 - std::pow(b1, ep), bc2 = 1.0 - std::pow(b2, ep);
    GROOT_LAUNCH(tr_adam_kernel, grid_for(np), 256, 0, np, prm.p, grad.p, m1.p, m2.p, lr, b1, b2, eps, bc1, bc2);
  }
  std::vector<double> h(2 * static_cast<size_t>(epochs));
  if (epochs) ld.download(h.data(), h.size());
  prm.download(params_out, np);
  stream_sync();
  for (uint32_t e = 0; e < epochs; ++e) {
    if (!std::isfinite(h[2 * e])) fail(GROOT_ERUNTIME, "train: loss diverged (non-finite)");
    if (loss_out) loss_out[e] = h[2 * e];
    if (acc_out) acc_out[e] = h[2 * e + 1];
  }
}

// loss_and_grads (src/gnn.cpp:180-209) for a given parameter vector.
double loss_and_grads_device(const groot_graph* g, uint32_t depth, uint32_t in_dim, uint32_t hidden, uint32_t classes,
                             const double* params, double* grads_out) {
  require(in_dim == 4, "train: the device path supports in_dim 4");
  require(depth >= 1 && hidden >= 1 && hidden <= 64 && classes >= 1 && classes <= 8, "train: model shape unsupported");
  if (g->n == 0) fail(GROOT_EINVAL, "train: empty graph");
  const Shape s{depth, in_dim, hidden, classes};
  const uint64_t np = s.count();
  DevBuf<double> prm(np), grad(np), ld(2);
  prm.upload(params, np);
  Trainer tr(g, s);
  tr.loss_and_grads(prm.p, grad.p, ld.p, ld.p + 1);
  double h[2];
  ld.download(h, 2);
  if (grads_out) grad.download(grads_out, np);
  stream_sync();
  return h[0];
}

}  // namespace groot
