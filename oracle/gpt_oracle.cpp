// =============================================================================
// TEST INFRASTRUCTURE ONLY -- fp64 CPU restatement of the TMP transformer
// layer stack (the parity oracle). Only tests/, __graft_entry__.smoke() and
// bench.py's cpu_baseline leg may load this library; the product library never
// links or calls it.
//
// Parity pinning: with attention, LayerNorm, biases, residual and dropout all
// disabled, a 1-layer FFN-only stack IS the reference toy checker, and this
// file reproduces it bit-for-bit:
//   matmul            i-k-j loop with zero skip      proj/src/numerics.cpp:13-24
//   transpose/add/hadamard                            numerics.cpp:26-46
//   gelu / gelu_grad  exact erf, same expression      numerics.cpp:50-55
//   random init       mt19937 + U(-s, s), draw order  numerics.cpp:57-62,136-154
//   forward           z = sum_i gelu(X W_in[i]) W_out[i] (literal sum, worker order)
//                                                     numerics.cpp:158-165
//   loss head         1/2 sum gelu(z)^2, gelu(z)gelu'(z)  numerics.cpp:175-188
//   backward          replayed pre/y, dW_out, dy, dpre, dW_in, dX += ...
//                                                     numerics.cpp:192-210
// tests/golden/toy_*.json (made by oracle/ref_dump.cpp from the reference
// itself) pin that reduction exactly. The extra ops (LN, causal softmax
// attention, biases, bias-dropout-residual, Philox dropout) are parity
// UNPINNED by the reference (it has none, numerics.hpp:37-44); they follow the
// same conventions and are cross-checked against torch.float64 autograd in
// tests/test_oracle.py.
//
// Layout conventions (per TMP worker r of t):
//   block 2l (attention): LN gamma/beta [h]; W_COL [h x 3h/t] columns
//     [Q heads of r | K heads of r | V heads of r], each head d = h/a wide;
//     B_COL [3h/t]; W_ROW [h/t x h]; B_ROW [h] (replicated)
//   block 2l+1 (FFN): LN; W_COL [h x f/t]; B_COL [f/t]; W_ROW [f/t x h]; B_ROW [h]
//   activations: tokens row-major [batch*seq x h], sample-major.
//   x_0 = input; x_{b+1} = (res ? x_b : 0) + dropout(sum_r partial_r + B_ROW)
//   loss = 1/2 sum gelu(x_B)^2.
// Dropout keys: offset = (block*2 + sub_batch)*4 + kind (kind 0 hidden,
//   1 attention); element index local to the sub-batch tensor; attention uses
//   the GLOBAL head index so the mask is TMP-degree invariant.
// =============================================================================
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <random>
#include <vector>

#include "philox.h"

namespace {

struct Mat {
  int rows = 0, cols = 0;
  std::vector<double> d;
  Mat() = default;
  Mat(int r, int c) : rows(r), cols(c), d(static_cast<size_t>(r) * c, 0.0) {}
  double& at(int r, int c) { return d[static_cast<size_t>(r) * cols + c]; }
  double at(int r, int c) const { return d[static_cast<size_t>(r) * cols + c]; }
};

// numerics.cpp:13-24: c[i][j] = sum_k a[i][k] b[k][j], accumulated in
// ascending k with the terms of a[i][k] == 0 skipped. The blocking below
// (B packed into 8-column panels, row/column tiles in parallel, k-blocks in
// ascending order, a 4x8 register tile) changes WHICH element is updated when,
// but never the sequence of additions into any one element, so the result is
// bit-identical to the reference loop (pinned by tests/test_oracle.py against
// the reference's own tensors); -ffp-contract=off keeps mul and add separate.
// A row quad whose k-block holds a zero takes the select form of the skip.
typedef double v4d __attribute__((vector_size(32)));
typedef long long v4l __attribute__((vector_size(32)));

template <bool kSkip>
__attribute__((always_inline)) inline void mm_quad(const double* __restrict ar, int lda, const double* __restrict bp, double* __restrict c, int ldc,
                    int ncols, int k0, int k1) {
  alignas(32) double tmp[4][8] = {};
  for (int r = 0; r < 4; ++r)
    for (int t = 0; t < ncols; ++t) tmp[r][t] = c[static_cast<size_t>(r) * ldc + t];
  v4d a00, a01, a10, a11, a20, a21, a30, a31;
  std::memcpy(&a00, tmp[0], 32); std::memcpy(&a01, tmp[0] + 4, 32);
  std::memcpy(&a10, tmp[1], 32); std::memcpy(&a11, tmp[1] + 4, 32);
  std::memcpy(&a20, tmp[2], 32); std::memcpy(&a21, tmp[2] + 4, 32);
  std::memcpy(&a30, tmp[3], 32); std::memcpy(&a31, tmp[3] + 4, 32);
  for (int k = k0; k < k1; ++k) {
    v4d b0, b1;
    std::memcpy(&b0, bp + static_cast<size_t>(k) * 8, 32);
    std::memcpy(&b1, bp + static_cast<size_t>(k) * 8 + 4, 32);
#define OASES_ORACLE_ROW(R, A0, A1)                         \
  {                                                         \
    const double av = ar[static_cast<size_t>(R) * lda + k]; \
    const v4d avv = {av, av, av, av};                       \
    const v4d s0 = A0 + avv * b0, s1 = A1 + avv * b1;       \
    if (kSkip) {                                            \
      const long long kk = av != 0.0 ? -1LL : 0LL;          \
      const v4l m = {kk, kk, kk, kk};                       \
      A0 = m ? s0 : A0;                                     \
      A1 = m ? s1 : A1;                                     \
    } else {                                                \
      A0 = s0;                                              \
      A1 = s1;                                              \
    }                                                       \
  }
    OASES_ORACLE_ROW(0, a00, a01)
    OASES_ORACLE_ROW(1, a10, a11)
    OASES_ORACLE_ROW(2, a20, a21)
    OASES_ORACLE_ROW(3, a30, a31)
#undef OASES_ORACLE_ROW
  }
  std::memcpy(tmp[0], &a00, 32); std::memcpy(tmp[0] + 4, &a01, 32);
  std::memcpy(tmp[1], &a10, 32); std::memcpy(tmp[1] + 4, &a11, 32);
  std::memcpy(tmp[2], &a20, 32); std::memcpy(tmp[2] + 4, &a21, 32);
  std::memcpy(tmp[3], &a30, 32); std::memcpy(tmp[3] + 4, &a31, 32);
  for (int r = 0; r < 4; ++r)
    for (int t = 0; t < ncols; ++t) c[static_cast<size_t>(r) * ldc + t] = tmp[r][t];
}

// rows [i0, i1) x panels [p0, p1) x k in [k0, k1); bpk = packed B ([panel][K][8])
__attribute__((target_clones("avx2", "default")))
void mm_block(const double* __restrict a, int lda, const double* __restrict bpk, int K, double* __restrict c, int ldc,
              int ncol, int i0, int i1, int p0, int p1, int k0, int k1) {
  int i = i0;
  for (; i + 4 <= i1; i += 4) {
    const double* ar = a + static_cast<size_t>(i) * lda;
    bool zero = false;
    for (int r = 0; r < 4 && !zero; ++r)
      for (int k = k0; k < k1; ++k)
        if (ar[static_cast<size_t>(r) * lda + k] == 0.0) {
          zero = true;
          break;
        }
    for (int pnl = p0; pnl < p1; ++pnl) {
      const double* bp = bpk + static_cast<size_t>(pnl) * K * 8;
      double* cc = c + static_cast<size_t>(i) * ldc + pnl * 8;
      const int nc = std::min(8, ncol - pnl * 8);
      if (zero) mm_quad<true>(ar, lda, bp, cc, ldc, nc, k0, k1);
      else mm_quad<false>(ar, lda, bp, cc, ldc, nc, k0, k1);
    }
  }
  for (; i < i1; ++i)
    for (int k = k0; k < k1; ++k) {
      const double av = a[static_cast<size_t>(i) * lda + k];
      if (av == 0.0) continue;
      for (int pnl = p0; pnl < p1; ++pnl) {
        const double* bk = bpk + (static_cast<size_t>(pnl) * K + k) * 8;
        double* ci = c + static_cast<size_t>(i) * ldc + pnl * 8;
        const int nc = std::min(8, ncol - pnl * 8);
        for (int t = 0; t < nc; ++t) ci[t] += av * bk[t];
      }
    }
}

Mat matmul(const Mat& a, const Mat& b) {
  Mat c(a.rows, b.cols);
  const int K = a.cols, N = b.cols, np = (N + 7) / 8;
  const bool par = static_cast<long long>(a.rows) * K * N > 200000;
  std::vector<double> bpk(static_cast<size_t>(np) * K * 8, 0.0);
#pragma omp parallel for schedule(static) if (par)
  for (int pnl = 0; pnl < np; ++pnl)
    for (int k = 0; k < K; ++k)
      for (int t = 0; t < 8 && pnl * 8 + t < N; ++t)
        bpk[(static_cast<size_t>(pnl) * K + k) * 8 + t] = b.d[static_cast<size_t>(k) * N + pnl * 8 + t];
  constexpr int IB = 64, PB = 32, KB = 256;  // 64 rows x 256 columns x 256 k per task step
  const int nib = (a.rows + IB - 1) / IB, npb = (np + PB - 1) / PB;
#pragma omp parallel for collapse(2) schedule(dynamic) if (par)
  for (int ib = 0; ib < nib; ++ib)
    for (int pb = 0; pb < npb; ++pb) {
      const int i0 = ib * IB, i1 = std::min(a.rows, i0 + IB), p0 = pb * PB, p1 = std::min(np, p0 + PB);
      for (int k0 = 0; k0 < K; k0 += KB)
        mm_block(a.d.data(), K, bpk.data(), K, c.d.data(), N, N, i0, i1, p0, p1, k0, std::min(K, k0 + KB));
    }
  return c;
}

Mat transpose(const Mat& a) {
  Mat t(a.cols, a.rows);
#pragma omp parallel for schedule(static) if (static_cast<long long>(a.rows) * a.cols > 1000000)
  for (int i = 0; i < a.rows; ++i)
    for (int j = 0; j < a.cols; ++j) t.at(j, i) = a.at(i, j);
  return t;
}

Mat add(const Mat& a, const Mat& b) {
  Mat c = a;
  for (size_t i = 0; i < c.d.size(); ++i) c.d[i] += b.d[i];
  return c;
}

double gelu_s(double x) { return 0.5 * x * (1.0 + std::erf(x / std::sqrt(2.0))); }
double gelu_grad_s(double x) {
  const double phi = std::exp(-0.5 * x * x) / std::sqrt(2.0 * M_PI);
  return 0.5 * (1.0 + std::erf(x / std::sqrt(2.0))) + x * phi;
}

void fill_uniform(Mat& m, std::mt19937& rng, double scale) {
  std::uniform_real_distribution<double> dist(-scale, scale);
  for (double& v : m.d) v = dist(rng);
}

enum Param { LN_GAMMA = 0, LN_BETA = 1, W_COL = 2, B_COL = 3, W_ROW = 4, B_ROW = 5, NPARAM = 6 };

}  // namespace

extern "C" {

typedef struct {
  int hidden, ffn, heads, seq, batch, layers, tp;
  int use_attention, use_layernorm, use_bias, use_residual;
  float hidden_dropout, attention_dropout;
  double ln_eps;
  uint64_t seed;
} oracle_cfg;

}  // extern "C"

namespace {

struct WorkerBlock {
  Mat p[NPARAM], g[NPARAM];
  // forward activations kept for backward (the oracle keeps everything; the
  // GPU recomputes, which is value-identical)
  Mat ln_out, col_out, act, P, Pd;  // col_out = pre (FFN) / qkv (attention); act = gelu(pre) / ctx
};

struct BlockState {
  bool attention = false;
  std::vector<WorkerBlock> w;
  Mat ar;  // sum of partials (pre-bias)
};

struct Oracle {
  oracle_cfg cfg{};
  int nblocks = 0, T = 0, hs = 0, fs = 0, Ht = 0, dh = 0;
  std::vector<BlockState> blocks;
  std::vector<Mat> x;  // x_0 .. x_B
  Mat input, input_grad;
  double loss = 0.0;

  explicit Oracle(const oracle_cfg& c) : cfg(c) {
    nblocks = cfg.layers * (cfg.use_attention ? 2 : 1);
    T = cfg.batch * cfg.seq;
    hs = cfg.hidden / cfg.tp;
    fs = cfg.ffn / cfg.tp;
    Ht = cfg.heads / cfg.tp;
    dh = cfg.use_attention ? cfg.hidden / cfg.heads : 0;
    blocks.resize(nblocks);
    const int h = cfg.hidden;
    for (int b = 0; b < nblocks; ++b) {
      BlockState& bs = blocks[b];
      bs.attention = cfg.use_attention && (b % 2 == 0);
      bs.w.resize(cfg.tp);
      for (auto& wb : bs.w) {
        const int ncol = bs.attention ? 3 * hs : fs;
        const int nrow = bs.attention ? hs : fs;
        wb.p[LN_GAMMA] = Mat(1, h);
        wb.p[LN_BETA] = Mat(1, h);
        for (double& v : wb.p[LN_GAMMA].d) v = 1.0;
        wb.p[W_COL] = Mat(h, ncol);
        wb.p[B_COL] = Mat(1, ncol);
        wb.p[W_ROW] = Mat(nrow, h);
        wb.p[B_ROW] = Mat(1, h);
        for (int k = 0; k < NPARAM; ++k) wb.g[k] = Mat(wb.p[k].rows, wb.p[k].cols);
      }
    }
    input = Mat(T, h);
    input_grad = Mat(T, h);
    x.assign(nblocks + 1, Mat(T, h));
  }

  int half() const { return (cfg.batch % 2 == 0) ? cfg.batch / 2 : cfg.batch; }

  uint64_t offset(int block, int sb, int kind) const { return (static_cast<uint64_t>(block) * 2 + sb) * 4 + kind; }

  // ---------------------------------------------------------------- LayerNorm
  void ln_fwd(const Mat& xin, const Mat& g, const Mat& be, Mat& y) const {
    const int h = cfg.hidden;
    y = Mat(T, h);
#pragma omp parallel for schedule(static)
    for (int r = 0; r < T; ++r) {
      double mean = 0.0;
      for (int c = 0; c < h; ++c) mean += xin.at(r, c);
      mean /= h;
      double var = 0.0;
      for (int c = 0; c < h; ++c) var += (xin.at(r, c) - mean) * (xin.at(r, c) - mean);
      var /= h;
      const double rstd = 1.0 / std::sqrt(var + cfg.ln_eps);
      for (int c = 0; c < h; ++c) y.at(r, c) = (xin.at(r, c) - mean) * rstd * g.d[c] + be.d[c];
    }
  }
  void ln_bwd(const Mat& xin, const Mat& g, const Mat& dy, Mat& dx, Mat& dg, Mat& db) const {
    const int h = cfg.hidden;
    dx = Mat(T, h);
    Mat xhat(T, h);
    // rows in parallel; the parameter gradients are summed over rows in row
    // order afterwards (same per-element order as a serial row loop)
#pragma omp parallel for schedule(static)
    for (int r = 0; r < T; ++r) {
      double mean = 0.0;
      for (int c = 0; c < h; ++c) mean += xin.at(r, c);
      mean /= h;
      double var = 0.0;
      for (int c = 0; c < h; ++c) var += (xin.at(r, c) - mean) * (xin.at(r, c) - mean);
      var /= h;
      const double rstd = 1.0 / std::sqrt(var + cfg.ln_eps);
      double s1 = 0.0, s2 = 0.0;
      for (int c = 0; c < h; ++c) {
        const double xh = (xin.at(r, c) - mean) * rstd;
        xhat.at(r, c) = xh;
        const double gg = dy.at(r, c) * g.d[c];
        s1 += gg;
        s2 += gg * xh;
      }
      s1 /= h;
      s2 /= h;
      for (int c = 0; c < h; ++c) {
        const double xh = (xin.at(r, c) - mean) * rstd;
        dx.at(r, c) = rstd * (dy.at(r, c) * g.d[c] - s1 - xh * s2);
      }
    }
#pragma omp parallel for schedule(static)
    for (int c = 0; c < h; ++c)
      for (int r = 0; r < T; ++r) {
        dg.d[c] += dy.at(r, c) * xhat.at(r, c);
        db.d[c] += dy.at(r, c);
      }
  }

  // ---------------------------------------------------------------- attention
  // qkv [T x 3*Ht*dh] of worker r -> ctx [T x Ht*dh]; keeps P, Pd [batch*Ht*s x s]
  void attn_fwd(int block, int r, const Mat& qkv, Mat& ctx, Mat& P, Mat& Pd) const {
    const int s = cfg.seq, d = dh, H = cfg.heads;
    const double scale = 1.0 / std::sqrt(static_cast<double>(d));
    const float p = cfg.attention_dropout;
    const uint32_t thr = oracle::keep_threshold(p);
    const double ks = oracle::keep_scale(p);
    ctx = Mat(T, Ht * d);
    P = Mat(cfg.batch * Ht * s, s);
    Pd = Mat(cfg.batch * Ht * s, s);
#pragma omp parallel for collapse(2) schedule(static)
    for (int n = 0; n < cfg.batch; ++n)
      for (int jl = 0; jl < Ht; ++jl) {
        const int sb = n / half(), nl = n % half();
        const int jg = r * Ht + jl;
        std::vector<double> sc(s);
        for (int i = 0; i < s; ++i) {
          const int row = (n * Ht + jl) * s + i;
          double mx = -INFINITY;
          for (int j = 0; j <= i; ++j) {
            double acc = 0.0;
            for (int e = 0; e < d; ++e) acc += qkv.at(n * s + i, jl * d + e) * qkv.at(n * s + j, Ht * d + jl * d + e);
            sc[j] = acc * scale;
            mx = std::max(mx, sc[j]);
          }
          double sum = 0.0;
          for (int j = 0; j <= i; ++j) {
            sc[j] = std::exp(sc[j] - mx);
            sum += sc[j];
          }
          for (int j = 0; j <= i; ++j) {
            const double pv = sc[j] / sum;
            P.at(row, j) = pv;
            double pdv = pv;
            if (p > 0.f) {
              const uint64_t e = ((static_cast<uint64_t>(nl) * H + jg) * s + i) * static_cast<uint64_t>(s) + j;
              pdv = oracle::keep(cfg.seed, offset(block, sb, 1), e, thr) ? pv * ks : 0.0;
            }
            Pd.at(row, j) = pdv;
          }
          // ctx[i][e] = sum_{j<=i} Pd[i][j] V[j][e], ascending j per element (j outer for locality)
          std::vector<double> acc(d, 0.0);
          for (int j = 0; j <= i; ++j) {
            const double pj = Pd.at(row, j);
            const double* vj = &qkv.d[static_cast<size_t>(n * s + j) * qkv.cols + 2 * Ht * d + jl * d];
            for (int e = 0; e < d; ++e) acc[e] += pj * vj[e];
          }
          for (int e = 0; e < d; ++e) ctx.at(n * s + i, jl * d + e) = acc[e];
        }
      }
  }

  void attn_bwd(int block, const Mat& qkv, const Mat& P, const Mat& Pd, const Mat& dctx, Mat& dqkv) const {
    const int s = cfg.seq, d = dh;
    const double scale = 1.0 / std::sqrt(static_cast<double>(d));
    const float p = cfg.attention_dropout;
    const uint32_t thr = oracle::keep_threshold(p);
    const double ks = oracle::keep_scale(p);
    const int H = cfg.heads;
    (void)H;
    dqkv = Mat(T, 3 * Ht * d);
    const int r = worker_of_current;
#pragma omp parallel for collapse(2) schedule(static)
    for (int n = 0; n < cfg.batch; ++n)
      for (int jl = 0; jl < Ht; ++jl) {
        const int sb = n / half(), nl = n % half();
        const int jg = r * Ht + jl;
        std::vector<double> dP(s), dS(static_cast<size_t>(s) * s, 0.0);
        for (int i = 0; i < s; ++i) {
          const int row = (n * Ht + jl) * s + i;
          double dot = 0.0;
          for (int j = 0; j <= i; ++j) {
            double acc = 0.0;
            for (int e = 0; e < d; ++e) acc += dctx.at(n * s + i, jl * d + e) * qkv.at(n * s + j, 2 * Ht * d + jl * d + e);
            if (p > 0.f) {
              const uint64_t el = ((static_cast<uint64_t>(nl) * cfg.heads + jg) * s + i) * static_cast<uint64_t>(s) + j;
              acc = oracle::keep(cfg.seed, offset(block, sb, 1), el, thr) ? acc * ks : 0.0;
            }
            dP[j] = acc;
            dot += P.at(row, j) * acc;
          }
          for (int j = 0; j <= i; ++j) dS[static_cast<size_t>(i) * s + j] = scale * P.at(row, j) * (dP[j] - dot);
        }
        // loop orders below keep every element's summation order (ascending j for dQ,
        // ascending i for dK/dV) with the reduction index outside the e loop
        std::vector<double> dq(d), dk(d), dv(d);
        for (int i = 0; i < s; ++i) {
          std::fill(dq.begin(), dq.end(), 0.0);
          for (int j = 0; j <= i; ++j) {
            const double sij = dS[static_cast<size_t>(i) * s + j];
            const double* kj = &qkv.d[static_cast<size_t>(n * s + j) * qkv.cols + Ht * d + jl * d];
            for (int e = 0; e < d; ++e) dq[e] += sij * kj[e];
          }
          for (int e = 0; e < d; ++e) dqkv.at(n * s + i, jl * d + e) = dq[e];
        }
        for (int j = 0; j < s; ++j) {
          std::fill(dk.begin(), dk.end(), 0.0);
          std::fill(dv.begin(), dv.end(), 0.0);
          for (int i = j; i < s; ++i) {
            const double sij = dS[static_cast<size_t>(i) * s + j];
            const double pij = Pd.at((n * Ht + jl) * s + i, j);
            const double* qi = &qkv.d[static_cast<size_t>(n * s + i) * qkv.cols + jl * d];
            const double* oi = &dctx.d[static_cast<size_t>(n * s + i) * dctx.cols + jl * d];
            for (int e = 0; e < d; ++e) {
              dk[e] += sij * qi[e];
              dv[e] += pij * oi[e];
            }
          }
          for (int e = 0; e < d; ++e) {
            dqkv.at(n * s + j, Ht * d + jl * d + e) = dk[e];
            dqkv.at(n * s + j, 2 * Ht * d + jl * d + e) = dv[e];
          }
        }
      }
  }
  int worker_of_current = 0;

  // ---------------------------------------------------------------- dropout helpers
  // out = (res ? res : 0) + dropout(in + bias)
  void bdr_fwd(int block, const Mat& in, const Mat* bias, const Mat* res, Mat& out) const {
    const int h = cfg.hidden, s = cfg.seq;
    const float p = cfg.hidden_dropout;
    const uint32_t thr = oracle::keep_threshold(p);
    const double ks = oracle::keep_scale(p);
    out = Mat(T, h);
#pragma omp parallel for schedule(static)
    for (int r = 0; r < T; ++r) {
      const int n = r / s, sb = n / half();
      const uint64_t rl = static_cast<uint64_t>(r - sb * half() * s);
      for (int c = 0; c < h; ++c) {
        double v = in.at(r, c);
        if (bias) v += bias->d[c];
        if (p > 0.f) v = oracle::keep(cfg.seed, offset(block, sb, 0), rl * h + c, thr) ? v * ks : 0.0;
        out.at(r, c) = res ? res->at(r, c) + v : v;
      }
    }
  }
  void dropout_bwd(int block, const Mat& g, Mat& out) const {
    const int h = cfg.hidden, s = cfg.seq;
    const float p = cfg.hidden_dropout;
    out = g;
    if (!(p > 0.f)) return;
    const uint32_t thr = oracle::keep_threshold(p);
    const double ks = oracle::keep_scale(p);
#pragma omp parallel for schedule(static)
    for (int r = 0; r < T; ++r) {
      const int n = r / s, sb = n / half();
      const uint64_t rl = static_cast<uint64_t>(r - sb * half() * s);
      for (int c = 0; c < h; ++c)
        out.at(r, c) = oracle::keep(cfg.seed, offset(block, sb, 0), rl * h + c, thr) ? g.at(r, c) * ks : 0.0;
    }
  }

  // ---------------------------------------------------------------- full step
  void forward() {
    x[0] = input;
    for (int b = 0; b < nblocks; ++b) {
      BlockState& bs = blocks[b];
      Mat ar(T, cfg.hidden);
      for (int r = 0; r < cfg.tp; ++r) {
        WorkerBlock& wb = bs.w[r];
        if (cfg.use_layernorm) ln_fwd(x[b], wb.p[LN_GAMMA], wb.p[LN_BETA], wb.ln_out);
        else wb.ln_out = x[b];
        wb.col_out = matmul(wb.ln_out, wb.p[W_COL]);
        if (cfg.use_bias)
          for (int i = 0; i < T; ++i)
            for (int c = 0; c < wb.col_out.cols; ++c) wb.col_out.at(i, c) += wb.p[B_COL].d[c];
        if (bs.attention) {
          attn_fwd(b, r, wb.col_out, wb.act, wb.P, wb.Pd);
        } else {
          wb.act = wb.col_out;
#pragma omp parallel for schedule(static)
          for (size_t i = 0; i < wb.act.d.size(); ++i) wb.act.d[i] = gelu_s(wb.act.d[i]);
        }
        ar = add(ar, matmul(wb.act, wb.p[W_ROW]));  // the literal in-process AllReduce
      }
      bs.ar = ar;
      const Mat* bias = cfg.use_bias ? &bs.w[0].p[B_ROW] : nullptr;
      const Mat* res = cfg.use_residual ? &x[b] : nullptr;
      if (!bias && !res && !(cfg.hidden_dropout > 0.f)) x[b + 1] = ar;
      else bdr_fwd(b, ar, bias, res, x[b + 1]);
    }
  }

  void backward() {
    const Mat& z = x[nblocks];
    loss = 0.0;
    for (double v : z.d) {
      const double g = gelu_s(v);
      loss += 0.5 * g * g;
    }
    Mat g = z;  // dL/dx_B
    for (double& v : g.d) v = gelu_s(v) * gelu_grad_s(v);
    for (auto& bs : blocks)
      for (auto& wb : bs.w)
        for (auto& m : wb.g) std::fill(m.d.begin(), m.d.end(), 0.0);
    for (int b = nblocks - 1; b >= 0; --b) {
      BlockState& bs = blocks[b];
      Mat g_ar;
      dropout_bwd(b, g, g_ar);
      if (cfg.use_bias) {
        for (int r = 0; r < cfg.tp; ++r)
          for (int i = 0; i < T; ++i)
            for (int c = 0; c < cfg.hidden; ++c) bs.w[r].g[B_ROW].d[c] += g_ar.at(i, c);
      }
      Mat dln(T, cfg.hidden);
      for (int r = 0; r < cfg.tp; ++r) {
        WorkerBlock& wb = bs.w[r];
        wb.g[W_ROW] = add(wb.g[W_ROW], matmul(transpose(wb.act), g_ar));
        const Mat du = matmul(g_ar, transpose(wb.p[W_ROW]));
        Mat dcol;
        if (bs.attention) {
          worker_of_current = r;
          attn_bwd(b, wb.col_out, wb.P, wb.Pd, du, dcol);
        } else {
          dcol = du;
#pragma omp parallel for schedule(static)
          for (size_t i = 0; i < dcol.d.size(); ++i) dcol.d[i] *= gelu_grad_s(wb.col_out.d[i]);
        }
        if (cfg.use_bias)
          for (int i = 0; i < T; ++i)
            for (int c = 0; c < dcol.cols; ++c) wb.g[B_COL].d[c] += dcol.at(i, c);
        wb.g[W_COL] = add(wb.g[W_COL], matmul(transpose(wb.ln_out), dcol));
        dln = add(dln, matmul(dcol, transpose(wb.p[W_COL])));  // the f-backward AllReduce
      }
      Mat dx;
      if (cfg.use_layernorm) {
        Mat dg(1, cfg.hidden), db(1, cfg.hidden);
        ln_bwd(x[b], bs.w[0].p[LN_GAMMA], dln, dx, dg, db);
        for (int r = 0; r < cfg.tp; ++r) {
          bs.w[r].g[LN_GAMMA] = dg;
          bs.w[r].g[LN_BETA] = db;
        }
      } else {
        dx = dln;
      }
      g = cfg.use_residual ? add(g, dx) : dx;
    }
    input_grad = g;
  }
};

}  // namespace

extern "C" {

void* oracle_create(const oracle_cfg* cfg) {
  if (!cfg || cfg->tp < 1 || cfg->ffn % cfg->tp || cfg->batch < 1 || cfg->seq < 1 ||
      cfg->layers < 0)
    return nullptr;
  if (cfg->use_attention && (cfg->heads < 1 || cfg->hidden % cfg->heads || cfg->heads % cfg->tp || cfg->hidden % cfg->tp))
    return nullptr;
  return new Oracle(*cfg);
}
void oracle_destroy(void* o) { delete static_cast<Oracle*>(o); }
int oracle_num_blocks(void* o) { return static_cast<Oracle*>(o)->nblocks; }
int oracle_block_is_attention(void* o, int b) { return static_cast<Oracle*>(o)->blocks[b].attention ? 1 : 0; }

long long oracle_param_numel(void* o, int block, int param) {
  auto* s = static_cast<Oracle*>(o);
  return static_cast<long long>(s->blocks[block].w[0].p[param].d.size());
}
int oracle_param_rows(void* o, int block, int param) {
  return static_cast<Oracle*>(o)->blocks[block].w[0].p[param].rows;
}
double* oracle_param(void* o, int worker, int block, int param) {
  return static_cast<Oracle*>(o)->blocks[block].w[worker].p[param].d.data();
}
double* oracle_grad(void* o, int worker, int block, int param) {
  return static_cast<Oracle*>(o)->blocks[block].w[worker].g[param].d.data();
}
double* oracle_input(void* o) { return static_cast<Oracle*>(o)->input.d.data(); }
double* oracle_input_grad(void* o) { return static_cast<Oracle*>(o)->input_grad.d.data(); }
double* oracle_activation(void* o, int block) { return static_cast<Oracle*>(o)->x[block].d.data(); }
double oracle_loss(void* o) { return static_cast<Oracle*>(o)->loss; }

// mt19937 draws in the toy's order (numerics.cpp:142-152): input U(-1,1), then
// per block per worker W_COL U(+-1/sqrt(fan_in)), W_ROW U(+-1/sqrt(fan_in)).
// With `extras`, LN gamma = 1 + U(+-0.1), beta/biases U(+-0.1) are drawn
// afterwards (so the weight draws stay the toy's).
void oracle_init_params(void* o, unsigned seed, int extras) {
  auto* s = static_cast<Oracle*>(o);
  std::mt19937 rng(seed);
  fill_uniform(s->input, rng, 1.0);
  for (auto& bs : s->blocks) {
    for (auto& wb : bs.w) {
      fill_uniform(wb.p[W_COL], rng, 1.0 / std::sqrt(static_cast<double>(s->cfg.hidden)));
      const int fan_in_row = bs.attention ? s->cfg.hidden : s->cfg.ffn;
      fill_uniform(wb.p[W_ROW], rng, 1.0 / std::sqrt(static_cast<double>(fan_in_row)));
    }
  }
  if (extras) {
    for (auto& bs : s->blocks) {
      Mat gam(1, s->cfg.hidden), bet(1, s->cfg.hidden), brow(1, s->cfg.hidden);
      fill_uniform(gam, rng, 0.1);
      for (double& v : gam.d) v += 1.0;
      fill_uniform(bet, rng, 0.1);
      fill_uniform(brow, rng, 0.1);
      for (auto& wb : bs.w) {
        wb.p[LN_GAMMA] = gam;
        wb.p[LN_BETA] = bet;
        wb.p[B_ROW] = brow;
        fill_uniform(wb.p[B_COL], rng, 0.1);
      }
    }
  }
}

void oracle_run(void* o) {
  auto* s = static_cast<Oracle*>(o);
  s->forward();
  s->backward();
}

}  // extern "C"
