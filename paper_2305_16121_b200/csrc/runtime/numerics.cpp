// The reference's value-level checker API (proj/include/tmpsim/numerics.hpp:10-60,
// proj/src/numerics.cpp) computed on the B200.
//
//  * Matrix primitives: f64 device kernels with the reference's scalar
//    arithmetic (numerics_f64.cu, and the f64 instantiation of the FMA-pipe
//    GEMM, whose k-ascending, zero-skipping, unfused accumulation is the
//    reference's i-k-j loop).
//  * make_toy_sharded_model: the reference's mt19937 draws (numerics.cpp:136-154)
//    -- input generation, kept bit-identical so both sides see the same model.
//  * sharded_output_deviation / recompute_elision_equivalence: the toy is an
//    f64 FFN block (column GEMM + GeLU, row GEMM, literal worker-order
//    AllReduce, 1/2 sum gelu(z)^2 loss head) run by this build's runtime --
//    Stack + plan Executor, `workers` TMP ranks in-process. The elision check
//    runs the CrossPass plan (recompute replays the block with its AllReduce)
//    and the Oases plan (recompute elided, Eq. 1) and compares every gradient.
//  * allreduce_grad_identity: the literal AllReduce and phi on the device; the
//    backward of the AllReduce is the identity the runtime's backward f uses.
#include <cmath>
#include <memory>
#include <random>

#include "../kernels/gemm.h"
#include "../kernels/kernels.h"
#include "oases/tmpsim.hpp"
#include "stack.h"
#include "status.h"

namespace tmpsim {

namespace {

using oases::check_cuda;

void need_device() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    throw oases::CudaError("no CUDA device: the value-level numerics run on the GPU (no CPU fallback)");
  }
}

// one device f64 buffer
struct Dev {
  double* p = nullptr;
  size_t n = 0;
  explicit Dev(size_t count) : n(count) {
    check_cuda(cudaMalloc(&p, std::max<size_t>(1, n) * sizeof(double)), "cudaMalloc");
  }
  Dev(const Matrix& m) : Dev(m.data.size()) { up(m.data.data()); }
  ~Dev() { cudaFree(p); }
  Dev(const Dev&) = delete;
  Dev& operator=(const Dev&) = delete;
  void up(const double* h) {
    if (n) check_cuda(cudaMemcpy(p, h, n * sizeof(double), cudaMemcpyHostToDevice), "H2D");
  }
  void down(double* h) const {
    check_cuda(cudaDeviceSynchronize(), "sync");
    if (n) check_cuda(cudaMemcpy(h, p, n * sizeof(double), cudaMemcpyDeviceToHost), "D2H");
  }
};

Matrix to_host(const Dev& d, int rows, int cols) {
  Matrix m(rows, cols);
  d.down(m.data.data());
  return m;
}

Matrix map_op(int op, const Matrix& a, const Matrix* b, const char* name) {
  if (b && (a.rows != b->rows || a.cols != b->cols)) throw ConfigError(std::string(name) + ": shape mismatch");
  need_device();
  Dev da(a);
  std::unique_ptr<Dev> db;
  if (b) db = std::make_unique<Dev>(*b);
  Dev out(a.data.size());
  if (!a.data.empty())
    check_cuda(oases::map_f64(op, da.p, db ? db->p : nullptr, out.p, static_cast<long long>(a.data.size()), nullptr),
               name);
  return to_host(out, a.rows, a.cols);
}

Matrix random_matrix(int rows, int cols, std::mt19937& rng, double scale) {
  std::uniform_real_distribution<double> dist(-scale, scale);
  Matrix m(rows, cols);
  for (double& v : m.data) v = dist(rng);
  return m;
}

// ---------------------------------------------------------------- toy on the runtime
// A ToyShardedModel as an f64 FFN-only block stack: hidden = model_dim, ffn =
// hidden_dim, seq 1, the batch padded to an even row count (two sub-batches)
// with zero rows, which contribute exactly nothing (gelu(0) = 0, so their
// output, loss term and gradient rows are 0).
struct ToyRun {
  std::unique_ptr<oases::Context> ctx;
  std::unique_ptr<oases::Stack> stack;
  int rows = 0, rows_padded = 0, model_dim = 0, workers = 1;
};

ToyRun make_toy_run(int workers, int rows, int model_dim, int hidden_dim) {
  need_device();
  if (workers > 8) throw ConfigError("toy model: at most 8 in-process workers on one device");
  ToyRun r;
  r.rows = rows;
  r.rows_padded = rows + (rows % 2);
  r.model_dim = model_dim;
  r.workers = workers;
  oases_ctx_desc d{};
  d.tp = workers;
  d.rank = 0;
  int dev = 0;
  check_cuda(cudaGetDevice(&dev), "cudaGetDevice");
  d.device = dev;
  d.local_workers = workers;
  r.ctx = oases::make_context(d);
  oases::ModelCfg c;
  c.h = model_dim;
  c.f = hidden_dim;
  c.heads = 1;
  c.s = 1;
  c.b = r.rows_padded;
  c.layers = 1;
  c.bytes = 8;
  c.recompute = true;
  c.attention = c.ln = c.bias = c.residual = false;
  r.stack = std::make_unique<oases::Stack>(*r.ctx, c);
  return r;
}

void upload_toy(ToyRun& r, const Matrix& input, const std::vector<Matrix>& w_in, const std::vector<Matrix>& w_out) {
  for (int i = 0; i < r.workers; ++i) {
    r.stack->set_param(i, 0, OASES_P_W_COL, w_in[static_cast<size_t>(i)].data.data());
    r.stack->set_param(i, 0, OASES_P_W_ROW, w_out[static_cast<size_t>(i)].data.data());
  }
  std::vector<double> x(static_cast<size_t>(r.rows_padded) * r.model_dim, 0.0);
  std::copy(input.data.begin(), input.data.end(), x.begin());
  r.stack->set_input(x.data(), OASES_F64, r.ctx->compute);
  check_cuda(cudaStreamSynchronize(r.ctx->compute), "set_input");
}

ModelGraph toy_graph(int batch_padded, int model_dim) {
  ModelSpec spec;
  spec.hidden_size = model_dim;
  spec.num_layers = 1;
  spec.seq_len = 1;
  spec.attention_heads = 1;
  spec.global_batch = batch_padded;
  spec.bytes_per_element = 8;
  spec.recompute_enabled = true;
  return build_block_graph(build_ffn_sequence(spec), spec);
}

struct ToyGrads {
  double loss = 0.0;
  Matrix input;
  std::vector<Matrix> w_in, w_out;
};

ToyGrads run_plan(ToyRun& r, const SchedulePlan& plan, const ToyShardedModel& m) {
  oases::Executor ex(*r.stack, plan);
  const SimResult res = ex.step(false);
  (void)res;
  ToyGrads g;
  g.loss = r.stack->read_loss();
  std::vector<double> dx(static_cast<size_t>(r.rows_padded) * r.model_dim);
  r.stack->get_input_grad(dx.data());
  g.input = Matrix(r.rows, r.model_dim);
  std::copy(dx.begin(), dx.begin() + static_cast<std::ptrdiff_t>(g.input.data.size()), g.input.data.begin());
  for (int i = 0; i < r.workers; ++i) {
    Matrix wi(m.w_in[static_cast<size_t>(i)].rows, m.w_in[static_cast<size_t>(i)].cols);
    Matrix wo(m.w_out[static_cast<size_t>(i)].rows, m.w_out[static_cast<size_t>(i)].cols);
    r.stack->get_grad(i, 0, OASES_P_W_COL, wi.data.data());
    r.stack->get_grad(i, 0, OASES_P_W_ROW, wo.data.data());
    g.w_in.push_back(std::move(wi));
    g.w_out.push_back(std::move(wo));
  }
  return g;
}

// the stack's output x_B = the AllReduce output z (no bias / residual / dropout)
Matrix forward_output(ToyRun& r) {
  oases::Executor ex(*r.stack, schedule_oases(toy_graph(r.rows_padded, r.model_dim)));
  ex.step(false);
  Matrix z(r.rows, r.model_dim);
  std::vector<double> half(static_cast<size_t>(r.rows_padded / 2) * r.model_dim);
  const int nb = r.stack->num_blocks();
  size_t at = 0;
  for (int sb = 0; sb < 2; ++sb) {
    r.stack->get_activation(0, nb, sb, half.data());
    for (double v : half)
      if (at < z.data.size()) z.data[at++] = v;
  }
  return z;
}

void check_model(const ToyShardedModel& m) {
  if (m.workers < 1 || static_cast<int>(m.w_in.size()) != m.workers || static_cast<int>(m.w_out.size()) != m.workers)
    throw ConfigError("toy model: one w_in / w_out shard per worker");
  for (int i = 0; i < m.workers; ++i) {
    const Matrix& wi = m.w_in[static_cast<size_t>(i)];
    const Matrix& wo = m.w_out[static_cast<size_t>(i)];
    if (wi.rows != m.input.cols || wo.cols != m.input.cols || wi.cols != wo.rows ||
        wi.cols != m.w_in.front().cols)
      throw ConfigError("toy model: shard shapes do not match the input");
  }
}

}  // namespace

// ---------------------------------------------------------------- primitives
Matrix matmul(const Matrix& a, const Matrix& b) {
  if (a.cols != b.rows) throw ConfigError("matmul: shape mismatch");
  Matrix c(a.rows, b.cols);
  if (c.data.empty()) return c;
  if (a.cols == 0) return c;
  need_device();
  Dev da(a), db(b), dc(c.data.size());
  oases_gemm_desc d{};
  d.dtype = OASES_F64;
  d.c_dtype = OASES_F64;
  d.M = a.rows;
  d.N = b.cols;
  d.K = a.cols;
  d.batch = d.batch_inner = 1;
  d.a.ptr = da.p;
  d.a.rows = a.rows;
  d.a.cols = a.cols;
  d.a.ld = a.cols;
  d.a.mn_major = 0;
  d.b.ptr = db.p;  // B stored [K][N]: N contiguous = MN-major
  d.b.rows = b.rows;
  d.b.cols = b.cols;
  d.b.ld = b.cols;
  d.b.mn_major = 1;
  d.c = dc.p;
  d.ldc = b.cols;
  d.alpha = 1.f;
  const oases::GemmStatus st = oases::gemm_simt(d, nullptr);
  if (!st.ok) {
    if (st.cuda) throw oases::CudaError(st.err);
    throw ConfigError(st.err);
  }
  return to_host(dc, c.rows, c.cols);
}

Matrix transpose(const Matrix& a) {
  Matrix t(a.cols, a.rows);
  if (a.data.empty()) return t;
  need_device();
  Dev da(a), dt(a.data.size());
  check_cuda(oases::transpose_f64(da.p, dt.p, a.rows, a.cols, nullptr), "transpose");
  return to_host(dt, a.cols, a.rows);
}

Matrix add(const Matrix& a, const Matrix& b) { return map_op(oases::F64_ADD, a, &b, "add"); }
Matrix hadamard(const Matrix& a, const Matrix& b) { return map_op(oases::F64_HADAMARD, a, &b, "hadamard"); }
Matrix gelu(const Matrix& a) { return map_op(oases::F64_GELU, a, nullptr, "gelu"); }
Matrix gelu_grad(const Matrix& a) { return map_op(oases::F64_GELU_GRAD, a, nullptr, "gelu_grad"); }

double max_abs_diff(const Matrix& a, const Matrix& b) {
  if (a.rows != b.rows || a.cols != b.cols) throw ConfigError("max_abs_diff: shape mismatch");
  if (a.data.empty()) return 0.0;
  need_device();
  Dev da(a), db(b), out(1);
  check_cuda(oases::max_abs_diff_f64(da.p, db.p, static_cast<long long>(a.data.size()), out.p, nullptr),
             "max_abs_diff");
  double r = 0.0;
  out.down(&r);
  return r;
}

// ---------------------------------------------------------------- checks
GradIdentityCheck allreduce_grad_identity(int workers, int rows, int cols, unsigned seed) {
  if (workers < 1 || rows < 1 || cols < 1)
    throw ConfigError("allreduce_grad_identity: workers and shape must be positive");
  if (workers > 8) throw ConfigError("allreduce_grad_identity: at most 8 in-process workers on one device");
  need_device();
  std::mt19937 rng(seed);  // numerics.cpp:92-95 draw order
  std::vector<Matrix> inputs;
  for (int i = 0; i < workers; ++i) inputs.push_back(random_matrix(rows, cols, rng, 1.0));
  const Matrix weights = random_matrix(rows, cols, rng, 1.0);
  const int n = rows * cols;
  // worker buffers on the device, summed by the runtime's literal AllReduce kernel
  Dev xs(static_cast<size_t>(workers) * n), w(weights), y(static_cast<size_t>(workers) * n);
  for (int i = 0; i < workers; ++i)
    check_cuda(cudaMemcpy(xs.p + static_cast<size_t>(i) * n, inputs[static_cast<size_t>(i)].data.data(),
                          static_cast<size_t>(n) * sizeof(double), cudaMemcpyHostToDevice),
               "H2D");
  check_cuda(cudaMemcpy(y.p, xs.p, static_cast<size_t>(workers) * n * sizeof(double), cudaMemcpyDeviceToDevice), "D2D");
  std::vector<void*> bufs;
  for (int i = 0; i < workers; ++i) bufs.push_back(y.p + static_cast<size_t>(i) * n);
  check_cuda(oases::local_allreduce(OASES_F64, bufs.data(), workers, n, nullptr), "allreduce");
  // d phi / d y = w + y ; reverse mode through the sum hands every summand the same adjoint
  Dev grad_y(static_cast<size_t>(n)), grad_x(static_cast<size_t>(workers) * n), dev(1);
  check_cuda(oases::map_f64(oases::F64_ADD, w.p, y.p, grad_y.p, n, nullptr), "grad_y");
  for (int i = 0; i < workers; ++i)
    check_cuda(cudaMemcpy(grad_x.p + static_cast<size_t>(i) * n, grad_y.p, static_cast<size_t>(n) * sizeof(double),
                          cudaMemcpyDeviceToDevice),
               "adjoint");
  GradIdentityCheck check;
  Dev fd(static_cast<size_t>(workers) * n);
  check_cuda(oases::grad_identity_fd_f64(xs.p, w.p, workers, n, 1e-5, fd.p, nullptr), "finite differences");
  for (int i = 0; i < workers; ++i) {
    double a = 0.0, f = 0.0;
    check_cuda(oases::max_abs_diff_f64(grad_x.p + static_cast<size_t>(i) * n, grad_y.p, n, dev.p, nullptr), "dev");
    dev.down(&a);
    check_cuda(oases::max_abs_diff_f64(fd.p + static_cast<size_t>(i) * n, grad_y.p, n, dev.p, nullptr), "dev");
    dev.down(&f);
    check.autodiff_deviation = std::max(check.autodiff_deviation, a);
    check.finite_difference_deviation = std::max(check.finite_difference_deviation, f);
  }
  return check;
}

ToyShardedModel make_toy_sharded_model(int workers, int batch, int model_dim, int hidden_dim, unsigned seed) {
  if (workers < 1 || batch < 1 || model_dim < 1 || hidden_dim < workers || hidden_dim % workers != 0)
    throw ConfigError("toy model: hidden_dim must be a positive multiple of workers");
  std::mt19937 rng(seed);  // numerics.cpp:142-152 draw order
  ToyShardedModel model;
  model.workers = workers;
  model.input = random_matrix(batch, model_dim, rng, 1.0);
  const int shard = hidden_dim / workers;
  const double s_in = 1.0 / std::sqrt(static_cast<double>(model_dim));
  const double s_out = 1.0 / std::sqrt(static_cast<double>(hidden_dim));
  for (int i = 0; i < workers; ++i) {
    model.w_in.push_back(random_matrix(model_dim, shard, rng, s_in));
    model.w_out.push_back(random_matrix(shard, model_dim, rng, s_out));
  }
  return model;
}

double sharded_output_deviation(const ToyShardedModel& m) {
  check_model(m);
  const int shard = m.w_in.front().cols, hidden = shard * m.workers;
  // TMP = workers (partials summed by the runtime's AllReduce) ...
  ToyRun sharded = make_toy_run(m.workers, m.input.rows, m.input.cols, hidden);
  upload_toy(sharded, m.input, m.w_in, m.w_out);
  const Matrix z = forward_output(sharded);
  // ... vs TMP = 1 on the concatenated (unsharded) weights
  Matrix w_in_full(m.input.cols, hidden), w_out_full(hidden, m.w_out.front().cols);
  for (int i = 0; i < m.workers; ++i) {
    for (int r = 0; r < m.w_in[static_cast<size_t>(i)].rows; ++r)
      for (int c = 0; c < shard; ++c) w_in_full.at(r, i * shard + c) = m.w_in[static_cast<size_t>(i)].at(r, c);
    for (int r = 0; r < shard; ++r)
      for (int c = 0; c < m.w_out[static_cast<size_t>(i)].cols; ++c)
        w_out_full.at(i * shard + r, c) = m.w_out[static_cast<size_t>(i)].at(r, c);
  }
  ToyRun full = make_toy_run(1, m.input.rows, m.input.cols, hidden);
  upload_toy(full, m.input, {w_in_full}, {w_out_full});
  const Matrix z_full = forward_output(full);
  return max_abs_diff(z_full, z);
}

ElisionCheck recompute_elision_equivalence(const ToyShardedModel& m) {
  check_model(m);
  const int hidden = m.w_in.front().cols * m.workers;
  ToyRun run = make_toy_run(m.workers, m.input.rows, m.input.cols, hidden);
  upload_toy(run, m.input, m.w_in, m.w_out);
  const ModelGraph g = toy_graph(run.rows_padded, m.input.cols);
  // full replay: recompute reruns the block including its AllReduce (CrossPass)
  const ToyGrads full = run_plan(run, schedule_cross_pass(g), m);
  // elided replay: recompute restarts from the stored post-AllReduce tensor (Oases)
  const ToyGrads elided = run_plan(run, schedule_oases(g), m);
  ElisionCheck check;
  check.loss_bit_identical = full.loss == elided.loss;
  double dev = max_abs_diff(full.input, elided.input);
  for (int i = 0; i < m.workers; ++i) {
    dev = std::max(dev, max_abs_diff(full.w_in[static_cast<size_t>(i)], elided.w_in[static_cast<size_t>(i)]));
    dev = std::max(dev, max_abs_diff(full.w_out[static_cast<size_t>(i)], elided.w_out[static_cast<size_t>(i)]));
  }
  check.grad_deviation = dev;
  return check;
}

}  // namespace tmpsim
