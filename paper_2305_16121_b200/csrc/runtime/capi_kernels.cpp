// extern "C" kernel entry points of include/oases.h. Each validates its
// arguments, launches on the given stream and allocates nothing.
#include <cuda_runtime.h>

#include <string>

#include "../../../include/oases.h"
#include "../../../include/oases/tmpsim.hpp"
#include "../kernels/gemm.h"
#include "../kernels/kernels.h"
#include "status.h"

namespace oases {

thread_local std::string g_last_error;

void set_last_error(const std::string& msg) { g_last_error = msg; }

}  // namespace oases

using oases::check_cuda;
using oases::guarded;

namespace {
cudaStream_t S(void* s) { return static_cast<cudaStream_t>(s); }
void need_device() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    throw oases::CudaError("no CUDA device: the Oases kernels have no CPU fallback");
  }
}
void check_dtype(int dtype) {
  if (dtype != OASES_F32 && dtype != OASES_BF16) throw tmpsim::ConfigError("unknown dtype");
}
}  // namespace

extern "C" {

const char* oases_last_error(void) { return oases::g_last_error.c_str(); }
const char* oases_version(void) { return "oases-b200 0.1.0 (sm_100a)"; }

int oases_device_sm_count(void) {
  int n = 0, dev = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    return 0;
  }
  cudaGetDevice(&dev);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

oases_status oases_gemm(const oases_gemm_desc* d, void* stream) {
  return guarded([&] {
    if (!d) throw tmpsim::ConfigError("oases_gemm: null descriptor");
    need_device();
    oases::GemmStatus st;
    if (d->dtype == OASES_BF16) st = oases::gemm_tc(*d, S(stream));
    else if (d->dtype == OASES_F32) st = oases::gemm_simt(*d, S(stream));
    else throw tmpsim::ConfigError("oases_gemm: unknown dtype");
    if (!st.ok) {
      if (st.cuda) throw oases::CudaError(st.err);
      throw tmpsim::ConfigError(st.err);
    }
  });
}

oases_status oases_gemm_grouped(const oases_gemm_desc* d, int32_t count, void* stream) {
  return guarded([&] {
    if (!d || count < 1) throw tmpsim::ConfigError("oases_gemm_grouped: need at least one descriptor");
    need_device();
    for (int i = 0; i < count; ++i)
      if (d[i].dtype != OASES_BF16) throw tmpsim::ConfigError("oases_gemm_grouped: bf16 problems only");
    const oases::GemmStatus st = oases::gemm_tc_group(d, count, S(stream));
    if (!st.ok) {
      if (st.cuda) throw oases::CudaError(st.err);
      throw tmpsim::ConfigError(st.err);
    }
  });
}

namespace {
void gemm_status_throw(const oases::GemmStatus& st) {
  if (st.ok) return;
  if (st.cuda) throw oases::CudaError(st.err);
  throw tmpsim::ConfigError(st.err);
}
}  // namespace

int32_t oases_attention_supported(int dtype, int32_t head_dim, int32_t seq) {
  return oases::attention_supported(dtype, head_dim, seq) ? 1 : 0;
}

oases_status oases_attention_fwd(const oases_attn_desc* d, void* stream) {
  return guarded([&] {
    if (!d) throw tmpsim::ConfigError("oases_attention_fwd: null descriptor");
    need_device();
    gemm_status_throw(oases::attention_fwd(*d, S(stream)));
  });
}

size_t oases_attention_bwd_workspace(const oases_attn_desc* d) {
  return d ? oases::attention_bwd_workspace(*d) : 0;
}

size_t oases_attention_mask_bytes(const oases_attn_desc* d) { return d ? oases::attention_mask_bytes(*d) : 0; }

oases_status oases_attention_masks(const oases_attn_desc* d, void* stream) {
  return guarded([&] {
    if (!d) throw tmpsim::ConfigError("oases_attention_masks: null descriptor");
    need_device();
    gemm_status_throw(oases::attention_masks(*d, S(stream)));
  });
}

oases_status oases_attention_bwd(const oases_attn_desc* d, void* stream) {
  return guarded([&] {
    if (!d) throw tmpsim::ConfigError("oases_attention_bwd: null descriptor");
    need_device();
    gemm_status_throw(oases::attention_bwd(*d, S(stream)));
  });
}

oases_status oases_layernorm_fwd(int dtype, const void* x, const void* gamma, const void* beta, void* y,
                                 int64_t rows, int64_t cols, float eps, void* stream) {
  return guarded([&] {
    check_dtype(dtype);
    need_device();
    if (cols % 8) throw tmpsim::ConfigError("layernorm: cols must be a multiple of 8");
    check_cuda(oases::layernorm_fwd(dtype, x, gamma, beta, y, rows, static_cast<int>(cols), eps, S(stream)),
               "layernorm_fwd");
  });
}

oases_status oases_bias_dropout_residual_layernorm_fwd(int dtype, const void* x, const void* bias,
                                                       const void* residual, void* x_out, const void* gamma,
                                                       const void* beta, void* y, int64_t rows, int64_t cols,
                                                       float eps, float dropout_p, uint64_t seed, uint64_t offset,
                                                       void* stream) {
  return guarded([&] {
    check_dtype(dtype);
    need_device();
    if (!oases::bdr_layernorm_supported(rows, static_cast<int>(cols)))
      throw tmpsim::ConfigError("bias_dropout_residual_layernorm_fwd: shape not covered by the fused kernel");
    check_cuda(oases::bias_dropout_residual_layernorm_fwd(dtype, x, bias, residual, x_out, gamma, beta, y, rows,
                                                          static_cast<int>(cols), eps, dropout_p, seed, offset,
                                                          S(stream)),
               "bias_dropout_residual_layernorm_fwd");
  });
}

size_t oases_layernorm_bwd_workspace(int64_t rows, int64_t cols) {
  return oases::layernorm_bwd_workspace(rows, static_cast<int>(cols));
}

oases_status oases_layernorm_bwd(int dtype, const void* x, const void* gamma, const void* dy, void* dx,
                                 int accumulate_dx, float* dgamma, float* dbeta, int acc_params, float* workspace,
                                 int64_t rows, int64_t cols, float eps, void* stream) {
  return guarded([&] {
    check_dtype(dtype);
    need_device();
    if (cols % 8) throw tmpsim::ConfigError("layernorm: cols must be a multiple of 8");
    check_cuda(oases::layernorm_bwd(dtype, x, gamma, dy, dx, accumulate_dx, dgamma, dbeta, acc_params, workspace,
                                    rows, static_cast<int>(cols), eps, S(stream)),
               "layernorm_bwd");
  });
}

oases_status oases_softmax_fwd(int dtype, const void* s_in, void* p_out, void* p_drop, int64_t batch, int64_t seq,
                               float scale, float dropout_p, uint64_t seed, uint64_t offset, int32_t heads_local,
                               int32_t heads_total, int32_t head_offset, void* stream) {
  return guarded([&] {
    check_dtype(dtype);
    need_device();
    if (seq % 8) throw tmpsim::ConfigError("softmax: seq must be a multiple of 8");
    if (heads_local < 1 || batch % heads_local) throw tmpsim::ConfigError("softmax: batch must be samples * heads_local");
    check_cuda(oases::softmax_fwd(dtype, s_in, p_out, p_drop, batch, static_cast<int>(seq), scale, dropout_p, seed,
                                  offset, heads_local, heads_total, head_offset, S(stream)),
               "softmax_fwd");
  });
}

oases_status oases_softmax_bwd(int dtype, const void* p, const void* dp_drop, void* ds, int64_t batch, int64_t seq,
                               float scale, float dropout_p, uint64_t seed, uint64_t offset, int32_t heads_local,
                               int32_t heads_total, int32_t head_offset, void* stream) {
  return guarded([&] {
    check_dtype(dtype);
    need_device();
    if (seq % 8) throw tmpsim::ConfigError("softmax: seq must be a multiple of 8");
    if (heads_local < 1 || batch % heads_local) throw tmpsim::ConfigError("softmax: batch must be samples * heads_local");
    check_cuda(oases::softmax_bwd(dtype, p, dp_drop, ds, batch, static_cast<int>(seq), scale, dropout_p, seed, offset,
                                  heads_local, heads_total, head_offset, S(stream)),
               "softmax_bwd");
  });
}

oases_status oases_bias_dropout_residual_fwd(int dtype, const void* x, const void* bias, const void* residual,
                                             void* out, int64_t rows, int64_t cols, float dropout_p, uint64_t seed,
                                             uint64_t offset, void* stream) {
  return guarded([&] {
    check_dtype(dtype);
    need_device();
    check_cuda(oases::bias_dropout_residual_fwd(dtype, x, bias, residual, out, rows, static_cast<int>(cols),
                                                dropout_p, seed, offset, S(stream)),
               "bias_dropout_residual_fwd");
  });
}

oases_status oases_bias_dropout_residual_bwd(int dtype, const void* dout, void* dx, float* dbias, int acc_bias,
                                             float* workspace, int64_t rows, int64_t cols, float dropout_p,
                                             uint64_t seed, uint64_t offset, void* stream) {
  return guarded([&] {
    check_dtype(dtype);
    need_device();
    check_cuda(oases::col_pass(dtype, dout, dx, dbias, acc_bias, workspace, rows, static_cast<int>(cols), dropout_p,
                               seed, offset, S(stream)),
               "bias_dropout_residual_bwd");
  });
}

size_t oases_colsum_workspace(int64_t rows, int64_t cols) {
  return oases::colsum_workspace(rows, static_cast<int>(cols));
}

oases_status oases_colsum(int dtype, const void* x, float* out, int accumulate, float* workspace, int64_t rows,
                          int64_t cols, void* stream) {
  return guarded([&] {
    check_dtype(dtype);
    need_device();
    check_cuda(oases::col_pass(dtype, x, nullptr, out, accumulate, workspace, rows, static_cast<int>(cols), 0.f, 0, 0,
                               S(stream)),
               "colsum");
  });
}

oases_status oases_colsum_finalize(const float* partials, int64_t chunks, int64_t cols, float* out, int accumulate,
                                   void* stream) {
  return guarded([&] {
    if (!partials || !out || chunks <= 0 || cols <= 0) throw tmpsim::ConfigError("oases_colsum_finalize: empty");
    need_device();
    check_cuda(oases::col_finalize(partials, chunks, static_cast<int>(cols), out, accumulate, S(stream)),
               "colsum_finalize");
  });
}

oases_status oases_gelu_fwd(int dtype, const void* x, void* y, int64_t n, void* stream) {
  return guarded([&] {
    check_dtype(dtype);
    need_device();
    check_cuda(oases::gelu_fwd(dtype, x, y, n, S(stream)), "gelu_fwd");
  });
}

oases_status oases_gelu_bwd(int dtype, const void* x, const void* dy, void* dx, int64_t n, void* stream) {
  return guarded([&] {
    check_dtype(dtype);
    need_device();
    check_cuda(oases::gelu_bwd(dtype, x, dy, dx, n, S(stream)), "gelu_bwd");
  });
}

oases_status oases_gelu_sq_loss(int dtype, const void* z, void* dz, double* loss_out, int acc, double* workspace,
                                int64_t n, void* stream) {
  return guarded([&] {
    check_dtype(dtype);
    need_device();
    check_cuda(oases::gelu_sq_loss(dtype, z, dz, loss_out, acc, workspace, n, S(stream)), "gelu_sq_loss");
  });
}

oases_status oases_local_allreduce(int dtype, void* const* bufs, int workers, int64_t n, void* stream) {
  return guarded([&] {
    check_dtype(dtype);
    need_device();
    if (workers < 1 || workers > 8) throw tmpsim::ConfigError("local_allreduce: 1..8 workers");
    check_cuda(oases::local_allreduce(dtype, bufs, workers, n, S(stream)), "local_allreduce");
  });
}

}  // extern "C"
