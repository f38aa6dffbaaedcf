// Internal launchers of the HBM-bound kernels (rowwise.cu, elementwise.cu).
#pragma once
#include <cuda_runtime.h>
#include <stddef.h>
#include <stdint.h>

#include "../../../include/oases.h"

namespace oases {

// Fused bias-dropout-residual + LayerNorm forward: xout = res + dropout(in + bias)
// (as bias_dropout_residual_fwd), y = LN(xout) (bit-identical to layernorm_fwd
// of xout). cudaErrorNotSupported when bdr_layernorm_supported() is false.
bool bdr_layernorm_supported(long long rows, int cols);
// keep_bits (optional): stores the dropout keep decisions, 1 bit per element
// (bit e % 16 of word e / 16), for the backward's dropout gradient.
cudaError_t bias_dropout_residual_layernorm_fwd(int dtype, const void* in, const void* bias, const void* res,
                                                void* xout, const void* gamma, const void* beta, void* y,
                                                long long rows, int cols, float eps, float p, uint64_t seed,
                                                uint64_t offset, cudaStream_t st, uint16_t* keep_bits = nullptr,
                                                int max_sms = 0);
// max_sms: SM cap of the persistent LayerNorm grid (0 = all; TMP > 1 leaves SMs to NCCL)
cudaError_t layernorm_fwd(int dtype, const void* x, const void* gamma, const void* beta, void* y, long long rows,
                          int cols, float eps, cudaStream_t st, int max_sms = 0);
size_t layernorm_bwd_workspace(long long rows, int cols);
cudaError_t layernorm_bwd(int dtype, const void* x, const void* gamma, const void* dy, void* dx, int acc_dx,
                          float* dgamma, float* dbeta, int acc_params, void* workspace, long long rows, int cols,
                          float eps, cudaStream_t st, int max_sms = 0);
// which: 1 = dx and row statistics (into workspace), 2 = dgamma/dbeta from those statistics
// gout (optional, part 1 only): also write dropout'(dx) under (drop_p, seed,
// offset) -- the bias-dropout-residual backward fused into the LN backward
// pass; cudaErrorNotSupported unless ln_bwd_dropout_supported().
bool ln_bwd_dropout_supported(int dtype, long long rows, int cols);
cudaError_t layernorm_bwd_part(int which, int dtype, const void* x, const void* gamma, const void* dy, void* dx,
                               int acc_dx, float* dgamma, float* dbeta, int acc_params, void* workspace,
                               long long rows, int cols, float eps, cudaStream_t st, void* gout = nullptr,
                               float drop_p = 0.f, uint64_t seed = 0, uint64_t offset = 0,
                               const uint16_t* keep_bits = nullptr);
// Persistent bulk-copy-pipelined LayerNorm (rowpipe.cu). Supported when
// cols = 16 * TPR with TPR a power of two in [8, 512] (cols 128..8192).
bool lnp_supported(long long rows, int cols);
// Forward: xout == nullptr -> y = LN(in); else the fused bias-dropout-residual
// xout = res + dropout(in + bias), y = LN(xout) (keep_bits: optional 1-bit
// keep decisions). max_sms caps the SMs the persistent grid uses (0 = all).
cudaError_t lnp_layernorm_fwd(int dtype, const void* in, const void* bias, const void* res, void* xout,
                              const void* gamma, const void* beta, void* y, long long rows, int cols, float eps,
                              float p, uint64_t seed, uint64_t offset, uint16_t* keep_bits, int max_sms,
                              cudaStream_t st);
// Backward: dx (+)= LN'(dy); gout (optional) = dropout'(dx) under (p, seed,
// offset) or keep_bits; part (optional) receives lnp_partial_rows(...) rows of
// [3][cols] f32 column partials (sum dy*xhat, sum dy, sum of gout -- or of dx
// when gout is null); stats (optional) the per-row (mean, rstd).
cudaError_t lnp_layernorm_bwd(int dtype, const void* x, const void* gamma, const void* dy, void* dx, int acc_dx,
                              void* gout, float p, uint64_t seed, uint64_t offset, const uint16_t* keep_bits,
                              float* part, float2* stats, long long rows, int cols, float eps, int max_sms,
                              cudaStream_t st);
// Persistent LayerNorm kernels in use: unless OASES_LNP=0 (A/B runs of the one-shot kernels).
bool lnp_enabled();
// Upper bound of lnp_partial_rows over dtypes, acc and SM caps (workspace sizing).
long long lnp_partial_rows_max(long long rows, int cols);
// Partial rows one lnp_layernorm_bwd launch of this shape writes (0 if unsupported).
long long lnp_partial_rows(int dtype, long long rows, int cols, int acc_dx, int max_sms);
// dgamma / dbeta / dbias (+)= fixed-order sums of prows partial rows (null outputs skipped).
cudaError_t lnp_finalize(const float* part, long long prows, int cols, float* dgamma, float* dbeta, float* dbias,
                         int acc_gamma, int acc_beta, int acc_bias, cudaStream_t st);
// batch = n_samples * heads_local; rows are (sample, local head, query).
cudaError_t softmax_fwd(int dtype, const void* s, void* p, void* pd, long long batch, int seq, float scale,
                        float dropout_p, uint64_t seed, uint64_t offset, int heads_local, int heads_total,
                        int head_offset, cudaStream_t st);
cudaError_t softmax_bwd(int dtype, const void* p, const void* dpd, void* ds, long long batch, int seq, float scale,
                        float dropout_p, uint64_t seed, uint64_t offset, int heads_local, int heads_total,
                        int head_offset, cudaStream_t st);
// Device-side U(-scale, scale) fill (Philox keyed by seed/offset) and constant fill.
cudaError_t fill_uniform(int dtype, void* p, long long n, float scale, uint64_t seed, uint64_t offset, cudaStream_t st);
cudaError_t fill_const(int dtype, void* p, long long n, float v, cudaStream_t st);
// Elementwise dtype conversion of a contiguous buffer (f32 <-> bf16).
cudaError_t convert(int src_dtype, const void* src, int dst_dtype, void* dst, long long n, cudaStream_t st);
cudaError_t bias_dropout_residual_fwd(int dtype, const void* x, const void* bias, const void* res, void* out,
                                      long long rows, int cols, float p, uint64_t seed, uint64_t offset,
                                      cudaStream_t st);
size_t colsum_workspace(long long rows, int cols);
// dx = dropout'(in) (if dx), out (+)= column sums of dx (if out).
cudaError_t col_pass(int dtype, const void* in, void* dx, float* out, int acc, void* ws, long long rows, int cols,
                     float p, uint64_t seed, uint64_t offset, cudaStream_t st);
// out (+)= sum over `chunks` rows of part[chunks][cols] (fixed order).
cudaError_t col_finalize(const float* part, long long chunks, int cols, float* out, int acc, cudaStream_t st);
cudaError_t gelu_fwd(int dtype, const void* x, void* y, long long n, cudaStream_t st);
cudaError_t gelu_bwd(int dtype, const void* x, const void* dy, void* dx, long long n, cudaStream_t st);
size_t loss_workspace();
cudaError_t gelu_sq_loss(int dtype, const void* z, void* dz, double* loss, int acc, double* ws, long long n,
                         cudaStream_t st);
cudaError_t local_allreduce(int dtype, void* const* bufs, int w, long long n, cudaStream_t st);
// In-process AllGather: bufs[i] holds chunk i (n elements at offset i * n); afterwards every
// buffer holds all w chunks (16-byte aligned buffers, n * element size % 16 == 0).
cudaError_t local_allgather(int dtype, void* const* bufs, int w, long long n, cudaStream_t st);

}  // namespace oases

namespace oases {
// f64 value-level numerics (numerics_f64.cu; the reference's numerics.hpp:10-60 on the device)
enum { F64_ADD = 0, F64_HADAMARD = 1, F64_GELU = 2, F64_GELU_GRAD = 3 };
cudaError_t map_f64(int op, const double* a, const double* b, double* out, long long n, cudaStream_t st);
cudaError_t transpose_f64(const double* a, double* t, int rows, int cols, cudaStream_t st);
cudaError_t max_abs_diff_f64(const double* a, const double* b, long long n, double* out, cudaStream_t st);
cudaError_t grad_identity_fd_f64(const double* x, const double* weights, int workers, int n, double h, double* fd,
                                 cudaStream_t st);
}  // namespace oases
