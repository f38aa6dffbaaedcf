/*
 * oases.h -- C-ABI of the B200-native Oases TMP hot path.
 *
 * This is the drop-in boundary. The reference (tmpsim) has no
 * C-ABI; its operator API is the C++ header set proj/include/tmpsim/ *.hpp,
 * mirrored 1:1 by pybind11 in proj/python/bindings.cpp:28-236. Every entry
 * point below either replaces one of those functions with a real-hardware
 * counterpart, or exposes one kernel of the layer arithmetic that the reference
 * restates in fp64 (proj/src/numerics.cpp). Plain pointers and sizes only: no
 * torch or C++ types cross this boundary.
 *
 * Conventions
 *   - Status codes mirror the reference CLI exit codes (proj/tools/main.cpp:30-32,
 *     281-293): CONFIG=2 <-> tmpsim::ConfigError, INFEASIBLE=3 <-> InfeasibleError,
 *     IO=4 <-> IoError (proj/include/tmpsim/errors.hpp:11-26). CUDA/NCCL failures
 *     get their own codes. oases_last_error() returns a thread-local message.
 *   - Kernel entry points take device pointers and a cudaStream_t (as void*), and
 *     allocate nothing. Runtime objects (ctx, stack) own all device memory.
 *   - There is no CPU fallback: every compute entry point launches CUDA kernels
 *     and fails with OASES_ERR_CUDA when no device is present.
 */
#ifndef OASES_H_
#define OASES_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  OASES_OK = 0,
  OASES_ERR_CONFIG = 2,     /* tmpsim::ConfigError   (errors.hpp:11-14) */
  OASES_ERR_INFEASIBLE = 3, /* tmpsim::InfeasibleError (errors.hpp:17-20) */
  OASES_ERR_IO = 4,         /* tmpsim::IoError       (errors.hpp:22-25) */
  OASES_ERR_CUDA = 5,
  OASES_ERR_NCCL = 6
} oases_status;

typedef enum { OASES_F32 = 0, OASES_BF16 = 1, OASES_F64 = 2 } oases_dtype;

const char* oases_last_error(void);
const char* oases_version(void);
/* Number of SMs of the current device (0 when no device). */
int oases_device_sm_count(void);

/* ------------------------------------------------------------------------ */
/* GEMM: C[z](m,n) = epilogue( alpha * sum_k A[z](m,k) * B[z](n,k) )        */
/* Replaces matmul (numerics.cpp:13-24) and transpose (numerics.cpp:26-32):  */
/* transposes are operand major-ness, never a kernel.                        */
/* ------------------------------------------------------------------------ */

/* Operand in a 2-D row-major storage buffer [rows x cols], leading dim ld.
 * mn_major = 0: logical element (mn, k) lives at [row = mn, col = k] (K contiguous)
 * mn_major = 1: logical element (mn, k) lives at [row = k,  col = mn] (MN contiguous)
 * Batch z = zo * batch_inner + zi adds row offset row_off[0]*zo + row_off[1]*zi
 * and column offset col_off[0]*zo + col_off[1]*zi. */
typedef struct {
  const void* ptr;
  int64_t rows, cols, ld;
  int32_t mn_major;
  int32_t pad_;
  int64_t row_off[2];
  int64_t col_off[2];
} oases_gemm_operand;

typedef enum {
  OASES_EPI_NONE = 0,      /* C = alpha*acc (+ C if accumulate) */
  OASES_EPI_BIAS = 1,      /* C = alpha*acc + bias[n] */
  OASES_EPI_BIAS_GELU = 2, /* C = v = alpha*acc + bias[n];  C2 = gelu(v)  (erf GeLU, numerics.cpp:50);
                              C2 == NULL: C = gelu(v) only (the pre-activation is not stored) */
  OASES_EPI_DGELU = 3,     /* C = alpha*acc * gelu'(AUX[m,n])  (hadamard+gelu_grad, numerics.cpp:204) */
  OASES_EPI_BIAS_GELU_GRAD = 4, /* v = alpha*acc + bias[n]; C = gelu'(v), C2 = gelu(v)  (the recompute FC1:
                                   stores the factor the dgrad needs instead of the pre-activation) */
  OASES_EPI_MUL = 5,       /* C = alpha*acc * AUX[m,n]  (dgrad with a stored gelu'(pre)) */
  OASES_EPI_ROWDOT = 6     /* C = alpha*acc (bf16); ROWDOT[(m / seq * heads + g) * seq + m % seq] =
                              sum over the columns of group g (rowdot_group wide) of C[m,n]*AUX[m,n]:
                              the attention backward's D = rowsum(dO o O) per head, fused into the
                              GEMM producing dO */
} oases_epilogue;

typedef enum {
  OASES_CAUSAL_NONE = 0,
  OASES_CAUSAL_SKIP_UPPER = 1, /* output tiles strictly above the diagonal are not computed */
  OASES_CAUSAL_K_UPTO_M = 2,   /* reduction limited to k < m_tile_end (P.V, dS.K) */
  OASES_CAUSAL_K_FROM_M = 3    /* reduction limited to k >= m_tile_begin (P^T.dO, dS^T.Q) */
} oases_causal;

typedef struct {
  int32_t dtype;  /* operand dtype: OASES_BF16 -> tcgen05/TMEM/TMA kernel, OASES_F32 -> FFMA kernel */
  int32_t c_dtype;
  int64_t M, N, K;
  int64_t batch, batch_inner;
  oases_gemm_operand a, b;
  void* c;
  int64_t ldc;
  int64_t c_row_off[2];
  int64_t c_col_off[2];
  int32_t epilogue;
  int32_t causal;
  float alpha;
  int32_t accumulate;   /* C += result */
  const void* bias;     /* [N] in operand dtype (bf16 or f32) */
  const void* aux;      /* DGELU input, same layout/offsets/dtype as C */
  void* c2;             /* BIAS_GELU activation output, same layout/offsets/dtype as C */
  int32_t max_ctas;     /* persistent grid cap (0 = all SMs); leaves SMs to NCCL */
  int32_t pad_;
  float* rowdot;                    /* ROWDOT output (f32) */
  int32_t rowdot_group;             /* columns per group (head dim: 64 | 128) */
  int32_t rowdot_seq, rowdot_heads; /* rows per sample, groups per row */
  int32_t pad2_;
  float* colsum; /* MUL epilogue, optional: COLSUM[m / 32][n] = sum over rows m..m+31 of the stored C
                    (bf16-rounded), f32, N % 32 == 0; oases_colsum_finalize sums the [ceil(M/32), N]
                    partials into the bias gradient (replaces a column-sum pass over C) */
} oases_gemm_desc;

oases_status oases_gemm(const oases_gemm_desc* desc, void* stream);
/* `count` independent problems (bf16). Two CTA-pair-shaped problems share one
 * persistent launch (one tile list, longer-K problem first); results are
 * bit-identical to separate oases_gemm calls. */
oases_status oases_gemm_grouped(const oases_gemm_desc* descs, int32_t count, void* stream);

/* ------------------------------------------------------------------------ */
/* Fused causal attention (tcgen05 flash kernels; bf16, head_dim 64 | 128,   */
/* seq % 128 == 0). Same arithmetic as the unfused QK^T -> softmax ->        */
/* dropout -> PV chain (numerics.cpp attention, dropout keys of DESIGN.md)  */
/* without materialising the [seq, seq] probabilities.                      */
/*   qkv   [samples*seq, ld_qkv]: Q | K | V column blocks of                 */
/*         heads_local*head_dim each (head h at h*head_dim inside a block)   */
/*   out   [samples*seq, ld_out]: ctx, head h at column h*head_dim           */
/*   lse   [samples*heads_local*seq] f32 row log-sum-exp (log2 domain)       */
/*   bwd:  dout like out; dqkv like qkv (all three blocks written);          */
/*         ds [samples*heads_local*seq, seq] bf16 scratch (dS, causal band); */
/*         workspace: oases_attention_bwd_workspace() bytes                  */
/*   mask_bits (optional, dropout on): cache of the Philox keep bits, one    */
/*         bit per causal-band element, oases_attention_mask_bytes() bytes.  */
/*         mask_mode 0: generate (Philox); 1: generate and store (forward);  */
/*         2: read (recompute forward, backward) -- the bits ARE the Philox  */
/*         results, so every mode computes the same values.                  */
/* ------------------------------------------------------------------------ */
typedef struct {
  int32_t dtype; /* OASES_BF16 */
  int32_t samples, heads_local, heads_total, head_offset, head_dim, seq;
  int32_t max_ctas; /* dQ GEMM CTA cap (0 = all SMs) */
  const void* qkv;
  int64_t ld_qkv;
  void* out;
  int64_t ld_out;
  float* lse;
  const void* dout;
  int64_t ld_dout;
  void* dqkv;
  int64_t ld_dqkv;
  void* ds;
  void* workspace;
  float scale, dropout_p;
  uint64_t seed, offset;
  uint32_t* mask_bits;
  int32_t mask_mode;
  int32_t dsum_ready; /* bwd: workspace already holds D = rowsum(dO o O) (e.g. an EPI_ROWDOT GEMM) */
  /* dropout keys: sample n of this tensor is sample sample_offset + n of the
   * keyed sub-batch (0 normally; data-parallel groups of a mixed-degree stack
   * hold a slice of it) */
  int32_t sample_offset;
  int32_t pad_;
} oases_attn_desc;

int32_t oases_attention_supported(int dtype, int32_t head_dim, int32_t seq);
oases_status oases_attention_fwd(const oases_attn_desc* desc, void* stream);
size_t oases_attention_bwd_workspace(const oases_attn_desc* desc);
/* Generates the keep bits of every causal-band element into desc->mask_bits
 * (the Philox masks mask_mode 1 would store) with a separate fully parallel
 * kernel, so the forward can run with mask_mode 2. Needs dropout_p > 0. */
oases_status oases_attention_masks(const oases_attn_desc* desc, void* stream);
size_t oases_attention_mask_bytes(const oases_attn_desc* desc);
oases_status oases_attention_bwd(const oases_attn_desc* desc, void* stream);

/* ------------------------------------------------------------------------ */
/* HBM-bound kernels (vectorised, warp-shuffle reductions).                  */
/* All row-major [rows x cols]; dtype selects f32 or bf16 activations;       */
/* statistics, parameters' gradients and loss are always f32.               */
/* ------------------------------------------------------------------------ */

/* y = (x - mean) * rstd * gamma + beta; gamma/beta in activation dtype. */
oases_status oases_layernorm_fwd(int dtype, const void* x, const void* gamma, const void* beta,
                                 void* y, int64_t rows, int64_t cols, float eps, void* stream);
/* dx (+)= LN backward given dy; gamma-grad/beta-grad partials are reduced
 * deterministically into dgamma/dbeta (f32, accumulate if acc_params). */
oases_status oases_layernorm_bwd(int dtype, const void* x, const void* gamma, const void* dy,
                                 void* dx, int accumulate_dx, float* dgamma, float* dbeta,
                                 int acc_params, float* workspace, int64_t rows, int64_t cols,
                                 float eps, void* stream);
size_t oases_layernorm_bwd_workspace(int64_t rows, int64_t cols);

/* Causal scaled softmax over rows of S viewed as [batch*s, s], batch =
 * samples * heads_local (row r has query position r % s); optional Philox
 * dropout writes P_drop, keyed by the GLOBAL head (head_offset + local head of
 * heads_total) so masks do not depend on the TMP degree. s_in may alias p_out. */
oases_status oases_softmax_fwd(int dtype, const void* s_in, void* p_out, void* p_drop,
                               int64_t batch, int64_t seq, float scale, float dropout_p,
                               uint64_t seed, uint64_t offset, int32_t heads_local,
                               int32_t heads_total, int32_t head_offset, void* stream);
/* dS = scale * P o (dP - rowsum(P o dP)), dP = dropout'(dP_drop); ds may alias dp_drop. */
oases_status oases_softmax_bwd(int dtype, const void* p, const void* dp_drop, void* ds,
                               int64_t batch, int64_t seq, float scale, float dropout_p,
                               uint64_t seed, uint64_t offset, int32_t heads_local,
                               int32_t heads_total, int32_t head_offset, void* stream);

/* out = residual + dropout(x + bias): the Megatron bias-dropout-add. */
oases_status oases_bias_dropout_residual_fwd(int dtype, const void* x, const void* bias,
                                             const void* residual, void* out, int64_t rows,
                                             int64_t cols, float dropout_p, uint64_t seed,
                                             uint64_t offset, void* stream);
/* Fused: x_out = residual + dropout(x + bias) (as oases_bias_dropout_residual_fwd)
 * and y = LayerNorm(x_out) (bit-identical to oases_layernorm_fwd of x_out), one
 * HBM pass. The block-boundary step of the layer (SURVEY.md 8(a) block
 * partition: bias-dropout-residual on AR_{b-1}, then LN_b). Shapes the fused
 * kernel does not cover (cols % 16, or cols/16 not a multiple of 32 up to
 * 4*256) return OASES_ERR_CONFIG; callers then issue the two kernels. */
oases_status oases_bias_dropout_residual_layernorm_fwd(int dtype, const void* x, const void* bias,
                                                       const void* residual, void* x_out,
                                                       const void* gamma, const void* beta, void* y,
                                                       int64_t rows, int64_t cols, float eps,
                                                       float dropout_p, uint64_t seed, uint64_t offset,
                                                       void* stream);
/* dx = dropout'(dout); dbias (+)= column sums of dx (deterministic). */
oases_status oases_bias_dropout_residual_bwd(int dtype, const void* dout, void* dx, float* dbias,
                                             int acc_bias, float* workspace, int64_t rows,
                                             int64_t cols, float dropout_p, uint64_t seed,
                                             uint64_t offset, void* stream);
size_t oases_colsum_workspace(int64_t rows, int64_t cols);
/* dbias (+)= column sums of x. */
oases_status oases_colsum(int dtype, const void* x, float* out, int accumulate, float* workspace,
                          int64_t rows, int64_t cols, void* stream);
/* out[n] (+)= sum_k partials[k][n], k < chunks, fixed order (deterministic): the second half of
 * oases_colsum for partials a GEMM's MUL epilogue wrote (oases_gemm_desc.colsum). */
oases_status oases_colsum_finalize(const float* partials, int64_t chunks, int64_t cols, float* out,
                                   int accumulate, void* stream);

/* Exact-erf GeLU and its derivative (numerics.cpp:50-55,66-76). */
oases_status oases_gelu_fwd(int dtype, const void* x, void* y, int64_t n, void* stream);
oases_status oases_gelu_bwd(int dtype, const void* x, const void* dy, void* dx, int64_t n,
                            void* stream);

/* Loss head of the checker (numerics.cpp:175-188): loss = 1/2 sum gelu(z)^2,
 * dz = gelu(z) * gelu'(z). loss_out is a device f64 scalar (accumulated if acc). */
oases_status oases_gelu_sq_loss(int dtype, const void* z, void* dz, double* loss_out, int acc,
                                double* workspace, int64_t n, void* stream);

/* In-process AllReduce of `workers` equally sized buffers (sum in worker
 * order 0..w-1, result written to every buffer): the literal sum of
 * numerics.cpp:96-100,160-163 for single-GPU emulation of TMP ranks. */
oases_status oases_local_allreduce(int dtype, void* const* bufs, int workers, int64_t n,
                                   void* stream);

/* ------------------------------------------------------------------------ */
/* Runtime: context (devices, streams, NCCL), layer stack, plan, step.       */
/* ------------------------------------------------------------------------ */

typedef struct oases_ctx oases_ctx;
typedef struct oases_stack oases_stack;

#define OASES_UNIQUE_ID_BYTES 128

/* ncclGetUniqueId; rank 0 broadcasts the bytes to all ranks out of band. */
oases_status oases_get_unique_id(void* out /* OASES_UNIQUE_ID_BYTES */);

typedef struct {
  int32_t tp;             /* TMP degree of the group */
  int32_t rank;           /* this process' rank in the group (NCCL mode) */
  int32_t device;         /* CUDA device ordinal */
  int32_t local_workers;  /* >1: emulate `tp` ranks in-process on one device (tp == local_workers) */
  const void* unique_id;  /* NCCL id bytes (required when tp > 1 and local_workers == 1) */
  int32_t nccl_max_ctas;  /* 0 = NCCL default */
  int32_t gemm_max_ctas;  /* persistent GEMM grid cap while comm may overlap (0 = all SMs) */
  int32_t comm_disabled;  /* 1: one rank's shard of a tp-way group, AllReduces skipped (calibration
                             of per-degree compute costs on a single device) */
} oases_ctx_desc;

oases_status oases_ctx_create(const oases_ctx_desc* desc, oases_ctx** out);
oases_status oases_ctx_destroy(oases_ctx* ctx);

/* Model description: tmpsim::ModelSpec fields (model.hpp:28-38) plus the
 * numerics knobs of the real layer. */
typedef struct {
  int32_t hidden_size;
  int32_t num_layers;
  int32_t seq_len;
  int32_t attention_heads;
  int32_t global_batch;      /* micro-batch b; split into two sub-batches */
  int32_t bytes_per_element; /* 2 = bf16, 4 = f32 */
  int32_t recompute_enabled;
  int32_t ffn_hidden;        /* 0 -> 4*hidden */
  int32_t use_attention;     /* 0 -> FFN-only layers (the reference toy) */
  int32_t use_layernorm;
  int32_t use_bias;
  int32_t use_residual;
  float hidden_dropout;
  float attention_dropout;
  float ln_eps;
  int32_t pad_;
  uint64_t seed;             /* Philox key for dropout */
} oases_model_desc;

oases_status oases_stack_create(oases_ctx* ctx, const oases_model_desc* model, oases_stack** out);
/* Mixed per-block TMP degrees (the planner's non-uniform strategies,
 * planner.hpp Strategy::degrees): block_degrees[b] divides the world size
 * (ctx tp); a degree-d block runs data-parallel on tp/d groups of d ranks
 * (group g owns samples [g*b*d/tp, (g+1)*b*d/tp) of the micro-batch), the
 * executor inserts the resharding AllGathers between blocks of different
 * degree (sim.cpp:101-175) and sums the data-parallel gradients at step end.
 * Needs hidden_dropout == 0. */
oases_status oases_stack_create_mixed(oases_ctx* ctx, const oases_model_desc* model, const int32_t* block_degrees,
                                      int32_t num_blocks, oases_stack** out);
int oases_stack_block_degree(const oases_stack* s, int block);

/* Rank geometry of one block (host-only: callable without a device). The
 * stack on `world` ranks places rank `rank`'s share of block b at: tokens
 * [token_row0, token_row0 + 2 * tokens_per_sub_batch) of the micro-batch (its
 * data-parallel group's slice, two sub-batches), heads / FFN columns
 * [rank_in_group * w, (rank_in_group + 1) * w) of the block's weights, w =
 * col_width / 3 (attention QKV: q, k, v each heads_local * head_dim wide) or
 * col_width (FFN). Tensor-parallel group = `group` (ncclCommSplit colour
 * rank / degree), data-parallel peers share rank_in_group (colour rank %
 * degree). Replaces the rank arithmetic the reference does inline in
 * numerics.cpp:120-165 (uniform degree) and sim.cpp:101-175 (mixed). */
typedef struct {
  int32_t degree;
  int32_t group;          /* data-parallel group of the block (0 .. groups-1) */
  int32_t rank_in_group;  /* tensor-parallel rank inside the group */
  int32_t groups;         /* world / degree */
  int32_t heads_local;    /* attention blocks; 0 for FFN blocks */
  int32_t attention;      /* 1: attention block (QKV/proj), 0: FFN block */
  int64_t samples_per_sub_batch;
  int64_t tokens_per_sub_batch;
  int64_t token_row0;
  int64_t col_width;      /* local width of the column-parallel weight (QKV | FC1) */
  int64_t row_width;      /* local width of the row-parallel weight's input (proj | FC2) */
} oases_block_layout;

/* block_degrees: num_blocks entries (null: every block at the world degree);
 * out: num_blocks entries. Errors as oases_stack_create_mixed would raise. */
oases_status oases_rank_layout(const oases_model_desc* model, int32_t world, const int32_t* block_degrees,
                               int32_t num_blocks, int32_t rank, oases_block_layout* out);
oases_status oases_stack_destroy(oases_stack* stack);

/* Parameter tensors per block, identified by (block, param id). Host f64
 * views in the oracle's layout are converted and copied (non-owning). */
typedef enum {
  OASES_P_LN_GAMMA = 0, OASES_P_LN_BETA = 1,
  OASES_P_W_COL = 2,    /* column-parallel weight, oracle layout [in=h, out_shard] */
  OASES_P_B_COL = 3,    /* [out_shard] */
  OASES_P_W_ROW = 4,    /* row-parallel weight, oracle layout [in_shard, out=h] */
  OASES_P_B_ROW = 5,    /* [h], replicated */
  OASES_P_COUNT = 6
} oases_param;

/* Element count of a parameter of one worker (0 if the block has none). */
int64_t oases_stack_param_numel(const oases_stack* s, int block, int param);
int oases_stack_num_blocks(const oases_stack* s);
int oases_stack_num_workers(const oases_stack* s);
oases_status oases_stack_set_param(oases_stack* s, int worker, int block, int param,
                                   const double* host);
oases_status oases_stack_get_grad(oases_stack* s, int worker, int block, int param, double* host);
/* Random init following numerics.cpp:146-152 conventions with a Philox stream
 * on device (for perf runs where no oracle upload is wanted). */
oases_status oases_stack_init_random(oases_stack* s, uint64_t seed);

/* Flattened tmpsim::SchedulePlan (schedule.hpp:27-53). */
typedef struct {
  int32_t id, base_id, kind, pass, stream, block, sub_batch, blocking;
  int32_t dep_begin, dep_count; /* into deps[] */
} oases_plan_op;

typedef struct {
  int32_t variant;      /* tmpsim::ScheduleVariant */
  int32_t split_batch;
  int32_t has_recompute;
  int32_t n_forward;    /* ops[0..n_forward) are forward_ops */
  int32_t n_ops;
  int32_t n_deps;
  const oases_plan_op* ops;
  const int32_t* deps;
} oases_flat_plan;

oases_status oases_plan_bind(oases_stack* s, const oases_flat_plan* plan);

typedef struct {
  int32_t op_id;   /* plan id; tail ops get ids >= n_ops */
  int32_t stream;  /* 0 compute, 1 comm */
  double start, end; /* seconds from step start (cudaEvent) */
} oases_trace_event;

typedef struct {
  double makespan;              /* seconds */
  double compute_busy_fraction;
  double comm_exposed;          /* sim.cpp:178-199 interval algebra on measured events */
  double peak_memory;           /* bytes resident for the stack on this device */
  double loss;
  int32_t n_events;
  int32_t pad_;
  oases_trace_event* events;    /* owned by the stack; valid until the next step */
} oases_step_result;

/* One training step (forward, recompute, backward under the bound plan) on
 * input [b, s, h] (per worker identical). input_host != NULL: pinned/pageable
 * host buffer of dtype `input_dtype` (0 f32, 1 bf16, 2 f64) copied inside the
 * step; input_host == NULL: reuse the device-resident input. trace=1 records
 * per-op cudaEvents (needed for makespan/comm_exposed). */
oases_status oases_step(oases_stack* s, const void* input_host, int input_dtype, int trace,
                        oases_step_result* out);
/* Device-resident input upload without stepping. */
oases_status oases_stack_set_input(oases_stack* s, const void* host, int input_dtype);
/* Gradient of the loss w.r.t. the stack input, [b, s, h] as f64 on host. */
oases_status oases_stack_get_input_grad(oases_stack* s, double* host);
/* Block-boundary activation x_b (saved residual stream), sub-batch sb, as f64. */
oases_status oases_stack_get_activation(oases_stack* s, int worker, int block, int sb,
                                        double* host);
/* Capture the bound plan's step as a CUDA graph (trace off). */
oases_status oases_stack_capture_graph(oases_stack* s);
oases_status oases_stack_sync(oases_stack* s);
/* Number of kernels this stack has launched (all steps so far). */
int oases_stack_kernel_launches(const oases_stack* s);
/* Live cudaEvent timing of every linear-layer GEMM launch (QKV/proj/FC1/FC2
 * forward, dgrad, wgrad) on the compute stream, for the roofline in bench.py.
 * Stats accumulate over steps since the last read; reading resets them. */
typedef struct {
  double gemm_ms;     /* summed launch durations */
  double gemm_flops;  /* summed algorithmic 2*M*N*K */
  int32_t gemm_launches;
  int32_t pad_;
} oases_kernel_stats;
oases_status oases_stack_set_kernel_timing(oases_stack* s, int on);
oases_status oases_stack_kernel_stats(oases_stack* s, oases_kernel_stats* out);
/* The same GEMM statistics measured inside a replay of the captured step: the
 * timing events become graph nodes of a separately captured copy of the step,
 * which is replayed twice; the second replay's timings are returned. */
oases_status oases_stack_graph_kernel_stats(oases_stack* s, oases_kernel_stats* out);

#ifdef __cplusplus
}
#endif

#endif /* OASES_H_ */
