// Internal GEMM entry points behind oases_gemm (include/oases.h).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <string>

#include "../../../include/oases.h"

namespace oases {

struct GemmStatus {
  bool ok = false;
  bool cuda = false;
  std::string err;
};

// bf16 operands: tcgen05/TMEM/TMA persistent kernel (gemm_tc.cu).
GemmStatus gemm_tc(const oases_gemm_desc& d, cudaStream_t stream);
// n independent bf16 problems in one persistent launch when they are all
// CTA-pair shaped (n == 2), else one launch each.
GemmStatus gemm_tc_group(const oases_gemm_desc* d, int n, cudaStream_t stream);
// f32 operands: FFMA tiled kernel for the 1e-4 parity mode (gemm_simt.cu).
GemmStatus gemm_simt(const oases_gemm_desc& d, cudaStream_t stream);

// bf16 row-major [rows, cols] (row stride ld elements) tensor map, SWIZZLE_128B,
// box {box_inner columns, box_outer rows}.
bool make_tma_bf16_2d(CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld, uint32_t box_inner,
                      uint32_t box_outer, std::string* err);

// Fused causal attention (attention.cu): tcgen05 flash forward, dK/dV kernel
// + deterministic dQ GEMM backward.
bool attention_supported(int dtype, int head_dim, int seq);
GemmStatus attention_fwd(const oases_attn_desc& d, cudaStream_t stream);
size_t attention_bwd_workspace(const oases_attn_desc& d);
size_t attention_mask_bytes(const oases_attn_desc& d);
GemmStatus attention_bwd(const oases_attn_desc& d, cudaStream_t stream);
// keep bits of every causal-band element into d.mask_bits (read by mask_mode 2)
GemmStatus attention_masks(const oases_attn_desc& d, cudaStream_t stream);

}  // namespace oases
