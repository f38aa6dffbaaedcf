// Internal GEMM entry points behind oases_gemm (include/oases.h).
#pragma once
#include <cuda_runtime.h>
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
// f32 operands: FFMA tiled kernel for the 1e-4 parity mode (gemm_simt.cu).
GemmStatus gemm_simt(const oases_gemm_desc& d, cudaStream_t stream);

}  // namespace oases
