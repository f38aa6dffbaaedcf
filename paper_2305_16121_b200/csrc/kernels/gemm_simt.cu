// f32 / f64 FMA-pipe GEMM with the same operand/epilogue contract as the tcgen05 kernel.
//
// Used only in the parity modes: f32 (the north star's "fp32 within 1e-4
// relative"; TF32 tensor cores are too coarse for that bound) and f64 (the
// reference's own value-level toy checks, numerics.hpp:35-60, executed by the
// runtime -- runtime/toy.cpp).
// Tiles 64x64x16, 256 threads, 4x4 outputs per thread, strided so that global
// loads of K-contiguous and MN-contiguous operands both stay mostly coalesced.
#include "common.cuh"
#include "gemm.h"

namespace oases {
namespace {

constexpr int TM = 64, TN = 64, TK = 16;

template <typename T>
struct SimtParams {
  int M, N, K, batch_inner;
  const T* a;
  long long lda, a_row[2], a_col[2];
  int a_mn;
  const T* b;
  long long ldb, b_row[2], b_col[2];
  int b_mn;
  T* c;
  T* c2;
  const T* aux;
  const T* bias;
  long long ldc, c_row[2], c_col[2];
  int epilogue, causal, accumulate;
  float alpha;
};

__device__ __forceinline__ float fma_t(float a, float b, float c) { return fmaf(a, b, c); }
// f64: the reference matmul's arithmetic exactly (numerics.cpp:13-24): separate
// round-to-nearest multiply and add, terms with a zero A element skipped, k
// ascending per output element (the tile loop order) -- bit-identical sums.
__device__ __forceinline__ double fma_t(double a, double b, double c) {
  return a != 0.0 ? __dadd_rn(c, __dmul_rn(a, b)) : c;
}
__device__ __forceinline__ float gelu_t(float x) { return gelu_f(x); }
__device__ __forceinline__ double gelu_t(double x) { return gelu_d(x); }
__device__ __forceinline__ float gelu_grad_t(float x) { return gelu_grad_f(x); }
__device__ __forceinline__ double gelu_grad_t(double x) { return gelu_grad_d(x); }

template <typename T>
__global__ void __launch_bounds__(256) gemm_simt_kernel(const SimtParams<T> p) {
  __shared__ T As[TK][TM + 1];
  __shared__ T Bs[TK][TN + 1];
  const int z = blockIdx.z;
  const int zo = z / p.batch_inner, zi = z - zo * p.batch_inner;
  const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
  if (p.causal == OASES_CAUSAL_SKIP_UPPER && (n0 / 128) * 128 > (m0 / 128) * 128 + 127) return;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const T* A = p.a + (p.a_row[0] * zo + p.a_row[1] * zi) * p.lda + (p.a_col[0] * zo + p.a_col[1] * zi);
  const T* B = p.b + (p.b_row[0] * zo + p.b_row[1] * zi) * p.ldb + (p.b_col[0] * zo + p.b_col[1] * zi);
  T acc[4][4] = {};
  // Causal K ranges at the tcgen05 kernel's 128-row tile granularity: the
  // softmax only writes the band the tensor-core kernel reads.
  const int base = (m0 / 128) * 128;
  int kbeg = 0, kend = p.K;
  if (p.causal == OASES_CAUSAL_K_UPTO_M) kend = min(p.K, base + 128);
  if (p.causal == OASES_CAUSAL_K_FROM_M) kbeg = base;
  for (int k0 = kbeg; k0 < kend; k0 += TK) {
    // 64x16 tile of A and of B: 1024 elements, 4 per thread.
    for (int i = threadIdx.x; i < TM * TK; i += 256) {
      int mm, kk;
      if (p.a_mn) { mm = i % TM; kk = i / TM; } else { kk = i % TK; mm = i / TK; }
      const int m = m0 + mm, k = k0 + kk;
      T v = 0;
      if (m < p.M && k < kend) v = p.a_mn ? A[static_cast<long long>(k) * p.lda + m] : A[static_cast<long long>(m) * p.lda + k];
      As[kk][mm] = v;
    }
    for (int i = threadIdx.x; i < TN * TK; i += 256) {
      int nn, kk;
      if (p.b_mn) { nn = i % TN; kk = i / TN; } else { kk = i % TK; nn = i / TK; }
      const int n = n0 + nn, k = k0 + kk;
      T v = 0;
      if (n < p.N && k < kend) v = p.b_mn ? B[static_cast<long long>(k) * p.ldb + n] : B[static_cast<long long>(n) * p.ldb + k];
      Bs[kk][nn] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < TK; ++kk) {
      T a[4], b[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma_t(a[i], b[j], acc[i][j]);
    }
    __syncthreads();
  }
  const long long crow = p.c_row[0] * zo + p.c_row[1] * zi;
  const long long ccol = p.c_col[0] * zo + p.c_col[1] * zi;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty + 16 * i;
    if (m >= p.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx + 16 * j;
      if (n >= p.N) continue;
      const long long off = (crow + m) * p.ldc + ccol + n;
      T v = static_cast<T>(p.alpha) * acc[i][j];
      if ((p.epilogue == OASES_EPI_BIAS || p.epilogue == OASES_EPI_BIAS_GELU ||
           p.epilogue == OASES_EPI_BIAS_GELU_GRAD) && p.bias)
        v += p.bias[n];
      if (p.epilogue == OASES_EPI_DGELU) v *= gelu_grad_t(p.aux[off]);
      if (p.epilogue == OASES_EPI_MUL) v *= p.aux[off];
      if (p.epilogue == OASES_EPI_BIAS_GELU_GRAD) {
        p.c[off] = gelu_grad_t(v);
        p.c2[off] = gelu_t(v);
        continue;
      }
      if (p.accumulate) v += p.c[off];
      if (p.epilogue == OASES_EPI_BIAS_GELU && !p.c2) {
        p.c[off] = gelu_t(v);  // activation only
      } else {
        p.c[off] = v;
        if (p.epilogue == OASES_EPI_BIAS_GELU) p.c2[off] = gelu_t(v);
      }
    }
  }
}

}  // namespace

namespace {

template <typename T>
GemmStatus launch_simt(const oases_gemm_desc& d, cudaStream_t stream) {
  GemmStatus st;
  SimtParams<T> p{};
  p.M = static_cast<int>(d.M);
  p.N = static_cast<int>(d.N);
  p.K = static_cast<int>(d.K);
  p.batch_inner = static_cast<int>(d.batch_inner);
  p.a = static_cast<const T*>(d.a.ptr);
  p.lda = d.a.ld;
  p.a_mn = d.a.mn_major;
  p.b = static_cast<const T*>(d.b.ptr);
  p.ldb = d.b.ld;
  p.b_mn = d.b.mn_major;
  for (int i = 0; i < 2; ++i) {
    p.a_row[i] = d.a.row_off[i];
    p.a_col[i] = d.a.col_off[i];
    p.b_row[i] = d.b.row_off[i];
    p.b_col[i] = d.b.col_off[i];
    p.c_row[i] = d.c_row_off[i];
    p.c_col[i] = d.c_col_off[i];
  }
  p.c = static_cast<T*>(d.c);
  p.c2 = static_cast<T*>(d.c2);
  p.aux = static_cast<const T*>(d.aux);
  p.bias = static_cast<const T*>(d.bias);
  p.ldc = d.ldc;
  p.epilogue = d.epilogue;
  p.causal = d.causal;
  p.accumulate = d.accumulate;
  p.alpha = d.alpha;
  dim3 grid(static_cast<unsigned>((d.N + TN - 1) / TN), static_cast<unsigned>((d.M + TM - 1) / TM),
            static_cast<unsigned>(d.batch));
  gemm_simt_kernel<T><<<grid, 256, 0, stream>>>(p);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    st.err = std::string("gemm_simt launch: ") + cudaGetErrorString(e);
    st.cuda = true;
    return st;
  }
  st.ok = true;
  return st;
}

}  // namespace

GemmStatus gemm_simt(const oases_gemm_desc& d, cudaStream_t stream) {
  GemmStatus st;
  if (d.dtype != OASES_F32 && d.dtype != OASES_F64) {
    st.err = "gemm_simt: operands must be f32 or f64";
    return st;
  }
  if (d.c_dtype != d.dtype) {
    st.err = "gemm_simt: the output dtype must equal the operand dtype (f32 or f64)";
    return st;
  }
  if (d.colsum) {
    st.err = "gemm_simt: COLSUM partials are implemented on the bf16 tensor-core path only";
    return st;
  }
  if (d.epilogue == OASES_EPI_ROWDOT) {
    st.err = "gemm_simt: the ROWDOT epilogue is implemented on the bf16 tensor-core path only";
    return st;
  }
  if (d.M <= 0 || d.N <= 0 || d.K <= 0 || d.batch <= 0 || d.batch_inner <= 0) {
    st.err = "gemm_simt: empty problem";
    return st;
  }
  return d.dtype == OASES_F64 ? launch_simt<double>(d, stream) : launch_simt<float>(d, stream);
}

}  // namespace oases
