// f64 device kernels behind the reference's value-level numerics API
// (proj/include/tmpsim/numerics.hpp:10-60; runtime/numerics.cpp drives them).
//
// Every kernel reproduces the reference's scalar arithmetic element for
// element -- round-to-nearest multiplies and adds with no FMA contraction, the
// reference's summation order where it sums -- so the device results equal the
// CPU reference's bit for bit except where a libm function (erf, exp inside
// GeLU) is evaluated by the CUDA math library instead of glibc (<= 2 ulp).
#include "common.cuh"
#include "kernels.h"

namespace oases {
namespace {

constexpr int kThreads = 256;

unsigned blocks_for(long long n) {
  long long g = (n + kThreads - 1) / kThreads;
  if (g > 148LL * 8) g = 148LL * 8;
  return static_cast<unsigned>(g < 1 ? 1 : g);
}

// numerics.cpp:34-46,66-76
__global__ void map_f64_kernel(int op, const double* __restrict__ a, const double* __restrict__ b,
                               double* __restrict__ out, long long n) {
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const double x = a[i];
    double r;
    switch (op) {
      case F64_ADD: r = __dadd_rn(x, b[i]); break;
      case F64_HADAMARD: r = __dmul_rn(x, b[i]); break;
      case F64_GELU: r = gelu_d(x); break;
      default: r = gelu_grad_d(x); break;
    }
    out[i] = r;
  }
}

// numerics.cpp:26-32
__global__ void transpose_f64_kernel(const double* __restrict__ a, double* __restrict__ t, int rows, int cols) {
  const long long n = static_cast<long long>(rows) * cols;
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int r = static_cast<int>(i / cols), c = static_cast<int>(i % cols);
    t[static_cast<long long>(c) * rows + r] = a[i];
  }
}

// max |a - b| (numerics.cpp:78-85): max is order-independent, so a tree is exact
__global__ void max_abs_diff_kernel(const double* __restrict__ a, const double* __restrict__ b, long long n,
                                    double* __restrict__ out) {
  __shared__ double sm[kThreads];
  double m = 0.0;
  for (long long i = threadIdx.x; i < n; i += kThreads) m = fmax(m, fabs(__dadd_rn(a[i], -b[i])));
  sm[threadIdx.x] = m;
  __syncthreads();
  for (int w = kThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sm[threadIdx.x] = fmax(sm[threadIdx.x], sm[threadIdx.x + w]);
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sm[0];
}

// allreduce_grad_identity's central differences (numerics.cpp:87-134): one
// thread per (worker i, element e) evaluates phi(reduce(bumped)) at +-h with the
// reference's loop order (literal sum over workers in order 0..w-1, then phi
// summed over elements in index order); x is [w][n], weights [n].
__global__ void grad_identity_fd_kernel(const double* __restrict__ x, const double* __restrict__ weights, int w,
                                        int n, double h, double* __restrict__ fd) {
  const int t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= w * n) return;
  const int bi = t / n, be = t % n;
  double phi[2];
  for (int side = 0; side < 2; ++side) {
    // bumped[i](r,c) += h, then -= 2h: the reference's bump arithmetic
    const double xb = x[static_cast<long long>(bi) * n + be];
    const double up = __dadd_rn(xb, h);
    const double bumped = side == 0 ? up : __dadd_rn(up, -2.0 * h);
    double acc = 0.0;
    for (int e = 0; e < n; ++e) {
      double y = 0.0;  // reduce: y = 0 + x_0 + x_1 + ...
      for (int k = 0; k < w; ++k) y = __dadd_rn(y, (k == bi && e == be) ? bumped : x[static_cast<long long>(k) * n + e]);
      acc = __dadd_rn(acc, __dadd_rn(__dmul_rn(weights[e], y), __dmul_rn(__dmul_rn(0.5, y), y)));
    }
    phi[side] = acc;
  }
  fd[t] = __ddiv_rn(__dadd_rn(phi[0], -phi[1]), 2.0 * h);
}

}  // namespace

cudaError_t map_f64(int op, const double* a, const double* b, double* out, long long n, cudaStream_t st) {
  map_f64_kernel<<<blocks_for(n), kThreads, 0, st>>>(op, a, b, out, n);
  return cudaGetLastError();
}

cudaError_t transpose_f64(const double* a, double* t, int rows, int cols, cudaStream_t st) {
  transpose_f64_kernel<<<blocks_for(static_cast<long long>(rows) * cols), kThreads, 0, st>>>(a, t, rows, cols);
  return cudaGetLastError();
}

cudaError_t max_abs_diff_f64(const double* a, const double* b, long long n, double* out, cudaStream_t st) {
  max_abs_diff_kernel<<<1, kThreads, 0, st>>>(a, b, n, out);
  return cudaGetLastError();
}

cudaError_t grad_identity_fd_f64(const double* x, const double* weights, int workers, int n, double h, double* fd,
                                 cudaStream_t st) {
  const int total = workers * n;
  grad_identity_fd_kernel<<<(total + 127) / 128, 128, 0, st>>>(x, weights, workers, n, h, fd);
  return cudaGetLastError();
}

}  // namespace oases
