// Test/bench-only: times the REFERENCE's own CPU implementation of the path --
// tmpsim::recompute_elision_equivalence (proj/src/numerics.cpp:234-256: sharded
// forward twice + backward twice through the toy TMP FFN) -- on host cores.
// Each OpenMP thread runs its own independent toy model (data parallel over
// samples), so the run uses every core the reference code can use.
//
// usage: ref_bench workers rows model_dim hidden min_seconds threads
// prints: {"calls": C, "seconds": S, "macs": M, "macs_per_s": R, "threads": T}
#include <omp.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "tmpsim/numerics.hpp"

int main(int argc, char** argv) {
  if (argc != 7) {
    std::fprintf(stderr, "usage: ref_bench workers rows model_dim hidden min_seconds threads\n");
    return 2;
  }
  const int w = std::atoi(argv[1]), rows = std::atoi(argv[2]), d = std::atoi(argv[3]), h = std::atoi(argv[4]);
  const double min_s = std::atof(argv[5]);
  const int threads = std::atoi(argv[6]);
  // MACs per call: 2 sharded forwards (2 matmuls each over the full hidden) and
  // 2 backwards (5 matmuls each: replayed pre, dW_out, dy, dW_in, dX).
  const double macs_per_call = 14.0 * rows * static_cast<double>(d) * h;
  long long calls = 0;
  const auto t0 = std::chrono::steady_clock::now();
  double elapsed = 0.0;
#pragma omp parallel num_threads(threads) reduction(+ : calls)
  {
    const auto model = tmpsim::make_toy_sharded_model(w, rows, d, h, 1234u + omp_get_thread_num());
    for (;;) {
      const auto chk = tmpsim::recompute_elision_equivalence(model);
      if (!chk.loss_bit_identical) std::abort();
      ++calls;
      const double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (s >= min_s) break;
    }
  }
  elapsed = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  std::printf("{\"calls\": %lld, \"seconds\": %.6f, \"macs\": %.6e, \"macs_per_s\": %.6e, \"threads\": %d}\n", calls,
              elapsed, calls * macs_per_call, calls * macs_per_call / elapsed, threads);
  return 0;
}
