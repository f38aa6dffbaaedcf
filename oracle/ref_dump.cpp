// Test-only: runs the REFERENCE tmpsim numerics (built from /root/reference by
// oracle/Makefile) and prints every tensor of its toy FFN checker as JSON, so
// tests/golden can pin the fp64 restatement (oracle/gpt_oracle.cpp) bit-exactly.
//
// The reference keeps sharded_forward/backward_from in an anonymous namespace
// (proj/src/numerics.cpp:156-212); this dumper re-drives the same sequence of
// PUBLIC reference primitives (matmul, gelu, gelu_grad, add, hadamard,
// transpose; numerics.hpp:21-27) in the same order, and also records the
// reference's own checker results (recompute_elision_equivalence,
// sharded_output_deviation, allreduce_grad_identity) for cross-checking.
//
// usage: ref_dump workers batch model_dim hidden seed
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "tmpsim/numerics.hpp"

using namespace tmpsim;

static void put_matrix(const char* name, const Matrix& m, bool comma = true) {
  std::printf("\"%s\": {\"rows\": %d, \"cols\": %d, \"data\": [", name, m.rows, m.cols);
  for (std::size_t i = 0; i < m.data.size(); ++i) std::printf("%s%.17g", i ? ", " : "", m.data[i]);
  std::printf("]}%s\n", comma ? "," : "");
}

int main(int argc, char** argv) {
  if (argc != 6) {
    std::fprintf(stderr, "usage: ref_dump workers batch model_dim hidden seed\n");
    return 2;
  }
  const int w = std::atoi(argv[1]), batch = std::atoi(argv[2]), d = std::atoi(argv[3]), h = std::atoi(argv[4]);
  const unsigned seed = static_cast<unsigned>(std::strtoul(argv[5], nullptr, 10));
  const ToyShardedModel model = make_toy_sharded_model(w, batch, d, h, seed);

  // forward: z = sum_i gelu(X W_in[i]) W_out[i]  (order of numerics.cpp:158-165)
  Matrix z(model.input.rows, model.w_out.front().cols);
  std::vector<Matrix> pres, ys;
  for (int i = 0; i < w; ++i) {
    Matrix pre = matmul(model.input, model.w_in[i]);
    Matrix y = gelu(pre);
    z = add(z, matmul(y, model.w_out[i]));
    pres.push_back(pre);
    ys.push_back(y);
  }
  // loss head (numerics.cpp:175-188)
  const Matrix gz = gelu(z);
  double loss = 0.0;
  for (double v : gz.data) loss += 0.5 * v * v;
  const Matrix grad_z = hadamard(gelu(z), gelu_grad(z));
  // backward (numerics.cpp:192-210)
  Matrix grad_x(model.input.rows, model.input.cols);
  std::vector<Matrix> dwin, dwout;
  for (int i = 0; i < w; ++i) {
    const Matrix pre = matmul(model.input, model.w_in[i]);
    const Matrix y = gelu(pre);
    dwout.push_back(matmul(transpose(y), grad_z));
    const Matrix grad_y = matmul(grad_z, transpose(model.w_out[i]));
    const Matrix grad_pre = hadamard(grad_y, gelu_grad(pre));
    dwin.push_back(matmul(transpose(model.input), grad_pre));
    grad_x = add(grad_x, matmul(grad_pre, transpose(model.w_in[i])));
  }
  const ElisionCheck ec = recompute_elision_equivalence(model);
  const double dev = sharded_output_deviation(model);

  std::printf("{\n\"workers\": %d, \"batch\": %d, \"model_dim\": %d, \"hidden\": %d, \"seed\": %u,\n", w, batch, d,
              h, seed);
  put_matrix("input", model.input);
  for (int i = 0; i < w; ++i) {
    put_matrix(("w_in_" + std::to_string(i)).c_str(), model.w_in[i]);
    put_matrix(("w_out_" + std::to_string(i)).c_str(), model.w_out[i]);
    put_matrix(("pre_" + std::to_string(i)).c_str(), pres[i]);
    put_matrix(("y_" + std::to_string(i)).c_str(), ys[i]);
    put_matrix(("grad_w_in_" + std::to_string(i)).c_str(), dwin[i]);
    put_matrix(("grad_w_out_" + std::to_string(i)).c_str(), dwout[i]);
  }
  put_matrix("z", z);
  put_matrix("grad_z", grad_z);
  put_matrix("grad_input", grad_x);
  std::printf("\"loss\": %.17g,\n", loss);
  std::printf("\"ref_elision_grad_deviation\": %.17g, \"ref_elision_loss_bit_identical\": %s,\n",
              ec.grad_deviation, ec.loss_bit_identical ? "true" : "false");
  std::printf("\"ref_sharded_output_deviation\": %.17g\n}\n", dev);
  return 0;
}
