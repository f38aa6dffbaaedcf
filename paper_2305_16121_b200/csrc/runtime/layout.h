// Rank geometry of the TMP layer stack, host-only (no CUDA): which tokens,
// heads and weight columns a rank owns in each block, for uniform and mixed
// per-block degrees. The Stack computes every buffer
// offset and NCCL sub-communicator colour from these functions, and
// oases_rank_layout() exposes them through the C-ABI so the multi-rank
// partition can be checked without a device (tests/test_multirank_cpu.py).
//
// A degree-d block on a world of N ranks runs data-parallel on N/d groups of d
// ranks: group g = rank / d owns samples [g b d / N, (g+1) b d / N) of the
// micro-batch b (two sub-batches of b d / 2N samples), and inside the group the
// rank rank % d holds heads (or FFN columns) [r H/d, (r+1) H/d) like a
// uniform TMP rank of the reference's column/row split (numerics.cpp:120-165,
// the weight slicing of sharding.cpp). Degree-d tensor-parallel groups are the
// ncclCommSplit colour rank / d, their data-parallel complements colour rank % d.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "../../../include/oases/tmpsim.hpp"

namespace oases {

struct ModelCfg {
  int h = 0, f = 0, heads = 0, s = 0, b = 0, layers = 0;
  int bytes = 2;
  bool recompute = true, attention = true, ln = true, bias = true, residual = true;
  float p_hidden = 0.f, p_attn = 0.f, eps = 1e-5f;
  uint64_t seed = 0;
};

inline int num_blocks(const ModelCfg& c) { return c.layers * (c.attention ? 2 : 1); }
// block 2l is layer l's attention block when the layers have attention
inline bool attention_block(const ModelCfg& c, int block) { return c.attention && block % 2 == 0; }
inline int group_of(int rank, int d) { return rank / d; }
inline int rank_in_group(int rank, int d) { return rank % d; }
inline int64_t samples_per_sub(const ModelCfg& c, int world, int d) {
  return static_cast<int64_t>(c.b) * d / world / 2;
}
inline int64_t tokens_per_sub(const ModelCfg& c, int world, int d) { return samples_per_sub(c, world, d) * c.s; }
// first token row of the rank's group slice (two sub-batches of tokens_per_sub rows)
inline int64_t token_row0(const ModelCfg& c, int world, int d, int rank) {
  return static_cast<int64_t>(group_of(rank, d)) * 2 * tokens_per_sub(c, world, d);
}
inline int heads_local(const ModelCfg& c, int d) { return c.attention ? c.heads / d : 0; }
inline int head_dim(const ModelCfg& c) { return c.attention ? c.h / c.heads : 0; }
// local widths of the block's column-parallel (QKV | FC1) and row-parallel (proj | FC2) weights
inline int64_t col_width(const ModelCfg& c, int d, bool att) {
  return att ? 3LL * heads_local(c, d) * head_dim(c) : c.f / d;
}
inline int64_t row_width(const ModelCfg& c, int d, bool att) {
  return att ? static_cast<int64_t>(heads_local(c, d)) * head_dim(c) : c.f / d;
}

// The per-block degrees of a stack on `world` ranks (empty: every block at the
// world degree), validated; *mixed is set when any block runs below the world.
inline std::vector<int> resolve_degrees(const ModelCfg& c, int world, const std::vector<int>& degrees,
                                        bool* mixed) {
  using tmpsim::ConfigError;
  if (world < 1) throw ConfigError("layout: world size must be >= 1");
  const int nb = num_blocks(c);
  std::vector<int> deg;
  if (degrees.empty()) {
    deg.assign(static_cast<size_t>(nb), world);
  } else {
    if (static_cast<int>(degrees.size()) != nb) throw ConfigError("stack: one degree per block (" + std::to_string(nb) + ")");
    deg = degrees;
  }
  bool mx = false;
  for (int d : deg) {
    if (d < 1 || world % d)
      throw ConfigError("stack: every block degree must divide the world size " + std::to_string(world));
    if ((static_cast<int64_t>(c.b) * d) % (2LL * world))
      throw ConfigError("stack: a degree-" + std::to_string(d) + " block splits the micro-batch over " +
                        std::to_string(world / d) + " groups of two sub-batches: global_batch * d / world must be even");
    if (d != world) mx = true;
  }
  for (int blk = 0; blk < nb; ++blk) {
    const int d = deg[static_cast<size_t>(blk)];
    if (c.f % d) throw ConfigError("stack: ffn hidden must be divisible by the block degree");
    if (c.attention && (c.heads < 1 || c.h % c.heads || c.heads % d))
      throw ConfigError("stack: hidden % heads and heads % degree must be 0");
  }
  if (mixed) *mixed = mx;
  return deg;
}

}  // namespace oases
