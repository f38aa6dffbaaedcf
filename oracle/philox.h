// TEST INFRASTRUCTURE (oracle). Philox4x32-10 exactly as specified for the
// dropout masks of the B200 build: element e of a
// tensor under key (seed, offset) is kept iff byte (e & 15) of the 16 output
// bytes of Philox(counter = e >> 4 | offset << 64, key = seed) is >= thr8,
// thr8 = round(p * 256) clamped to [1, 255]; kept values scale by 256/(256-thr8).
#pragma once
#include <cstdint>

namespace oracle {

inline void philox4x32_10(uint64_t seed, uint64_t offset, uint64_t ctr, uint32_t out[4]) {
  uint32_t c[4] = {static_cast<uint32_t>(ctr), static_cast<uint32_t>(ctr >> 32), static_cast<uint32_t>(offset),
                   static_cast<uint32_t>(offset >> 32)};
  uint32_t k0 = static_cast<uint32_t>(seed), k1 = static_cast<uint32_t>(seed >> 32);
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = 0xD2511F53ull * c[0];
    const uint64_t p1 = 0xCD9E8D57ull * c[2];
    const uint32_t n0 = static_cast<uint32_t>(p1 >> 32) ^ c[1] ^ k0;
    const uint32_t n1 = static_cast<uint32_t>(p1);
    const uint32_t n2 = static_cast<uint32_t>(p0 >> 32) ^ c[3] ^ k1;
    const uint32_t n3 = static_cast<uint32_t>(p0);
    c[0] = n0; c[1] = n1; c[2] = n2; c[3] = n3;
    if (r < 9) { k0 += 0x9E3779B9u; k1 += 0xBB67AE85u; }
  }
  for (int i = 0; i < 4; ++i) out[i] = c[i];
}

inline uint32_t keep_threshold(float p) {
  if (!(p > 0.f)) return 0u;
  int t = static_cast<int>(p * 256.f + 0.5f);
  return static_cast<uint32_t>(t < 1 ? 1 : (t > 255 ? 255 : t));
}

inline double keep_scale(float p) {
  const uint32_t t = keep_threshold(p);
  return t ? 256.0 / (256.0 - t) : 1.0;
}

inline bool keep(uint64_t seed, uint64_t offset, uint64_t e, uint32_t thr) {
  uint32_t u[4];
  philox4x32_10(seed, offset, e >> 4, u);
  const unsigned b = static_cast<unsigned>(e & 15);
  return ((u[b >> 2] >> (8 * (b & 3))) & 0xFFu) >= thr;
}

}  // namespace oracle
