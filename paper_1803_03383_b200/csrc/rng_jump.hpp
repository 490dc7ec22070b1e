// rng_jump.hpp -- GF(2) jump-ahead for the reference's xorshift64* stream.
//
// QuantRng (proj/include/lpopt/rng.hpp:27-64) advances its state with
//   s ^= s >> 12; s ^= s << 25; s ^= s >> 27
// which is linear over GF(2): s_{k} = X^k s_0 for a fixed 64x64 bit matrix X.
// A matrix is stored by columns (col[b] = image of bit b); applying it is a
// XOR of the columns of the set bits, or -- faster -- of 8 byte-indexed
// tables of 256 words (tab[byte][v] = image of v << 8*byte).  The device
// kernels use these tables to start any thread at any draw of the stream,
// which makes the sequential reference stream counter-indexed.
#pragma once
#include <array>
#include <cstdint>
#include <vector>

namespace halp {

using Mat64 = std::array<uint64_t, 64>;  // columns

inline uint64_t xs_step_host(uint64_t s) {
  s ^= s >> 12;
  s ^= s << 25;
  s ^= s >> 27;
  return s;
}

inline uint64_t mat_apply(const Mat64& m, uint64_t v) {
  uint64_t r = 0;
  while (v) {
    const int b = __builtin_ctzll(v);
    r ^= m[b];
    v &= v - 1;
  }
  return r;
}

inline Mat64 mat_mul(const Mat64& a, const Mat64& b) {  // a after b
  Mat64 r{};
  for (int i = 0; i < 64; ++i) r[i] = mat_apply(a, b[i]);
  return r;
}

inline Mat64 mat_xs() {
  Mat64 m{};
  for (int i = 0; i < 64; ++i) m[i] = xs_step_host(1ULL << i);
  return m;
}

// 8 x 256 byte tables of a matrix
inline void mat_tables(const Mat64& m, uint64_t* tab /*2048*/) {
  for (int byte = 0; byte < 8; ++byte)
    for (int v = 0; v < 256; ++v) tab[byte * 256 + v] = mat_apply(m, (uint64_t)v << (8 * byte));
}

struct JumpTables {
  std::vector<Mat64> pow;      // X^(2^b), b = 0..63
  std::vector<uint64_t> flat;  // 64 x 2048 tables of pow[b]
  JumpTables() : pow(64), flat(64 * 2048) {
    pow[0] = mat_xs();
    for (int b = 1; b < 64; ++b) pow[b] = mat_mul(pow[b - 1], pow[b - 1]);
    for (int b = 0; b < 64; ++b) mat_tables(pow[b], flat.data() + (size_t)b * 2048);
  }
  uint64_t jump(uint64_t s, uint64_t count) const {
    for (int b = 0; count; ++b, count >>= 1)
      if (count & 1) s = mat_apply(pow[b], s);
    return s;
  }
  Mat64 power(uint64_t count) const {
    Mat64 r{};
    for (int i = 0; i < 64; ++i) r[i] = 1ULL << i;
    for (int b = 0; count; ++b, count >>= 1)
      if (count & 1) r = mat_mul(pow[b], r);
    return r;
  }
  static const JumpTables& get() {
    static const JumpTables t;
    return t;
  }
};

// QuantRng seeding (rng.hpp:12-18, 29-32)
inline uint64_t split_mix_host(uint64_t x) {
  x += 0x9E3779B97F4A7C15ULL;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ULL;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBULL;
  return x ^ (x >> 31);
}
inline uint64_t rng_seed_state(uint64_t seed, uint64_t stream) {
  uint64_t s = split_mix_host(seed ^ split_mix_host(stream ^ 0xA5A5A5A5A5A5A5A5ULL));
  return s == 0 ? 0x9E3779B97F4A7C15ULL : s;
}

}  // namespace halp
