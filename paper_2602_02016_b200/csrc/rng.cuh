// NumPy-compatible seeding and PCG64 streams, usable on host and device.
//
// The reference derives per-block power-iteration start vectors from
//   np.random.SeedSequence([seed, index]).generate_state(1, uint64)   (spectral.py:53-55)
//   np.random.default_rng(seed).uniform(-1, 1, size=(pool, n))        (spectral.py:67-74)
// i.e. NumPy's SeedSequence hash (pool size 4, 32-bit hashmix / mix) and the PCG64 XSL-RR generator
// (128-bit LCG, set_seq seeding from generate_state(4, uint64)), uniform doubles = (next64 >> 11) * 2^-53.
// This header restates those published algorithms so the B200 start vectors are bit-identical to the
// reference's (tests/test_rng.py checks against numpy).
#pragma once
#include <cstdint>

#ifdef __CUDACC__
#define RNG_HD __host__ __device__ __forceinline__
#else
#define RNG_HD inline
#endif

namespace dash {
namespace rng {

constexpr uint32_t kInitA = 0x43b0d7e5u, kMultA = 0x931e8875u, kInitB = 0x8b51f9ddu, kMultB = 0x58f38dedu;
constexpr uint32_t kMixL = 0xca01f9ddu, kMixR = 0x4973f715u;

RNG_HD uint32_t hashmix(uint32_t v, uint32_t& hc) {
  v ^= hc;
  hc *= kMultA;
  v *= hc;
  v ^= v >> 16;
  return v;
}
RNG_HD uint32_t mix(uint32_t x, uint32_t y) {
  uint32_t r = kMixL * x - kMixR * y;
  r ^= r >> 16;
  return r;
}

// SeedSequence(entropy words).generate_state(n64, uint64); entropy given as 32-bit words (little endian).
RNG_HD void seedseq(const uint32_t* ent, int nent, uint64_t* out, int n64) {
  uint32_t pool[4];
  uint32_t hc = kInitA;
  for (int i = 0; i < 4; ++i) pool[i] = hashmix(i < nent ? ent[i] : 0u, hc);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = mix(pool[d], hashmix(pool[s], hc));
  for (int s = 4; s < nent; ++s)
    for (int d = 0; d < 4; ++d) pool[d] = mix(pool[d], hashmix(ent[s], hc));
  uint32_t hb = kInitB;
  for (int i = 0; i < 2 * n64; ++i) {
    uint32_t v = pool[i & 3];
    v ^= hb;
    hb *= kMultB;
    v *= hb;
    v ^= v >> 16;
    if (i & 1) out[i >> 1] |= static_cast<uint64_t>(v) << 32;
    else out[i >> 1] = v;
  }
}

// Append the 32-bit words of a non-negative integer (NumPy's _int_to_uint32_array: 0 -> [0]).
RNG_HD int push_words(uint64_t x, uint32_t* w, int n) {
  if (x == 0) { w[n++] = 0; return n; }
  while (x) { w[n++] = static_cast<uint32_t>(x); x >>= 32; }
  return n;
}

// SeedSequence([a, b]).generate_state(1, uint64)[0]  (spectral.block_seed)
RNG_HD uint64_t block_seed(uint64_t a, uint64_t b) {
  uint32_t w[4];
  int n = push_words(a, w, 0);
  n = push_words(b, w, n);
  uint64_t out[1];
  seedseq(w, n, out, 1);
  return out[0];
}

typedef unsigned __int128 u128;
RNG_HD u128 pcg_mult() {
  return (static_cast<u128>(0x2360ED051FC65DA4ull) << 64) | 0x4385DF649FCCF645ull;
}

struct Pcg64 {
  u128 state, inc;
  // default_rng(seed): PCG64(SeedSequence(seed)) -> generate_state(4) -> set_seq seeding
  RNG_HD void seed(uint64_t s) {
    uint32_t w[2];
    int n = push_words(s, w, 0);
    uint64_t st[4];
    seedseq(w, n, st, 4);
    const u128 initstate = (static_cast<u128>(st[0]) << 64) | st[1];
    const u128 initseq = (static_cast<u128>(st[2]) << 64) | st[3];
    inc = (initseq << 1) | 1u;
    state = 0;
    step();
    state += initstate;
    step();
  }
  RNG_HD void step() { state = state * pcg_mult() + inc; }
  RNG_HD uint64_t next64() {
    step();
    const uint64_t x = static_cast<uint64_t>(state >> 64) ^ static_cast<uint64_t>(state);
    const unsigned rot = static_cast<unsigned>(state >> 122);
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }
  // jump ahead by `delta` draws (LCG power; Brown's algorithm)
  RNG_HD void advance(uint64_t delta) {
    u128 acc_mult = 1, acc_plus = 0, cur_mult = pcg_mult(), cur_plus = inc;
    while (delta) {
      if (delta & 1) {
        acc_mult *= cur_mult;
        acc_plus = acc_plus * cur_mult + cur_plus;
      }
      cur_plus = (cur_mult + 1) * cur_plus;
      cur_mult *= cur_mult;
      delta >>= 1;
    }
    state = acc_mult * state + acc_plus;
  }
  // Generator.uniform(-1, 1): low + (high - low) * next_double
  RNG_HD double uniform_pm1() { return -1.0 + 2.0 * (static_cast<double>(next64() >> 11) * (1.0 / 9007199254740992.0)); }
};

}  // namespace rng
}  // namespace dash
