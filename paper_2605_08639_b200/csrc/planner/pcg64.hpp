// numpy-compatible random streams for the annealing chains.
//
// reorder._run_chain (reorder.py:299-326) draws from
//   np.random.default_rng(np.random.SeedSequence(seed))   -> PCG64 (XSL-RR 128/64)
// using Generator.integers(0, E, size=2) (32-bit Lemire on the bit generator's buffered
// next_uint32: low half of a 64-bit draw first, high half kept for the next call) and
// Generator.random() ((next_uint64 >> 11) * 2^-53, which does not touch the 32-bit buffer).
// SeedSequence entropy mixing (pool of four u32 words, hashmix/mix constants) and
// PCG64 seeding (srandom with state = words[0:2], inc = words[2:4]) are reproduced here so
// a chain seeded with the same integer yields the same stream as numpy.
#pragma once
#include <cstdint>
#include <vector>

namespace mbp {

typedef unsigned __int128 u128;

class SeedSequence {
 public:
  explicit SeedSequence(uint64_t entropy) {
    std::vector<uint32_t> ent;
    if (entropy == 0) ent.push_back(0);
    while (entropy) {
      ent.push_back(static_cast<uint32_t>(entropy & 0xFFFFFFFFu));
      entropy >>= 32;
    }
    mix_entropy(ent);
  }
  // generate_state(n_words32) as uint32 words
  std::vector<uint32_t> generate_state(int n_words32) const {
    std::vector<uint32_t> out(n_words32);
    uint32_t hash_const = INIT_B;
    for (int i = 0; i < n_words32; ++i) {
      uint32_t v = pool_[i % kPool];
      v ^= hash_const;
      hash_const *= MULT_B;
      v *= hash_const;
      v ^= v >> XSHIFT;
      out[i] = v;
    }
    return out;
  }

 private:
  static constexpr int kPool = 4;
  static constexpr uint32_t INIT_A = 0x43b0d7e5u, MULT_A = 0x931e8875u, INIT_B = 0x8b51f9ddu, MULT_B = 0x58f38dedu;
  static constexpr uint32_t MIX_MULT_L = 0xca01f9ddu, MIX_MULT_R = 0x4973f715u, XSHIFT = 16;
  uint32_t pool_[kPool];

  static uint32_t hashmix(uint32_t value, uint32_t& hash_const) {
    value ^= hash_const;
    hash_const *= MULT_A;
    value *= hash_const;
    value ^= value >> XSHIFT;
    return value;
  }
  static uint32_t mix(uint32_t x, uint32_t y) {
    uint32_t r = MIX_MULT_L * x - MIX_MULT_R * y;
    r ^= r >> XSHIFT;
    return r;
  }
  void mix_entropy(const std::vector<uint32_t>& ent) {
    uint32_t hc = INIT_A;
    for (int i = 0; i < kPool; ++i) pool_[i] = hashmix(i < int(ent.size()) ? ent[i] : 0u, hc);
    for (int s = 0; s < kPool; ++s)
      for (int d = 0; d < kPool; ++d)
        if (s != d) pool_[d] = mix(pool_[d], hashmix(pool_[s], hc));
    for (size_t s = kPool; s < ent.size(); ++s)
      for (int d = 0; d < kPool; ++d) pool_[d] = mix(pool_[d], hashmix(ent[s], hc));
  }
};

class PCG64 {
 public:
  explicit PCG64(const SeedSequence& ss) {
    const std::vector<uint32_t> w = ss.generate_state(8);
    auto u64 = [&](int i) { return static_cast<uint64_t>(w[2 * i]) | (static_cast<uint64_t>(w[2 * i + 1]) << 32); };
    const u128 initstate = (static_cast<u128>(u64(0)) << 64) | u64(1);
    const u128 initseq = (static_cast<u128>(u64(2)) << 64) | u64(3);
    state_ = 0;
    inc_ = (initseq << 1) | 1u;
    step();
    state_ += initstate;
    step();
  }
  // raw generator state {state_hi, state_lo, inc_hi, inc_lo} (a fresh stream: no buffered half)
  void raw(uint64_t* out4) const {
    out4[0] = static_cast<uint64_t>(state_ >> 64);
    out4[1] = static_cast<uint64_t>(state_);
    out4[2] = static_cast<uint64_t>(inc_ >> 64);
    out4[3] = static_cast<uint64_t>(inc_);
  }
  uint64_t next64() {
    step();
    const uint64_t hi = static_cast<uint64_t>(state_ >> 64), lo = static_cast<uint64_t>(state_);
    const unsigned rot = static_cast<unsigned>(state_ >> 122);
    const uint64_t v = hi ^ lo;
    return (v >> rot) | (v << ((-rot) & 63));
  }
  uint32_t next32() {
    if (has32_) {
      has32_ = false;
      return buf32_;
    }
    const uint64_t n = next64();
    has32_ = true;
    buf32_ = static_cast<uint32_t>(n >> 32);
    return static_cast<uint32_t>(n & 0xFFFFFFFFu);
  }
  double random() { return static_cast<double>(next64() >> 11) * (1.0 / 9007199254740992.0); }
  // Generator.integers(0, n) for n <= 2^32 (bounded Lemire, numpy's rejection threshold)
  uint32_t bounded(uint32_t n) {
    const uint32_t rng = n - 1u;
    if (rng == 0) return 0;
    const uint32_t rng_excl = n;
    uint64_t m = static_cast<uint64_t>(next32()) * rng_excl;
    uint32_t left = static_cast<uint32_t>(m & 0xFFFFFFFFu);
    if (left < rng_excl) {
      const uint32_t threshold = (0xFFFFFFFFu - rng) % rng_excl;
      while (left < threshold) {
        m = static_cast<uint64_t>(next32()) * rng_excl;
        left = static_cast<uint32_t>(m & 0xFFFFFFFFu);
      }
    }
    return static_cast<uint32_t>(m >> 32);
  }

 private:
  static constexpr u128 kMult = (static_cast<u128>(0x2360ED051FC65DA4ull) << 64) | 0x4385DF649FCCF645ull;
  u128 state_, inc_;
  bool has32_ = false;
  uint32_t buf32_ = 0;
  void step() { state_ = state_ * kMult + inc_; }
};

}  // namespace mbp
