// ORACLE (test infrastructure only — never linked into the product).
// Literal restatement of the reference RNG, /root/reference/proj/include/ngdb/
// common.hpp:60-127 (splitmix64 :60-66, Rng ctor :72-76, next :78, below :81-94,
// uniform :96-98, uniform(lo,hi) :100, gaussian :102-115, fork :117-121) and
// fnv1a64 :129-136. Pinned by tests/golden/rng_golden.json, produced by
// oracle/ref/rng_dump.cpp compiled against the reference header itself.
#pragma once

#include <cmath>
#include <cstdint>

namespace oracle {

struct OrRng {
  uint64_t s;
  double spare = 0.0;
  bool has_spare = false;

  static uint64_t mix(uint64_t& st) {
    st = st + 0x9e3779b97f4a7c15ULL;
    uint64_t z = st;
    z ^= z >> 30;
    z *= 0xbf58476d1ce4e5b9ULL;
    z ^= z >> 27;
    z *= 0x94d049bb133111ebULL;
    z ^= z >> 31;
    return z;
  }
  explicit OrRng(uint64_t seed) : s(seed) {
    mix(s);
    mix(s);
  }
  uint64_t next() { return mix(s); }
  uint64_t below(uint64_t n) {
    // Lemire: high 64 bits of x*n; reject while the low half < (2^64 mod n)
    uint64_t x = next();
    __uint128_t full = (__uint128_t)x * (__uint128_t)n;
    uint64_t low = (uint64_t)full;
    if (low < n) {
      uint64_t t = (uint64_t)(-n) % n;
      while (low < t) {
        x = next();
        full = (__uint128_t)x * (__uint128_t)n;
        low = (uint64_t)full;
      }
    }
    return (uint64_t)(full >> 64);
  }
  double uniform() { return (double)(next() >> 11) / 9007199254740992.0; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
  double gaussian() {
    if (has_spare) {
      has_spare = false;
      return spare;
    }
    double u1 = uniform(), u2 = uniform();
    while (u1 <= 1e-300) u1 = uniform();
    double r = std::sqrt(-2.0 * std::log(u1));
    spare = r * std::sin(6.283185307179586 * u2);
    has_spare = true;
    return r * std::cos(6.283185307179586 * u2);
  }
  OrRng fork(uint64_t tag) const {
    return OrRng(s ^ (0x6a09e667f3bcc909ULL + tag * 0x9e3779b97f4a7c15ULL));
  }
};

inline uint64_t or_fnv1a64(const char* p, size_t n) {
  uint64_t h = 1469598103934665603ULL;
  for (size_t i = 0; i < n; ++i) {
    h ^= (unsigned char)p[i];
    h *= 1099511628211ULL;
  }
  return h;
}

}  // namespace oracle
