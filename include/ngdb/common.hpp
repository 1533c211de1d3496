// ngdb/common.hpp — error taxonomy, portable RNG and hashing helpers.
//
// Drop-in for the reference interface /root/reference/proj/include/ngdb/common.hpp:
//   * ngdb::Error and the 25 per-module subclasses   (common.hpp:12-56)
//   * splitmix64 / Rng{next, below, uniform, gaussian, fork} with the SAME bit-stream
//                                                     (common.hpp:60-127)
//   * fnv1a64 / hex_u64                               (common.hpp:129-142)
// The RNG stream is part of the bit-exact contract (sampled indices, negatives,
// parameter init); tests/golden/rng_golden.json pins it against the reference
// header compiled by oracle/ref/Makefile.
#pragma once

#include <cmath>
#include <cstdint>
#include <cstdio>
#include <stdexcept>
#include <string>
#include <string_view>

namespace ngdb {

class Error : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

// Error taxonomy, grouped by the SPEC module that raises it.
#define NGDB_ERROR_LIST(X)                                              \
  /* kg-store     */ X(MissingFile) X(MalformedLine) X(IdOutOfRange)    \
                     X(UnsupportedPattern)                              \
  /* query-model  */ X(ArityMismatch) X(NotAUnionPattern)               \
  /* sampler      */ X(ExhaustedRetries) X(NonFiniteLoss)               \
  /* tensor-arena */ X(ZeroRefcount) X(DoubleRelease) X(IndexOutOfRange) \
  /* kernels      */ X(ShapeMismatch) X(ParamOutOfRange) X(DomainError) \
  /* scheduler    */ X(AllPoolsEmpty) X(MissingKernel)                  \
  /* trainer      */ X(NoNegativesAvailable) X(NonFinite) X(BadMagic)   \
                     X(CountMismatch) X(TruncatedFile)                  \
  /* evaluator    */ X(TargetFiltered) X(BackboneMismatch)              \
  /* cli          */ X(ConfigError) X(UnknownSubcommand)

#define NGDB_DECLARE_ERROR_CLASS(Name) \
  struct Name : ::ngdb::Error {        \
    using ::ngdb::Error::Error;        \
  };
NGDB_ERROR_LIST(NGDB_DECLARE_ERROR_CLASS)
#undef NGDB_DECLARE_ERROR_CLASS

// SplitMix64 step (Steele/Lea/Flood). Advances `state` and returns the mix.
inline uint64_t splitmix64(uint64_t& state) {
  constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ULL;
  constexpr uint64_t kMul1 = 0xbf58476d1ce4e5b9ULL;
  constexpr uint64_t kMul2 = 0x94d049bb133111ebULL;
  state += kGolden;
  uint64_t x = state;
  x = (x ^ (x >> 30)) * kMul1;
  x = (x ^ (x >> 27)) * kMul2;
  return x ^ (x >> 31);
}

// Deterministic generator; every draw algorithm is spelled out so the stream is
// identical on every platform (std:: distributions are implementation-defined).
class Rng {
 public:
  explicit Rng(uint64_t seed) : state_(seed) {
    // two discarded outputs decorrelate neighbouring seeds
    for (int i = 0; i < 2; ++i) (void)next();
  }

  uint64_t next() { return splitmix64(state_); }

  // Uniform integer in [0, n): Lemire's nearly-divisionless multiply-shift.
  uint64_t below(uint64_t n) {
    unsigned __int128 prod = static_cast<unsigned __int128>(next()) * n;
    uint64_t low = static_cast<uint64_t>(prod);
    if (low < n) {
      const uint64_t reject_under = (0ULL - n) % n;
      while (low < reject_under) {
        prod = static_cast<unsigned __int128>(next()) * n;
        low = static_cast<uint64_t>(prod);
      }
    }
    return static_cast<uint64_t>(prod >> 64);
  }

  // 53-bit mantissa uniform in [0, 1).
  double uniform() { return 0x1.0p-53 * static_cast<double>(next() >> 11); }
  double uniform(double lo, double hi) { return lo + uniform() * (hi - lo); }

  // Box-Muller pair; the second value is cached for the next call.
  double gaussian() {
    if (cached_) {
      cached_ = false;
      return cache_;
    }
    double u1 = uniform();
    const double u2 = uniform();
    while (u1 <= 1e-300) u1 = uniform();
    const double radius = std::sqrt(-2.0 * std::log(u1));
    const double angle = 6.283185307179586 * u2;
    cache_ = radius * std::sin(angle);
    cached_ = true;
    return radius * std::cos(angle);
  }

  // Independent child stream (one per producer worker / batch / rank).
  Rng fork(uint64_t tag) const {
    const uint64_t child = state_ ^ (0x6a09e667f3bcc909ULL + tag * 0x9e3779b97f4a7c15ULL);
    return Rng(child);
  }

 private:
  uint64_t state_;
  double cache_ = 0.0;
  bool cached_ = false;
};

// FNV-1a 64-bit (config hashes echoed into every artefact).
inline uint64_t fnv1a64(std::string_view bytes) {
  uint64_t h = 0xcbf29ce484222325ULL;  // 1469598103934665603
  for (const unsigned char b : bytes) h = (h ^ b) * 0x100000001b3ULL;
  return h;
}

inline std::string hex_u64(uint64_t v) {
  char out[17];
  std::snprintf(out, sizeof out, "%016llx", static_cast<unsigned long long>(v));
  return std::string(out);
}

}  // namespace ngdb
