// ngdb/radix.hpp — LSD radix sort of 64-bit keys for the host planner.
//
// The sparse-gradient CSR of a step (plan_training_step, build_shard_plan) is a
// sort of ~76k packed (row, code) keys per 512-query step; std::sort spent
// ~8 ms of a ~10 ms plan on it. Keys here have ≤ 54 significant bits and many
// constant digits, so a counting sort over 11-bit digits that skips constant
// digit positions finishes in ~4–5 linear passes. The result is the ascending
// order of the keys, i.e. identical to std::sort.
//
// `start_bit` > 0 sorts stably by key >> start_bit only: when the low bits of
// the keys already ascend in input order within every high part (the planner
// emits codes in ascending order), the result is still the full ascending
// order, in fewer passes.
#pragma once

#include <array>
#include <cstdint>
#include <vector>

namespace ngdb {

inline void radix_sort_u64(std::vector<uint64_t>& keys, std::vector<uint64_t>& scratch,
                           int start_bit = 0) {
  constexpr int kBits = 11;
  constexpr uint32_t kBuckets = 1u << kBits, kMask = kBuckets - 1;
  const size_t n = keys.size();
  if (n < 2) return;
  uint64_t any = 0;
  for (const uint64_t k : keys) any |= k ^ keys[0];  // bits that vary
  any >>= start_bit;
  int kPasses = 0;
  while (any) {
    ++kPasses;
    any >>= kBits;
  }
  static thread_local std::vector<std::array<uint32_t, kBuckets>> hist;
  hist.assign(kPasses, {});
  for (const uint64_t k : keys)
    for (int p = 0; p < kPasses; ++p) ++hist[p][(k >> (start_bit + p * kBits)) & kMask];
  scratch.resize(n);
  uint64_t* src = keys.data();
  uint64_t* dst = scratch.data();
  for (int p = 0; p < kPasses; ++p) {
    auto& h = hist[p];
    const int shift = start_bit + p * kBits;
    if (h[(src[0] >> shift) & kMask] == n) continue;  // digit constant over all keys
    uint32_t sum = 0;
    for (uint32_t b = 0; b < kBuckets; ++b) {
      const uint32_t c = h[b];
      h[b] = sum;
      sum += c;
    }
    for (size_t i = 0; i < n; ++i) dst[h[(src[i] >> shift) & kMask]++] = src[i];
    std::swap(src, dst);
  }
  if (src != keys.data()) keys.swap(scratch);
}

inline void radix_sort_u64(std::vector<uint64_t>& keys, int start_bit = 0) {
  static thread_local std::vector<uint64_t> scratch;
  radix_sort_u64(keys, scratch, start_bit);
}

}  // namespace ngdb
