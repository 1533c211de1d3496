// Golden-vector generator compiled AGAINST THE REFERENCE HEADER
// (/root/reference/proj/include/ngdb/common.hpp, via -I in oracle/ref/Makefile).
// Output: tests/golden/rng_golden.json (committed). Pins the RNG bit-stream,
// fnv1a64 and hex_u64 that the oracle and the product both restate.
#include <cinttypes>
#include <cstdio>
#include <string>

#include "ngdb/common.hpp"

static void emit_u64_list(const char* key, const uint64_t* v, int n, bool last = false) {
  std::printf("  \"%s\": [", key);
  for (int i = 0; i < n; ++i) std::printf("%s\"%" PRIu64 "\"", i ? ", " : "", v[i]);
  std::printf("]%s\n", last ? "" : ",");
}
static void emit_f64_list(const char* key, const double* v, int n) {
  std::printf("  \"%s\": [", key);
  for (int i = 0; i < n; ++i) std::printf("%s%.17g", i ? ", " : "", v[i]);
  std::printf("],\n");
}

int main() {
  std::printf("{\n  \"source\": \"/root/reference/proj/include/ngdb/common.hpp\",\n");
  const uint64_t seeds[] = {0, 1, 2, 3, 42, 0xdeadbeefULL, 18446744073709551615ULL};
  uint64_t buf[64];
  double dbuf[64];
  char key[128];
  for (uint64_t seed : seeds) {
    ngdb::Rng r(seed);
    for (int i = 0; i < 8; ++i) buf[i] = r.next();
    std::snprintf(key, sizeof key, "next_seed_%" PRIu64, seed);
    emit_u64_list(key, buf, 8);
  }
  {
    const uint64_t ns[] = {1, 2, 3, 7, 100, 14505, 63361, 2500604, 1000000007ULL,
                           (1ULL << 63) + 1, 18446744073709551615ULL};
    ngdb::Rng r(42);
    int k = 0;
    for (uint64_t n : ns)
      for (int i = 0; i < 4; ++i) buf[k++] = r.below(n);
    emit_u64_list("below_seed_42", buf, k);
  }
  {
    ngdb::Rng r(7);
    for (int i = 0; i < 8; ++i) dbuf[i] = r.uniform();
    emit_f64_list("uniform_seed_7", dbuf, 8);
    for (int i = 0; i < 8; ++i) dbuf[i] = r.uniform(-0.035, 0.035);
    emit_f64_list("uniform_pm_seed_7_cont", dbuf, 8);
  }
  {
    ngdb::Rng r(9);
    for (int i = 0; i < 9; ++i) dbuf[i] = r.gaussian();
    emit_f64_list("gaussian_seed_9", dbuf, 9);
  }
  {
    ngdb::Rng base(3);
    const uint64_t tags[] = {0, 1, 2, 511, 12345};
    int k = 0;
    for (uint64_t t : tags) {
      ngdb::Rng f = base.fork(t);
      buf[k++] = f.next();
      buf[k++] = f.below(14505);
    }
    emit_u64_list("fork_seed_3", buf, k);
  }
  {
    const char* strs[] = {"", "a", "ngdb", "backbone=gqe;d=400;batch=512"};
    for (int i = 0; i < 4; ++i) buf[i] = ngdb::fnv1a64(strs[i]);
    emit_u64_list("fnv1a64", buf, 4);
    std::printf("  \"hex_u64_255\": \"%s\",\n", ngdb::hex_u64(255).c_str());
  }
  {
    // the SURVEY §0 known answer: Rng(42).next(), then below(14505)
    ngdb::Rng r(42);
    buf[0] = r.next();
    buf[1] = r.below(14505);
    emit_u64_list("survey_known_answer", buf, 2, true);
  }
  std::printf("}\n");
  return 0;
}
