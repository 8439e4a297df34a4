// Host check of the pool-bound selection network (tb_common.cuh kth_of_32):
// the 16th and 12th smallest of 32 keys, against std::nth_element, on random,
// duplicate-heavy and all-unset (0xFFFFFFFF) inputs.  Built and run by
// tests/test_native_helpers.py with nvcc (host code only, no GPU needed).
#include <algorithm>
#include <cstdio>
#include <random>
#include "../../paper_2206_14148_b200/csrc/tb_common.cuh"

namespace tb {
void set_error(const std::string&) {}
int fail(int code, const std::string&) { return code; }
}  // namespace tb

int main() {
  std::mt19937 rng(7);
  for (int trial = 0; trial < 200000; ++trial) {
    unsigned v[32], w[32];
    const int mode = trial % 4;
    for (int i = 0; i < 32; ++i) {
      unsigned x = rng();
      if (mode == 1) x &= 7u;                                  // many ties
      if (mode == 2) x = (rng() % 3 == 0) ? 0xFFFFFFFFu : x;   // unset slots
      if (mode == 3) x = 0xFFFFFFFFu;
      v[i] = w[i] = x;
    }
    unsigned v2[32];
    for (int i = 0; i < 32; ++i) v2[i] = v[i];
    std::nth_element(w, w + 15, w + 32);
    const unsigned got = tb::kth_of_32<16>(v);
    if (got != w[15]) {
      std::printf("FAIL K=16 trial %d: got %u want %u\n", trial, got, w[15]);
      return 1;
    }
    std::nth_element(w, w + 11, w + 32);
    const unsigned got12 = tb::kth_of_32<12>(v2);
    if (got12 != w[11]) {
      std::printf("FAIL K=12 trial %d: got %u want %u\n", trial, got12, w[11]);
      return 1;
    }
  }
  std::printf("OK\n");
  return 0;
}
