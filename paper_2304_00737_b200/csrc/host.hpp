// Host-side schedule logic and error model of the SparDL B200 path.
// Internal C++ (exceptions); the C ABI (abi.cpp) maps them to status codes.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "spardl_cuda.h"

namespace sdlh {

// One exception type carrying the reference's exception class as a status.
struct Error : std::runtime_error {
  int code;
  Error(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};
[[noreturn]] inline void fail(int code, const std::string& msg) { throw Error(code, msg); }

// inc/mathutil.hpp:21-44
inline bool is_pow2(int64_t x) { return x > 0 && (x & (x - 1)) == 0; }
inline int ceil_log2(int64_t x) {
  int t = 0;
  int64_t v = 1;
  while (v < x) {
    v <<= 1;
    ++t;
  }
  return t;
}
inline int exact_log2(int64_t x) {
  int t = 0;
  while (x > 1) {
    x >>= 1;
    ++t;
  }
  return t;
}

struct Partition {
  int64_t n = 0;
  int count = 0;
  std::vector<int64_t> lo, hi;
  int block_of(int64_t i) const;
};
Partition partition(int64_t n, int count);           // inc/sparse.hpp:98-117

struct Bags {                                        // inc/reduce_scatter.hpp:40-49
  int m = 1, rank = 0, l = 0, preservation = 0, remainder = 0;
  std::vector<std::vector<int>> bags;                // bags[j-1] = B_j
};
Bags build_bags(int m, int rank);                    // inc/reduce_scatter.hpp:51-74

void validate(const spardl_config& c);               // inc/pipeline.hpp:54-78
void expected_cost_sag(int64_t P, int64_t k, int64_t d, int mode, int64_t* rounds,
                       int64_t* low, int64_t* high); // inc/sag.hpp:295-329
std::vector<double> dyadic_shares(int count);        // inc/sag.hpp:108-118
void hctrl_init(spardl_hctrl* c, int64_t P, int64_t k, int64_t d);  // inc/sag.hpp:40-53
void hctrl_observe(spardl_hctrl* c, int64_t n_t);    // inc/sag.hpp:66-81
int64_t hctrl_budget(const spardl_hctrl* c);         // inc/sag.hpp:61-63

}  // namespace sdlh
