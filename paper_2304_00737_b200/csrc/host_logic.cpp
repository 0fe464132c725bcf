// Host-side schedule logic: config validation, block partition, bag
// schedule, closed-form costs, dyadic shares and the B-SAG controller.
// Each function restates the reference function cited next to it; the
// error messages are the reference's, verbatim.
#include <algorithm>
#include <cmath>
#include <functional>

#include "host.hpp"

namespace sdlh {

int Partition::block_of(int64_t i) const {      // inc/sparse.hpp:88-95
  const int64_t base = n / count, rem = n % count;
  const int64_t split = rem * (base + 1);
  if (i < split) return static_cast<int>(i / (base + 1));
  return static_cast<int>(rem + (i - split) / base);
}

Partition partition(int64_t n, int count) {     // inc/sparse.hpp:98-117
  if (count <= 0 || static_cast<int64_t>(count) > n) {
    fail(SPARDL_E_PARTITION, "partition requires 1 <= B <= N, got B=" + std::to_string(count) +
                                 " N=" + std::to_string(n));
  }
  Partition p;
  p.n = n;
  p.count = count;
  const int64_t base = n / count, rem = n % count;
  int64_t lo = 0;
  for (int b = 0; b < count; ++b) {
    const int64_t len = base + (b < rem ? 1 : 0);
    p.lo.push_back(lo);
    p.hi.push_back(lo + len);
    lo += len;
  }
  return p;
}

Bags build_bags(int m, int rank) {              // inc/reduce_scatter.hpp:51-74
  if (m < 1 || rank < 0 || rank >= m) fail(SPARDL_E_CONFIG, "build_bags: rank out of range");
  Bags s;
  s.m = m;
  s.rank = rank;
  s.preservation = rank;
  s.l = ceil_log2(m);
  if (m == 1) return s;
  s.remainder = m - (1 << (s.l - 1));
  s.bags.resize(static_cast<size_t>(s.l));
  int next = rank + 1;
  for (int j = 1; j <= s.l; ++j) {
    const int size = (j < s.l) ? (1 << (j - 1)) : s.remainder;
    for (int q = 0; q < size; ++q) {
      s.bags[static_cast<size_t>(j - 1)].push_back(next % m);
      ++next;
    }
  }
  return s;
}

void validate(const spardl_config& c) {         // inc/pipeline.hpp:54-78
  if (c.workers < 1) fail(SPARDL_E_CONFIG, "P must be >= 1");
  if (c.dimension < 1) fail(SPARDL_E_CONFIG, "N must be >= 1");
  if (c.k < 1 || c.k > c.dimension) fail(SPARDL_E_CONFIG, "k must satisfy 1 <= k <= N");
  if (c.k % c.workers != 0) fail(SPARDL_E_CONFIG, "k must be divisible by P");
  if (c.teams < 1 || c.workers % c.teams != 0) fail(SPARDL_E_CONFIG, "d must divide P");
  if (c.sag == SPARDL_SAG_NONE && c.teams != 1) fail(SPARDL_E_CONFIG, "sag=none requires d=1");
  if (c.sag != SPARDL_SAG_NONE && c.teams == 1) fail(SPARDL_E_CONFIG, "d=1 requires sag=none");
  if (c.sag == SPARDL_SAG_RSAG && !is_pow2(c.teams))
    fail(SPARDL_E_CONFIG, "rsag requires power-of-two d");
  if (c.workers / c.teams > c.dimension) fail(SPARDL_E_CONFIG, "N must allow P/d blocks (N >= P/d)");
  if (c.sag < 0 || c.sag > 2 || c.residual < 0 || c.residual > 2 || c.timing < 0 || c.timing > 1)
    fail(SPARDL_E_CONFIG, "unknown enum value in ClusterConfig");
}

void expected_cost_sag(int64_t workers, int64_t k, int64_t teams, int mode, int64_t* rounds,
                       int64_t* low, int64_t* high) {  // inc/sag.hpp:295-329
  if (workers < 1 || k < 1 || k % workers != 0)
    fail(SPARDL_E_CONFIG, "expected_cost_sag: k must be divisible by P");
  if (teams < 1 || workers % teams != 0) fail(SPARDL_E_CONFIG, "expected_cost_sag: d must divide P");
  const int64_t c = k / workers, p = workers, d = teams;
  switch (mode) {
    case SPARDL_SAG_NONE: {
      if (d != 1) fail(SPARDL_E_CONFIG, "expected_cost_sag: none requires d=1");
      const int64_t sc = 4 * c * (p - 1);
      *rounds = 2 * ceil_log2(p);
      *low = *high = sc;
      return;
    }
    case SPARDL_SAG_RSAG: {
      if (d < 2 || !is_pow2(d)) fail(SPARDL_E_CONFIG, "rsag requires power-of-two d");
      const int64_t lg = exact_log2(d);
      const int64_t sc = 2 * c * (2 * p - 2 * d) + 2 * c * d * lg;
      *rounds = 2 * ceil_log2(p / d) + lg;
      *low = *high = sc;
      return;
    }
    case SPARDL_SAG_BSAG: {
      if (d < 2) fail(SPARDL_E_CONFIG, "bsag requires d >= 2");
      const int64_t m = p / d;
      *rounds = 2 * ceil_log2(m) + ceil_log2(d);
      *low = 2 * c * (d + m - 2);
      *high = 2 * c * (d * d + 2 * p - 3 * d);
      return;
    }
  }
  fail(SPARDL_E_CONFIG, "expected_cost_sag: unknown mode");
}

std::vector<double> dyadic_shares(int count) {  // inc/sag.hpp:108-118
  std::vector<double> shares{1.0};
  while (static_cast<int>(shares.size()) < count) {
    const double half = shares.front() / 2.0;
    shares.erase(shares.begin());
    shares.push_back(half);
    shares.push_back(half);
    std::sort(shares.begin(), shares.end(), std::greater<double>());
  }
  return shares;
}

void hctrl_init(spardl_hctrl* c, int64_t workers, int64_t k, int64_t teams) {  // sag.hpp:40-53
  if (workers < 1 || teams < 1 || k < 1 || k % workers != 0 || (teams * k) % workers != 0)
    fail(SPARDL_E_CONFIG, "HController: invalid (P, k, d)");
  c->lower = static_cast<double>(k) / static_cast<double>(workers);
  c->upper = static_cast<double>(teams * k) / static_cast<double>(workers);
  c->target = teams * k / workers;
  c->h = c->lower;
  c->step = 0.01 * static_cast<double>(k) * static_cast<double>(teams - 1) /
            static_cast<double>(workers);
  c->flag = 0;
  c->pad_ = 0;
}

void hctrl_observe(spardl_hctrl* c, int64_t n_t) {  // inc/sag.hpp:66-81
  const bool over = n_t > c->target;
  const bool rising = c->step > 0.0;
  if (over != rising) {
    if (c->flag) {
      c->step *= 2.0;
      c->flag = 0;
    } else {
      c->flag = 1;
    }
  } else {
    c->step = -c->step / 2.0;
    c->flag = 0;
  }
  c->h = std::clamp(c->h + c->step, c->lower, c->upper);
}

int64_t hctrl_budget(const spardl_hctrl* c) {   // inc/sag.hpp:61-63
  return std::max<int64_t>(1, static_cast<int64_t>(std::llround(c->h)));
}

}  // namespace sdlh
