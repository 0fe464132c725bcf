// C++ drop-in check: code written against the reference's spardl:: API
// (/root/reference/proj/include/spardl) compiled unchanged against
// include/spardl/*.hpp and run on the GPU.  The cases are the reference's
// own known answers (tests/test_sparse.cpp, test_fabric.cpp,
// test_collectives.cpp) and SPEC examples, on fp32-representable values.
//
// Build: g++ -std=c++20 -Iinclude tests/cpp/test_dropin.cpp
//            -Lpaper_2304_00737_b200 -lspardl_cuda -Wl,-rpath,<dir>
#include <cstdio>
#include <random>
#include <sstream>

#include "spardl/pipeline.hpp"
#include "spardl/sparse.hpp"

using namespace spardl;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                        \
  do {                                                                     \
    if (cond) {                                                            \
      ++g_pass;                                                            \
    } else {                                                               \
      ++g_fail;                                                            \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);          \
    }                                                                      \
  } while (0)
template <class E, class F>
static bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

static SparseBlock make_block(int id, IndexRange r, std::vector<Entry> e) {
  SparseBlock b;
  b.block_id = id;
  b.range = r;
  b.entries = std::move(e);
  return b;
}

static void test_sparse() {
  // test_sparse.cpp:34-58
  auto r = top_k_select(make_block(0, {0, 3}, {{0, 3.0}, {1, -5.0}, {2, 2.0}}), 1);
  CHECK(r.selected.nnz() == 1 && r.selected.entries[0] == (Entry{1, -5.0}));
  CHECK(r.discarded.nnz() == 2 && r.discarded.entries[0] == (Entry{0, 3.0}));
  auto blk = make_block(0, {0, 10}, {{1, 0.5}, {4, -0.25}, {9, 2.0}});
  for (Index b : {3, 4, 100}) {
    auto x = top_k_select(blk, b);
    CHECK(x.selected == blk && x.discarded.empty());
  }
  auto t = top_k_select(make_block(0, {0, 3}, {{0, 2.0}, {1, -2.0}, {2, 1.0}}), 1);
  CHECK(t.selected.entries.size() == 1 && t.selected.entries[0] == (Entry{0, 2.0}));
  // partition (test_sparse.cpp:92-128)
  auto p = partition(7, 3);
  CHECK(p.ranges[0] == (IndexRange{0, 3}) && p.ranges[1] == (IndexRange{3, 5}) &&
        p.ranges[2] == (IndexRange{5, 7}));
  CHECK(throws<partition_error>([] { partition(5, 6); }));
  CHECK(p.block_of(4) == 1);
  // merge_add (test_sparse.cpp:130-160)
  auto m = merge_add(make_block(0, {0, 8}, {{1, 2.0}, {3, 1.0}}),
                     make_block(0, {0, 8}, {{3, 4.0}, {5, -1.0}}));
  CHECK(m.nnz() == 3 && m.entries[1] == (Entry{3, 5.0}) && m.entries[2] == (Entry{5, -1.0}));
  auto z = merge_add(make_block(0, {0, 4}, {{2, 1.5}}), make_block(0, {0, 4}, {{2, -1.5}}));
  CHECK(z.nnz() == 1 && z.entries[0] == (Entry{2, 0.0}));
  CHECK(throws<block_mismatch_error>(
      [] { merge_add(make_block(0, {0, 4}, {}), make_block(1, {4, 8}, {})); }));
  // integer associativity (test_sparse.cpp:181-193)
  std::mt19937_64 rng(29);
  for (int trial = 0; trial < 30; ++trial) {
    auto rb = [&] {
      SparseBlock b = make_block(0, {0, 24}, {});
      for (Index i = 0; i < 24; ++i)
        if (rng() % 2) b.entries.push_back({i, double(int(rng() % 19) - 9)});
      return b;
    };
    auto a = rb(), b = rb(), c = rb();
    CHECK(merge_add(merge_add(a, b), c) == merge_add(a, merge_add(b, c)));
  }
  // dense slice (test_sparse.cpp:195-206 flavour)
  GradientVector g(std::vector<double>{0.5, -3.0, 2.0, 0.25});
  auto s = top_k_select_slice(g, 0, {0, 4}, 2);
  CHECK(s.selected.entries.size() == 2 && s.selected.entries[0] == (Entry{1, -3.0}) &&
        s.selected.entries[1] == (Entry{2, 2.0}) && s.discarded.nnz() == 2);
}

static void test_fabric() {
  // test_fabric.cpp:42-52 and the ledger CSV golden string :140-149
  Fabric f(2);
  Fabric::RoundPlan plan(2);
  SparseBlock b = make_block(0, {0, 3}, {{0, 1.0}, {1, 1.0}, {2, 1.0}});
  plan[0] = Fabric::Send{1, {b}};
  f.exchange(std::move(plan));
  std::ostringstream os;
  write_ledger_csv(os, f);
  CHECK(os.str() == "worker_id,rounds,scalars_received\n0,1,0\n1,1,6\n");
  Fabric f3(3);
  Fabric::RoundPlan dup(3);
  dup[0] = Fabric::Send{2, {b}};
  dup[1] = Fabric::Send{2, {b}};
  CHECK(throws<schedule_violation_error>([&] { f3.exchange(std::move(dup)); }));
}

static void test_schedule_api() {
  auto s = build_bags(6, 0);
  CHECK(s.sending_bags.size() == 3 && s.sending_bags[2] == (std::vector<int>{4, 5}) &&
        s.remainder == 2);
  CHECK(expected_cost_srs(4, 200).rounds == 2 && expected_cost_srs(4, 200).scalars == 300);
  auto c = expected_cost_sag(8, 800, 2, SagMode::rsag);
  CHECK(c.rounds == 5 && c.scalars_low == 2800 && c.exact());
  auto b = expected_cost_sag(6, 600, 3, SagMode::bsag);
  CHECK(b.rounds == 4 && b.scalars_low == 600 && b.scalars_high == 2400);
  CHECK(topka_cost(4, 100).scalars_low == 600);
  HController h(6, 600, 3);
  h.observe(250);
  h.observe(250);
  h.observe(320);
  CHECK(h.h() == 104.0);
  CHECK(dyadic_shares(3) == (std::vector<double>{0.5, 0.25, 0.25}));
  ClusterConfig bad;
  bad.workers = 6;
  bad.dimension = 6000;
  bad.k = 601;
  try {
    validate(bad);
    CHECK(false);
  } catch (const config_error& e) {
    CHECK(std::string(e.what()) == "k must be divisible by P");
  }
}

static ClusterConfig config(std::int64_t P, std::int64_t N, std::int64_t k, std::int64_t d = 1,
                            SagMode sag = SagMode::none) {
  ClusterConfig c;
  c.workers = P;
  c.dimension = N;
  c.k = k;
  c.teams = d;
  c.sag = sag;
  return c;
}

static std::vector<GradientVector> int_grads(std::mt19937_64& rng, int P, Index N) {
  std::vector<GradientVector> g;
  for (int w = 0; w < P; ++w) {
    GradientVector v(N);
    for (Index i = 0; i < N; ++i) v[i] = double(int(rng() % 5) - 2);
    g.push_back(v);
  }
  return g;
}

static void test_pipeline() {
  std::mt19937_64 rng(7);
  {  // SPEC: P=6 d=1 k=600 N=6000 -> ledger (6, 2000), consistent, exact conservation
    auto cfg = config(6, 6000, 600);
    Fabric fabric(6);
    auto states = make_worker_states(cfg);
    for (int it = 0; it < 3; ++it) {
      auto r = spardl_all_reduce(fabric, cfg, int_grads(rng, 6, 6000), states);
      CHECK(r.consistent && r.conservation_error == 0.0 && r.global.nnz() <= cfg.k);
      if (it == 0) CHECK(r.ledger.max_rounds == 6 && r.ledger.max_scalars_received == 2000);
      CHECK(r.predicted.rounds == 6 && r.predicted.scalars_low == 2000);
    }
  }
  {  // Eq. 5: P=8 k=800 d=2 rsag -> (5, 2800)
    auto cfg = config(8, 8000, 800, 2, SagMode::rsag);
    Fabric fabric(8);
    auto states = make_worker_states(cfg);
    std::vector<GradientVector> g;
    std::uniform_real_distribution<double> mag(0.5, 1.5);
    for (int w = 0; w < 8; ++w) {
      GradientVector v(8000);
      for (Index i = 0; i < 8000; ++i)
        v[i] = double(float((rng() % 2 ? 1 : -1) * mag(rng)));
      g.push_back(v);
    }
    auto r = spardl_all_reduce(fabric, cfg, g, states);
    CHECK(r.consistent && r.ledger.max_rounds == 5 && r.ledger.max_scalars_received == 2800);
  }
  {  // Eq. 7 interval: P=6 k=600 d=3 bsag, 5 iterations with exact conservation
    auto cfg = config(6, 6000, 600, 3, SagMode::bsag);
    Fabric fabric(6);
    auto states = make_worker_states(cfg);
    for (int it = 0; it < 5; ++it) {
      auto r = spardl_all_reduce(fabric, cfg, int_grads(rng, 6, 6000), states);
      CHECK(r.consistent && r.conservation_error == 0.0 && r.union_sizes.size() == 2);
      const auto pc = bsag_phase_cost(6, 600, 3);   // the B-SAG phase interval
      CHECK(r.sag_phase.scalars >= pc.scalars_low && r.sag_phase.scalars <= pc.scalars_high);
      CHECK(states[0].controller->h() >= 100.0 && states[0].controller->h() <= 300.0);
    }
  }
  {  // P=1 -> the local top-k, zero ledger
    auto cfg = config(1, 100, 10);
    Fabric fabric(1);
    auto states = make_worker_states(cfg);
    auto g = int_grads(rng, 1, 100);
    auto r = spardl_all_reduce(fabric, cfg, g, states);
    auto local = top_k_select_slice(g[0], 0, {0, 100}, 10);
    CHECK(r.global.entries == local.selected.entries && r.ledger.max_rounds == 0);
  }
  {  // full density -> the dense sum
    auto cfg = config(4, 40, 40);
    Fabric fabric(4);
    auto states = make_worker_states(cfg);
    auto g = int_grads(rng, 4, 40);
    auto r = spardl_all_reduce(fabric, cfg, g, states);
    bool ok = r.global.nnz() == 40;
    for (const Entry& e : r.global.entries)
      ok &= e.value == g[0][e.index] + g[1][e.index] + g[2][e.index] + g[3][e.index];
    CHECK(ok);
  }
}

static void test_reporting() {
  {  // Top-kA (inc/collectives.hpp:185-216): union of the local top-2s, Bruck ledger
    Fabric fabric(3);
    std::vector<GradientVector> g(3, GradientVector(6));
    const double v[3][6] = {{5, -1, 0, 3, 0, 0}, {0, 4, 0, -3, 1, 0}, {-2, 0, 0, 0, 0, 7}};
    for (int w = 0; w < 3; ++w)
      for (int i = 0; i < 6; ++i) g[size_t(w)][i] = v[w][i];
    auto r = topka_baseline(fabric, g, 2);
    // locals: {0:5, 3:3}, {1:4, 3:-3}, {0:-2, 5:7} -> 0:3, 1:4, 3:0 (kept), 5:7
    CHECK(r.size() == 3 && r[0].entries == r[2].entries);
    CHECK(r[0].nnz() == 4 && r[0].entries[0] == (Entry{0, 3.0}) &&
          r[0].entries[2] == (Entry{3, 0.0}) && r[0].entries[3] == (Entry{5, 7.0}));
    CHECK(fabric.report().max_rounds == 2 && fabric.report().max_scalars_received == 8);
    CHECK(throws<config_error>([&] { topka_baseline(fabric, g, 7); }));
  }
  {  // run report / controller trace CSV (inc/pipeline.hpp:344-361, inc/sag.hpp:349-358)
    ClusterConfig cfg;
    cfg.workers = 6;
    cfg.dimension = 6000;
    cfg.k = 600;
    RunResult r;
    r.ledger.max_rounds = 6;
    r.ledger.max_scalars_received = 2000;
    r.predicted = {6, 2000, 2000};
    r.consistent = true;
    std::ostringstream os;
    write_run_report_header(os);
    write_run_report_row(os, cfg, r);
    CHECK(os.str() == "P,N,k,d,sag,residual,timing,seed,max_rounds,max_scalars,"
                      "predicted_rounds,predicted_scalars_low,predicted_scalars_high,"
                      "consistent,conservation_error\n6,6000,600,1,none,gres,optimized,0,6,2000,"
                      "6,2000,2000,1,0\n");
    HController c(6, 600, 3);
    std::ostringstream t;
    write_controller_trace_header(t);
    write_controller_trace_row(t, 0, c, 199);
    CHECK(t.str().rfind("iteration,h,step,flag,N_t,L\n0,100,", 0) == 0);
  }
}

int main() {
  test_sparse();
  test_reporting();
  test_fabric();
  test_schedule_api();
  test_pipeline();
  std::printf("dropin: %d passed, %d failed\n", g_pass, g_fail);
  return g_fail == 0 ? 0 : 1;
}
