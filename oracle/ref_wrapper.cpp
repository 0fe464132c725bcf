// oracle/ref_wrapper.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Exposes the UNMODIFIED reference implementation (the header-only C++20
// library under /root/reference/proj/include/spardl) through the same flat
// C API as oracle/spardl_oracle.c (orc_*), so tests can diff the C
// restatement against the reference itself and bench.py can time the
// reference's own CPU path (cpu_baseline kind "reference").
//
// Built by oracle/Makefile into oracle/_ref/libspardl_ref.so, only where
// /root/reference exists (this container); the built .so travels to the GPU
// box with the repo snapshot.  No reference source is copied into the repo:
// this file only #includes the headers in place.
#include <chrono>
#include <cstdint>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "spardl/spardl.hpp"

#define EXPORT extern "C" __attribute__((visibility("default")))

namespace {

thread_local std::string g_msg;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const spardl::partition_error& e) {
    g_msg = e.what();
    return 2;
  } catch (const spardl::block_mismatch_error& e) {
    g_msg = e.what();
    return 3;
  } catch (const spardl::schedule_violation_error& e) {
    g_msg = e.what();
    return 4;
  } catch (const spardl::theorem_violation_error& e) {
    g_msg = e.what();
    return 5;
  } catch (const spardl::group_size_error& e) {
    g_msg = e.what();
    return 6;
  } catch (const spardl::config_error& e) {
    g_msg = e.what();
    return 7;
  } catch (const spardl::state_error& e) {
    g_msg = e.what();
    return 8;
  } catch (const spardl::consistency_error& e) {
    g_msg = e.what();
    return 9;
  } catch (const spardl::error& e) {
    g_msg = e.what();
    return 1;
  }
}

}  // namespace

struct orc_config {
  int64_t workers, dimension, k, teams;
  int32_t sag, residual, timing, pad_;
  uint64_t seed;
};

struct orc_run_info {
  int32_t consistent, conservation_applicable;
  double conservation_error;
  int64_t max_rounds, max_scalars;
  int64_t srs_rounds, srs_scalars, sag_rounds, sag_scalars, gather_rounds, gather_scalars;
  int64_t pred_rounds, pred_low, pred_high;
  int64_t n_union;
  int64_t global_nnz;
};

struct orc_hctrl {
  double lower, upper;
  int64_t target;
  double h, step;
  int32_t flag;
  int32_t pad_;
};

static spardl::ClusterConfig to_cluster(const orc_config* c) {
  spardl::ClusterConfig cfg;
  cfg.workers = c->workers;
  cfg.dimension = c->dimension;
  cfg.k = c->k;
  cfg.teams = c->teams;
  cfg.sag = c->sag == 0 ? spardl::SagMode::none
                        : (c->sag == 1 ? spardl::SagMode::rsag : spardl::SagMode::bsag);
  cfg.residual = c->residual == 0 ? spardl::ResidualMode::gres
                                  : (c->residual == 1 ? spardl::ResidualMode::pres
                                                      : spardl::ResidualMode::lres);
  cfg.timing = c->timing == 0 ? spardl::SrsTiming::optimized : spardl::SrsTiming::naive;
  cfg.seed = c->seed;
  return cfg;
}

struct orc_ctx {
  spardl::ClusterConfig cfg;
  std::unique_ptr<spardl::Fabric> fabric;
  std::vector<spardl::WorkerState> states;
  spardl::RunResult last;
  double last_seconds = 0.0;
};

EXPORT const char* orc_last_error() { return g_msg.c_str(); }

EXPORT int orc_validate(const orc_config* c) {
  return guarded([&] { spardl::validate(to_cluster(c)); });
}

EXPORT int orc_ctx_create(const orc_config* c, orc_ctx** out) {
  *out = nullptr;
  return guarded([&] {
    auto x = std::make_unique<orc_ctx>();
    x->cfg = to_cluster(c);
    x->states = spardl::make_worker_states(x->cfg);
    x->fabric = std::make_unique<spardl::Fabric>(static_cast<int>(x->cfg.workers));
    *out = x.release();
  });
}

EXPORT void orc_ctx_destroy(orc_ctx* x) { delete x; }

// grads[w] -> N doubles.  Converting to GradientVector is outside the timed
// region reported by orc_last_seconds().
EXPORT int orc_allreduce(orc_ctx* x, const double* const* grads) {
  return guarded([&] {
    std::vector<spardl::GradientVector> g;
    g.reserve(static_cast<size_t>(x->cfg.workers));
    for (int64_t w = 0; w < x->cfg.workers; ++w) {
      g.emplace_back(std::vector<double>(grads[w], grads[w] + x->cfg.dimension));
    }
    auto t0 = std::chrono::steady_clock::now();
    x->last = spardl::spardl_all_reduce(*x->fabric, x->cfg, g, x->states);
    auto t1 = std::chrono::steady_clock::now();
    x->last_seconds = std::chrono::duration<double>(t1 - t0).count();
  });
}

// float inputs widened to double (the bench path: identical arrays to the GPU run)
EXPORT int orc_allreduce_f32(orc_ctx* x, const float* const* grads) {
  return guarded([&] {
    std::vector<spardl::GradientVector> g;
    g.reserve(static_cast<size_t>(x->cfg.workers));
    for (int64_t w = 0; w < x->cfg.workers; ++w) {
      std::vector<double> v(static_cast<size_t>(x->cfg.dimension));
      for (int64_t i = 0; i < x->cfg.dimension; ++i) v[static_cast<size_t>(i)] = grads[w][i];
      g.emplace_back(std::move(v));
    }
    auto t0 = std::chrono::steady_clock::now();
    x->last = spardl::spardl_all_reduce(*x->fabric, x->cfg, g, x->states);
    auto t1 = std::chrono::steady_clock::now();
    x->last_seconds = std::chrono::duration<double>(t1 - t0).count();
  });
}

EXPORT double orc_last_seconds(const orc_ctx* x) { return x->last_seconds; }

EXPORT void orc_get_carry(const orc_ctx* x, int w, double* out) {
  const auto& c = x->states[static_cast<size_t>(w)].residual.carry();
  std::memcpy(out, c.values.data(), sizeof(double) * c.values.size());
}

EXPORT void orc_get_ledger(const orc_ctx* x, int64_t* rounds, int64_t* scalars) {
  const auto& l = x->fabric->ledger();
  for (size_t w = 0; w < l.size(); ++w) {
    rounds[w] = l[w].rounds;
    scalars[w] = l[w].scalars_received;
  }
}

EXPORT void orc_get_run_info(const orc_ctx* x, orc_run_info* o) {
  std::memset(o, 0, sizeof *o);
  const auto& r = x->last;
  o->consistent = r.consistent ? 1 : 0;
  o->conservation_applicable = r.conservation_applicable ? 1 : 0;
  o->conservation_error = r.conservation_error;
  o->max_rounds = r.ledger.max_rounds;
  o->max_scalars = r.ledger.max_scalars_received;
  o->srs_rounds = r.srs_phase.rounds;
  o->srs_scalars = r.srs_phase.scalars;
  o->sag_rounds = r.sag_phase.rounds;
  o->sag_scalars = r.sag_phase.scalars;
  o->gather_rounds = r.gather_phase.rounds;
  o->gather_scalars = r.gather_phase.scalars;
  o->pred_rounds = r.predicted.rounds;
  o->pred_low = r.predicted.scalars_low;
  o->pred_high = r.predicted.scalars_high;
  o->n_union = static_cast<int64_t>(r.union_sizes.size());
  o->global_nnz = r.global.nnz();
}

EXPORT void orc_get_global(const orc_ctx* x, int64_t* idx, double* val) {
  const auto& e = x->last.global.entries;
  for (size_t i = 0; i < e.size(); ++i) {
    idx[i] = e[i].index;
    val[i] = e[i].value;
  }
}

EXPORT void orc_get_union_sizes(const orc_ctx* x, int64_t* out) {
  for (size_t i = 0; i < x->last.union_sizes.size(); ++i) out[i] = x->last.union_sizes[i];
}

EXPORT int orc_get_controller(const orc_ctx* x, int w, orc_hctrl* out) {
  const auto& c = x->states[static_cast<size_t>(w)].controller;
  if (!c.has_value()) return 7;
  out->h = c->h();
  out->step = c->step();
  out->flag = c->flag() ? 1 : 0;
  out->target = c->target();
  out->lower = static_cast<double>(x->cfg.k) / static_cast<double>(x->cfg.workers);
  out->upper = static_cast<double>(x->cfg.teams * x->cfg.k) / static_cast<double>(x->cfg.workers);
  out->pad_ = 0;
  return 0;
}

static spardl::SparseBlock make_block(int id, int64_t lo, int64_t hi, const int64_t* idx,
                                      const double* val, int64_t n) {
  spardl::SparseBlock b;
  b.block_id = id;
  b.range = {lo, hi};
  b.entries.resize(static_cast<size_t>(n));
  for (int64_t i = 0; i < n; ++i) b.entries[static_cast<size_t>(i)] = {idx[i], val[i]};
  return b;
}

static void unpack(const spardl::SparseBlock& b, int64_t* idx, double* val, int64_t* n) {
  for (size_t i = 0; i < b.entries.size(); ++i) {
    idx[i] = b.entries[i].index;
    val[i] = b.entries[i].value;
  }
  *n = b.nnz();
}

EXPORT int orc_top_k_select(int block_id, int64_t lo, int64_t hi, const int64_t* idx,
                            const double* val, int64_t n, int64_t budget, int64_t* sel_idx,
                            double* sel_val, int64_t* n_sel, int64_t* disc_idx, double* disc_val,
                            int64_t* n_disc) {
  return guarded([&] {
    auto r = spardl::top_k_select(make_block(block_id, lo, hi, idx, val, n), budget);
    unpack(r.selected, sel_idx, sel_val, n_sel);
    unpack(r.discarded, disc_idx, disc_val, n_disc);
  });
}

EXPORT int orc_top_k_select_slice(const double* g, int64_t lo, int64_t hi, int64_t budget,
                                  int64_t* sel_idx, double* sel_val, int64_t* n_sel,
                                  int64_t* disc_idx, double* disc_val, int64_t* n_disc) {
  return guarded([&] {
    spardl::GradientVector gv(std::vector<double>(g, g + hi));
    auto r = spardl::top_k_select_slice(gv, 0, {lo, hi}, budget);
    unpack(r.selected, sel_idx, sel_val, n_sel);
    unpack(r.discarded, disc_idx, disc_val, n_disc);
  });
}

// inc/collectives.hpp:185-216, unmodified, on a fresh Fabric
EXPORT int orc_topka(int p, int64_t n, int64_t k, const double* const* grads, int64_t* out_idx,
                     double* out_val, int64_t* n_out, int64_t* rounds, int64_t* scalars) {
  return guarded([&] {
    std::vector<spardl::GradientVector> g;
    for (int w = 0; w < p; ++w) g.emplace_back(std::vector<double>(grads[w], grads[w] + n));
    spardl::Fabric fabric(p);
    auto res = spardl::topka_baseline(fabric, g, k);
    const auto& e = res[0].entries;
    for (size_t i = 0; i < e.size(); ++i) {
      out_idx[i] = e[i].index;
      out_val[i] = e[i].value;
    }
    *n_out = static_cast<int64_t>(e.size());
    for (int w = 1; w < p; ++w)
      if (!(res[static_cast<size_t>(w)] == res[0]))
        throw spardl::consistency_error("topka: workers disagree");
    const auto& l = fabric.ledger();
    for (size_t w = 0; w < l.size(); ++w) {
      rounds[w] = l[w].rounds;
      scalars[w] = l[w].scalars_received;
    }
  });
}

EXPORT int orc_merge_add(int a_id, const int64_t* a_idx, const double* a_val, int64_t na,
                         int b_id, const int64_t* b_idx, const double* b_val, int64_t nb,
                         int64_t* out_idx, double* out_val, int64_t* n_out) {
  return guarded([&] {
    auto r = spardl::merge_add(make_block(a_id, 0, 0, a_idx, a_val, na),
                               make_block(b_id, 0, 0, b_idx, b_val, nb));
    unpack(r, out_idx, out_val, n_out);
  });
}

EXPORT int orc_partition(int64_t n, int count, int64_t* lo, int64_t* hi) {
  return guarded([&] {
    auto p = spardl::partition(n, count);
    for (int b = 0; b < count; ++b) {
      lo[b] = p.ranges[static_cast<size_t>(b)].lo;
      hi[b] = p.ranges[static_cast<size_t>(b)].hi;
    }
  });
}

EXPORT int orc_build_bags(int m, int rank, int32_t* l, int32_t* remainder, int32_t* bag_size,
                          int32_t* positions) {
  return guarded([&] {
    auto s = spardl::build_bags(m, rank);
    *l = s.l;
    *remainder = s.remainder;
    int o = 0;
    for (size_t j = 0; j < s.sending_bags.size(); ++j) {
      bag_size[j] = static_cast<int32_t>(s.sending_bags[j].size());
      for (int p : s.sending_bags[j]) positions[o++] = p;
    }
  });
}

EXPORT int orc_expected_cost_srs(int64_t m, int64_t k, int64_t* rounds, int64_t* scalars) {
  return guarded([&] {
    auto c = spardl::expected_cost_srs(m, k);
    *rounds = c.rounds;
    *scalars = c.scalars;
  });
}

EXPORT int orc_expected_cost_sag(int64_t P, int64_t k, int64_t d, int mode, int64_t* rounds,
                                 int64_t* low, int64_t* high) {
  return guarded([&] {
    auto c = spardl::expected_cost_sag(
        P, k, d,
        mode == 0 ? spardl::SagMode::none
                  : (mode == 1 ? spardl::SagMode::rsag : spardl::SagMode::bsag));
    *rounds = c.rounds;
    *low = c.scalars_low;
    *high = c.scalars_high;
  });
}

EXPORT int orc_dyadic_shares(int count, double* out) {
  return guarded([&] {
    auto s = spardl::dyadic_shares(count);
    for (size_t i = 0; i < s.size(); ++i) out[i] = s[i];
  });
}

// Throughput leg for bench.py --impl reference: runs `threads` independent
// reference all-reduces concurrently (the reference itself is single
// threaded, inc/fabric.hpp:47-53), each on its own copy of the inputs, for
// `iters` iterations; returns wall seconds for the concurrent region.
EXPORT int orc_parallel_allreduce_f32(const orc_config* c, const float* const* grads,
                                      int threads, int iters, double* seconds) {
  return guarded([&] {
    const auto cfg = to_cluster(c);
    std::vector<std::vector<spardl::GradientVector>> inputs(static_cast<size_t>(threads));
    std::vector<std::vector<spardl::WorkerState>> states(static_cast<size_t>(threads));
    std::vector<std::unique_ptr<spardl::Fabric>> fabrics(static_cast<size_t>(threads));
    for (int t = 0; t < threads; ++t) {
      for (int64_t w = 0; w < cfg.workers; ++w) {
        std::vector<double> v(static_cast<size_t>(cfg.dimension));
        for (int64_t i = 0; i < cfg.dimension; ++i) v[static_cast<size_t>(i)] = grads[w][i];
        inputs[static_cast<size_t>(t)].emplace_back(std::move(v));
      }
      states[static_cast<size_t>(t)] = spardl::make_worker_states(cfg);
      fabrics[static_cast<size_t>(t)] = std::make_unique<spardl::Fabric>(static_cast<int>(cfg.workers));
    }
    std::vector<std::thread> pool;
    std::vector<int> bad(static_cast<size_t>(threads), 0);
    auto t0 = std::chrono::steady_clock::now();
    for (int t = 0; t < threads; ++t) {
      pool.emplace_back([&, t] {
        try {
          for (int it = 0; it < iters; ++it) {
            auto r = spardl::spardl_all_reduce(*fabrics[static_cast<size_t>(t)], cfg,
                                               inputs[static_cast<size_t>(t)],
                                               states[static_cast<size_t>(t)]);
            if (!r.consistent) bad[static_cast<size_t>(t)] = 1;
          }
        } catch (...) {
          bad[static_cast<size_t>(t)] = 1;
        }
      });
    }
    for (auto& th : pool) th.join();
    auto t1 = std::chrono::steady_clock::now();
    *seconds = std::chrono::duration<double>(t1 - t0).count();
    for (int b : bad)
      if (b) throw spardl::consistency_error("reference run failed or was inconsistent");
  });
}

// The reference on all host cores: `threads` independent unmodified
// reference instances (spardl_all_reduce is single-threaded by design,
// inc/fabric.hpp:47-53), instance t on slice [t*N, (t+1)*N) of every worker's
// gradient (N = c->dimension), run in lockstep: step_seconds[it] is the wall
// time until every instance has finished iteration it.
EXPORT int orc_parallel_slices_f32(const orc_config* c, const float* const* grads, int threads,
                                   int iters, double* step_seconds) {
  return guarded([&] {
    const auto cfg = to_cluster(c);
    const size_t n = static_cast<size_t>(cfg.dimension);
    std::vector<std::vector<spardl::GradientVector>> inputs(static_cast<size_t>(threads));
    std::vector<std::vector<spardl::WorkerState>> states(static_cast<size_t>(threads));
    std::vector<std::unique_ptr<spardl::Fabric>> fabrics(static_cast<size_t>(threads));
    {
      std::vector<std::thread> prep;
      for (int t = 0; t < threads; ++t)
        prep.emplace_back([&, t] {
          for (int64_t w = 0; w < cfg.workers; ++w) {
            const float* src = grads[w] + static_cast<size_t>(t) * n;
            inputs[static_cast<size_t>(t)].emplace_back(std::vector<double>(src, src + n));
          }
          states[static_cast<size_t>(t)] = spardl::make_worker_states(cfg);
          fabrics[static_cast<size_t>(t)] =
              std::make_unique<spardl::Fabric>(static_cast<int>(cfg.workers));
        });
      for (auto& th : prep) th.join();
    }
    std::vector<int> bad(static_cast<size_t>(threads), 0);
    for (int it = 0; it < iters; ++it) {
      std::vector<std::thread> pool;
      auto t0 = std::chrono::steady_clock::now();
      for (int t = 0; t < threads; ++t)
        pool.emplace_back([&, t] {
          try {
            auto r = spardl::spardl_all_reduce(*fabrics[static_cast<size_t>(t)], cfg,
                                               inputs[static_cast<size_t>(t)],
                                               states[static_cast<size_t>(t)]);
            if (!r.consistent) bad[static_cast<size_t>(t)] = 1;
          } catch (...) {
            bad[static_cast<size_t>(t)] = 1;
          }
        });
      for (auto& th : pool) th.join();
      step_seconds[it] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    }
    for (int b : bad)
      if (b) throw spardl::consistency_error("reference run failed or was inconsistent");
  });
}

EXPORT int orc_bsag_phase_cost(int64_t P, int64_t k, int64_t d, int64_t* rounds, int64_t* low,
                               int64_t* high) {
  return guarded([&] {
    auto c = spardl::bsag_phase_cost(P, k, d);
    *rounds = c.rounds;
    *low = c.scalars_low;
    *high = c.scalars_high;
  });
}

EXPORT int orc_topka_cost(int64_t P, int64_t k, int64_t* rounds, int64_t* low, int64_t* high) {
  return guarded([&] {
    auto c = spardl::topka_cost(P, k);
    *rounds = c.rounds;
    *low = c.scalars_low;
    *high = c.scalars_high;
  });
}

// Replays Algorithm 2 (inc/sag.hpp:37-90) over a sequence of union sizes.
EXPORT int orc_hctrl_trace(int64_t P, int64_t k, int64_t d, int64_t n_obs, const int64_t* ns,
                           double* h, double* step, int32_t* flag, int64_t* budget) {
  return guarded([&] {
    spardl::HController c(P, k, d);
    for (int64_t i = 0; i <= n_obs; ++i) {
      h[i] = c.h();
      step[i] = c.step();
      flag[i] = c.flag() ? 1 : 0;
      budget[i] = c.budget();
      if (i < n_obs) c.observe(ns[i]);
    }
  });
}
