// spardl_b200.hpp -- C++ drop-in surface of the B200 SparDL path.
//
// Mirrors the public API of the reference's header-only library
// (/root/reference/proj/include/spardl, "inc/") so that reference users keep
// their code: same namespace, type and function names, argument meaning and
// exception classes.  The implementation is a thin layer over the C ABI of
// libspardl_cuda.so (include/spardl_cuda.h): the sparse arithmetic and the
// whole all-reduce run on the GPU; this header only converts containers.
//
// Numerics: the device computes values in fp32 (indices int32); doubles are
// converted on the way in.  Inputs that are fp32-representable produce the
// reference's results bit-for-bit wherever the reference's own arithmetic
// stays fp32-exact (e.g. grid-snapped gradients); otherwise values agree to
// fp32 rounding.
//
// Link with -lspardl_cuda (paper_2304_00737_b200/libspardl_cuda.so).
#pragma once

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <memory>
#include <optional>
#include <ostream>
#include <stdexcept>
#include <string>
#include <vector>

#include "spardl_cuda.h"

namespace spardl {

// ---------------------------------------------------------------- errors (inc/error.hpp)
class error : public std::runtime_error {
 public:
  explicit error(const std::string& what) : std::runtime_error(what) {}
};
#define SPARDL_B200_ERROR_CLASS(name) \
  class name : public error {         \
   public:                            \
    using error::error;               \
  };
SPARDL_B200_ERROR_CLASS(partition_error)
SPARDL_B200_ERROR_CLASS(block_mismatch_error)
SPARDL_B200_ERROR_CLASS(schedule_violation_error)
SPARDL_B200_ERROR_CLASS(theorem_violation_error)
SPARDL_B200_ERROR_CLASS(group_size_error)
SPARDL_B200_ERROR_CLASS(config_error)
SPARDL_B200_ERROR_CLASS(state_error)
SPARDL_B200_ERROR_CLASS(consistency_error)
#undef SPARDL_B200_ERROR_CLASS

namespace b200 {
// status code of the C ABI -> the reference's exception class
inline void check(int rc) {
  if (rc == SPARDL_OK) return;
  const std::string m = spardl_last_error();
  switch (rc) {
    case SPARDL_E_PARTITION: throw partition_error(m);
    case SPARDL_E_BLOCK_MISMATCH: throw block_mismatch_error(m);
    case SPARDL_E_SCHEDULE: throw schedule_violation_error(m);
    case SPARDL_E_THEOREM: throw theorem_violation_error(m);
    case SPARDL_E_GROUP_SIZE: throw group_size_error(m);
    case SPARDL_E_CONFIG: throw config_error(m);
    case SPARDL_E_STATE: throw state_error(m);
    case SPARDL_E_CONSISTENCY: throw consistency_error(m);
    default: throw error(m);
  }
}
}  // namespace b200

// ---------------------------------------------------------------- inc/mathutil.hpp
constexpr bool is_power_of_two(std::int64_t x) { return x > 0 && (x & (x - 1)) == 0; }
constexpr int ceil_log2(std::int64_t x) { return x <= 1 ? 0 : 1 + ceil_log2((x + 1) / 2); }
constexpr int exact_log2(std::int64_t x) { return x <= 1 ? 0 : 1 + exact_log2(x / 2); }

// ---------------------------------------------------------------- inc/sparse.hpp
using Index = std::int64_t;

struct GradientVector {
  std::vector<double> values;
  GradientVector() = default;
  explicit GradientVector(Index n, double fill = 0.0) : values(static_cast<size_t>(n), fill) {}
  explicit GradientVector(std::vector<double> v) : values(std::move(v)) {}
  Index size() const { return static_cast<Index>(values.size()); }
  double& operator[](Index i) { return values[static_cast<size_t>(i)]; }
  double operator[](Index i) const { return values[static_cast<size_t>(i)]; }
};

struct IndexRange {
  Index lo = 0;
  Index hi = 0;
  Index size() const { return hi - lo; }
  bool contains(Index i) const { return lo <= i && i < hi; }
  bool operator==(const IndexRange&) const = default;
};

struct Entry {
  Index index = 0;
  double value = 0.0;
  bool operator==(const Entry&) const = default;
};

struct SparseBlock {
  int block_id = 0;
  IndexRange range;
  std::vector<Entry> entries;
  Index nnz() const { return static_cast<Index>(entries.size()); }
  bool empty() const { return entries.empty(); }
  bool operator==(const SparseBlock&) const = default;
};

struct BlockPartition {
  Index n = 0;
  int block_count = 0;
  std::vector<IndexRange> ranges;
  const IndexRange& range_of(int block_id) const { return ranges[static_cast<size_t>(block_id)]; }
  int block_of(Index i) const {
    std::int32_t b = 0;
    b200::check(spardl_block_of(n, block_count, i, &b));
    return b;
  }
};

inline BlockPartition partition(Index n, int block_count) {
  BlockPartition p;
  p.n = n;
  p.block_count = block_count;
  std::vector<std::int64_t> lo(static_cast<size_t>(std::max(block_count, 1)));
  std::vector<std::int64_t> hi(lo.size());
  b200::check(spardl_partition(n, block_count, lo.data(), hi.data()));
  for (int b = 0; b < block_count; ++b) p.ranges.push_back({lo[size_t(b)], hi[size_t(b)]});
  return p;
}

// The selection order of the device select (|v| desc, index asc).
inline bool selection_before(const Entry& a, const Entry& b) {
  const double x = a.value < 0 ? -a.value : a.value;
  const double y = b.value < 0 ? -b.value : b.value;
  return x != y ? x > y : a.index < b.index;
}

struct TopKResult {
  SparseBlock selected;
  SparseBlock discarded;
};

namespace b200 {
inline std::int32_t idx32(Index i) {
  if (i < 0 || i >= (Index(1) << 31)) throw error("index outside the device's int32 range");
  return static_cast<std::int32_t>(i);
}
}  // namespace b200

// Device selection; the entries returned carry the caller's own values.
// top_k_select / merge_add run on the GPU in double (the reference's
// semantics, spardl_topk_select_f64 / spardl_merge_add_f64); the values of
// the outputs are the inputs' values (selection) or their a + b sums.
inline TopKResult top_k_select(const SparseBlock& block, Index budget) {
  if (budget < 0) throw error("top_k_select: negative budget");
  TopKResult out;
  out.selected.block_id = out.discarded.block_id = block.block_id;
  out.selected.range = out.discarded.range = block.range;
  const size_t n = block.entries.size();
  std::vector<std::int64_t> idx(n);
  std::vector<double> val(n);
  for (size_t e = 0; e < n; ++e) {
    idx[e] = block.entries[e].index;
    val[e] = block.entries[e].value;
  }
  std::vector<std::uint8_t> flag(n + 1, 0);
  if (n > 0)
    b200::check(spardl_topk_select_f64_hostbuf(idx.data(), val.data(),
                                               static_cast<std::int64_t>(n), budget,
                                               flag.data()));
  for (size_t e = 0; e < n; ++e)
    (flag[e] ? out.selected : out.discarded).entries.push_back(block.entries[e]);
  return out;
}

// The dense slice [lo, hi) as a block (every index an entry, zeros
// included, inc/sparse.hpp:167-177), selected on the GPU.
inline TopKResult top_k_select_slice(const GradientVector& g, int block_id,
                                     const IndexRange& range, Index budget) {
  SparseBlock block;
  block.block_id = block_id;
  block.range = range;
  block.entries.reserve(static_cast<size_t>(range.size()));
  for (Index i = range.lo; i < range.hi; ++i) block.entries.push_back({i, g[i]});
  return top_k_select(block, budget);
}

inline SparseBlock merge_add(const SparseBlock& a, const SparseBlock& b) {
  if (a.block_id != b.block_id)
    throw block_mismatch_error("merge_add: block ids differ (" + std::to_string(a.block_id) +
                               " vs " + std::to_string(b.block_id) + ")");
  std::vector<std::int64_t> ai, bi;
  std::vector<double> av, bv;
  for (const Entry& e : a.entries) ai.push_back(e.index), av.push_back(e.value);
  for (const Entry& e : b.entries) bi.push_back(e.index), bv.push_back(e.value);
  std::vector<std::int64_t> oi(ai.size() + bi.size() + 1);
  std::vector<double> ov(oi.size());
  std::int64_t no = 0;
  b200::check(spardl_merge_add_f64_hostbuf(ai.data(), av.data(), std::int64_t(ai.size()),
                                           bi.data(), bv.data(), std::int64_t(bi.size()),
                                           oi.data(), ov.data(), &no));
  SparseBlock out;
  out.block_id = a.block_id;
  out.range = a.range;
  out.entries.reserve(static_cast<size_t>(no));
  for (std::int64_t e = 0; e < no; ++e) out.entries.push_back({oi[size_t(e)], ov[size_t(e)]});
  return out;
}

inline SparseBlock scale(const SparseBlock& block, double factor) {
  SparseBlock out = block;
  for (Entry& e : out.entries) e.value *= factor;
  return out;
}

struct GlobalSparseGradient {
  Index n = 0;
  std::vector<Entry> entries;
  Index nnz() const { return static_cast<Index>(entries.size()); }
  bool operator==(const GlobalSparseGradient&) const = default;
};

inline bool well_formed(const SparseBlock& block) {
  for (size_t e = 0; e < block.entries.size(); ++e) {
    if (!block.range.contains(block.entries[e].index)) return false;
    if (e && block.entries[e].index <= block.entries[e - 1].index) return false;
  }
  return true;
}

// ---------------------------------------------------------------- inc/fabric.hpp
using WorkerId = int;

struct WorkerCost {
  std::int64_t rounds = 0;
  std::int64_t scalars_received = 0;
  bool operator==(const WorkerCost&) const = default;
};

struct LedgerReport {
  std::vector<WorkerCost> per_worker;
  std::int64_t max_rounds = 0;
  std::int64_t max_scalars_received = 0;
};

struct ClusterConfig;
namespace b200 {
struct DeviceState;   // the GPU context a Fabric drives (created on first use)
}

// The fabric of the drop-in API.  spardl_all_reduce moves blocks GPU to GPU
// (NVLink); the ledger here is the reference's alpha-beta account of it.
class Fabric {
 public:
  struct Send {
    WorkerId target = 0;
    std::vector<SparseBlock> payload;
  };
  using RoundPlan = std::vector<std::optional<Send>>;

  explicit Fabric(int worker_count) : costs_(static_cast<size_t>(worker_count > 0 ? worker_count : 0)) {
    if (worker_count < 1) throw config_error("fabric needs >= 1 worker");
  }
  int worker_count() const { return static_cast<int>(costs_.size()); }

  // One lockstep round of host-side block delivery with the reference's
  // accounting (used by callers that drive their own schedules).
  std::vector<std::vector<SparseBlock>> exchange(RoundPlan plan) {
    const int p = worker_count();
    if (static_cast<int>(plan.size()) != p)
      throw schedule_violation_error("round plan size != worker count");
    std::vector<std::vector<SparseBlock>> inbox(plan.size());
    std::vector<char> hit(plan.size(), 0), active(plan.size(), 0);
    for (WorkerId s = 0; s < p; ++s) {
      auto& snd = plan[size_t(s)];
      if (!snd) continue;
      const WorkerId t = snd->target;
      if (t < 0 || t >= p)
        throw schedule_violation_error("message target out of range: " + std::to_string(t));
      if (hit[size_t(t)])
        throw schedule_violation_error("two messages target worker " + std::to_string(t) +
                                       " in one round");
      hit[size_t(t)] = active[size_t(s)] = active[size_t(t)] = 1;
      for (const SparseBlock& b : snd->payload) costs_[size_t(t)].scalars_received += 2 * b.nnz();
      inbox[size_t(t)] = std::move(snd->payload);
    }
    for (size_t w = 0; w < active.size(); ++w) costs_[w].rounds += active[w];
    return inbox;
  }

  const std::vector<WorkerCost>& ledger() const { return costs_; }
  LedgerReport report() const {
    LedgerReport r;
    r.per_worker = costs_;
    for (const WorkerCost& c : costs_) {
      r.max_rounds = std::max(r.max_rounds, c.rounds);
      r.max_scalars_received = std::max(r.max_scalars_received, c.scalars_received);
    }
    return r;
  }
  WorkerCost delta_since(const std::vector<WorkerCost>& snap) const {
    WorkerCost d;
    for (size_t w = 0; w < costs_.size(); ++w) {
      d.rounds = std::max(d.rounds, costs_[w].rounds - snap[w].rounds);
      d.scalars_received =
          std::max(d.scalars_received, costs_[w].scalars_received - snap[w].scalars_received);
    }
    return d;
  }

  // drop-in internals
  std::vector<WorkerCost>& mutable_ledger() { return costs_; }
  std::shared_ptr<b200::DeviceState> device;

 private:
  std::vector<WorkerCost> costs_;
};

inline void write_ledger_csv(std::ostream& os, const Fabric& fabric) {
  os << "worker_id,rounds,scalars_received\n";
  for (size_t w = 0; w < fabric.ledger().size(); ++w)
    os << w << ',' << fabric.ledger()[w].rounds << ',' << fabric.ledger()[w].scalars_received
       << '\n';
}

// ---------------------------------------------------------------- inc/collectives.hpp
// Host-side gathers over the drop-in Fabric (the reference's alpha-beta
// ledger).  The pipeline's own gathers run GPU to GPU (spardl_all_reduce);
// these are the component forms its callers and tests drive.
struct GroupGather {
  std::vector<WorkerId> workers;
  std::vector<SparseBlock> blocks;   // blocks[i] belongs to workers[i]
};
// result[i][s]: the block of group member s as held by member i
using GatherResult = std::vector<std::vector<SparseBlock>>;

namespace detail {
// inc/collectives.hpp:46-114: Bruck all-gather of several disjoint groups
// in shared rounds.  Member i keeps its blocks in rotated order (its own
// first); at distance 2^t it sends its first min(2^t, m - 2^t) blocks to
// member i - 2^t and appends what member i + 2^t sent; the final un-rotation
// is local.
inline std::vector<GatherResult> bruck_all_gather_multi(Fabric& fabric,
                                                        const std::vector<GroupGather>& groups) {
  std::vector<std::vector<std::vector<SparseBlock>>> rot(groups.size());
  int rounds = 0;
  for (size_t g = 0; g < groups.size(); ++g) {
    const size_t m = groups[g].workers.size();
    if (m == 0) throw group_size_error("all-gather on empty group");
    if (groups[g].blocks.size() != m) throw group_size_error("group has blocks != workers");
    for (size_t i = 0; i < m; ++i) rot[g].push_back({groups[g].blocks[i]});
    rounds = std::max(rounds, ceil_log2(static_cast<std::int64_t>(m)));
  }
  for (int t = 0; t < rounds; ++t) {
    const int dist = 1 << t;
    Fabric::RoundPlan plan(size_t(fabric.worker_count()));
    for (size_t g = 0; g < groups.size(); ++g) {
      const int m = static_cast<int>(groups[g].workers.size());
      if (dist >= m) continue;
      const int cnt = std::min(dist, m - dist);
      for (int i = 0; i < m; ++i) {
        Fabric::Send snd;
        snd.target = groups[g].workers[size_t((i - dist + m) % m)];
        snd.payload.assign(rot[g][size_t(i)].begin(), rot[g][size_t(i)].begin() + cnt);
        plan[size_t(groups[g].workers[size_t(i)])] = std::move(snd);
      }
    }
    auto inbox = fabric.exchange(std::move(plan));
    for (size_t g = 0; g < groups.size(); ++g) {
      const int m = static_cast<int>(groups[g].workers.size());
      if (dist >= m) continue;
      for (int i = 0; i < m; ++i)
        for (SparseBlock& b : inbox[size_t(groups[g].workers[size_t(i)])])
          rot[g][size_t(i)].push_back(std::move(b));
    }
  }
  std::vector<GatherResult> out(groups.size());
  for (size_t g = 0; g < groups.size(); ++g) {
    const int m = static_cast<int>(groups[g].workers.size());
    out[g].assign(size_t(m), std::vector<SparseBlock>(size_t(m)));
    for (int i = 0; i < m; ++i)
      for (int q = 0; q < m; ++q)   // rotated slot q holds source (i + q) mod m
        out[g][size_t(i)][size_t((i + q) % m)] = std::move(rot[g][size_t(i)][size_t(q)]);
  }
  return out;
}
}  // namespace detail

inline GatherResult bruck_all_gather(Fabric& fabric, const std::vector<WorkerId>& workers,
                                     const std::vector<SparseBlock>& blocks) {
  return detail::bruck_all_gather_multi(fabric, {GroupGather{workers, blocks}})[0];
}

// inc/collectives.hpp:130-178: pairwise XOR exchange of everything held,
// power-of-two groups only; same result as bruck_all_gather.
inline GatherResult recursive_doubling_all_gather(Fabric& fabric,
                                                  const std::vector<WorkerId>& workers,
                                                  const std::vector<SparseBlock>& blocks) {
  const int m = static_cast<int>(workers.size());
  if (m == 0) throw group_size_error("all-gather on empty group");
  if (!is_power_of_two(m))
    throw group_size_error("recursive doubling requires a power-of-two group, got m=" +
                           std::to_string(m));
  if (blocks.size() != workers.size()) throw group_size_error("group has blocks != workers");
  GatherResult have(static_cast<size_t>(m), std::vector<SparseBlock>(static_cast<size_t>(m)));
  for (int i = 0; i < m; ++i) have[size_t(i)][size_t(i)] = blocks[size_t(i)];
  for (int dist = 1; dist < m; dist <<= 1) {
    Fabric::RoundPlan plan(size_t(fabric.worker_count()));
    for (int i = 0; i < m; ++i) {   // i holds the aligned run of `dist` slots around i
      Fabric::Send snd;
      snd.target = workers[size_t(i ^ dist)];
      const int base = i & ~(dist - 1);
      snd.payload.assign(have[size_t(i)].begin() + base, have[size_t(i)].begin() + base + dist);
      plan[size_t(workers[size_t(i)])] = std::move(snd);
    }
    auto inbox = fabric.exchange(std::move(plan));
    for (int i = 0; i < m; ++i) {
      const int base = (i ^ dist) & ~(dist - 1);
      auto& got = inbox[size_t(workers[size_t(i)])];
      for (int q = 0; q < dist; ++q) have[size_t(i)][size_t(base + q)] = std::move(got[size_t(q)]);
    }
  }
  return have;
}

// ---------------------------------------------------------------- inc/reduce_scatter.hpp
enum class SrsTiming { optimized, naive };

struct BagSchedule {
  int team_size = 1;
  int worker_rank = 0;
  int l = 0;
  int preservation = 0;
  std::vector<std::vector<int>> sending_bags;
  int remainder = 0;
  bool operator==(const BagSchedule&) const = default;
};

inline BagSchedule build_bags(int team_size, int worker_rank) {
  std::int32_t l = 0, rem = 0;
  std::vector<std::int32_t> sizes(64), pos(static_cast<size_t>(std::max(team_size, 1)));
  b200::check(spardl_build_bags(team_size, worker_rank, &l, &rem, sizes.data(), pos.data()));
  BagSchedule s;
  s.team_size = team_size;
  s.worker_rank = worker_rank;
  s.preservation = worker_rank;
  s.l = l;
  s.remainder = rem;
  size_t o = 0;
  for (int j = 0; j < l; ++j) {
    s.sending_bags.emplace_back(pos.begin() + std::ptrdiff_t(o),
                                pos.begin() + std::ptrdiff_t(o + size_t(sizes[size_t(j)])));
    o += size_t(sizes[size_t(j)]);
  }
  return s;
}

struct SrsCost {
  std::int64_t rounds = 0;
  std::int64_t scalars = 0;
};
inline SrsCost expected_cost_srs(std::int64_t m, std::int64_t k) {
  SrsCost c;
  b200::check(spardl_expected_cost_srs(m, k, &c.rounds, &c.scalars));
  return c;
}

// The reduce-scatter schedule as a component (the tests and callers that
// drive their own phases): blocks move through the host Fabric (its ledger
// is the reference's), every merge and selection runs on the GPU (fp64
// components).  The pipeline's own reduce-scatter is planned once and runs
// on the device (spardl_all_reduce).
using DiscardSink = std::function<void(WorkerId, int, const SparseBlock&, double)>;
inline DiscardSink null_discard_sink() {
  return [](WorkerId, int, const SparseBlock&, double) {};
}

struct SrsTeam {
  std::vector<WorkerId> workers;                  // team rank = position here
  std::vector<std::vector<SparseBlock>> blocks;   // blocks[i][b]: member i, position b
};

namespace b200 {
// a held block back within the budget; the cut goes to the discard sink
inline void srs_sparsify(std::optional<SparseBlock>& slot, Index budget, WorkerId w,
                         const DiscardSink& sink) {
  if (!slot || slot->nnz() <= budget) return;
  TopKResult r = top_k_select(*slot, budget);
  if (!r.discarded.empty()) sink(w, r.discarded.block_id, r.discarded, 1.0);
  *slot = std::move(r.selected);
}
}  // namespace b200

// inc/reduce_scatter.hpp:120-236 (Spar-Reduce-Scatter of every team in
// lockstep); returns each team's preservation blocks, team-rank order.
inline std::vector<std::vector<SparseBlock>> run_srs_teams(
    Fabric& fabric, std::vector<SrsTeam> teams, Index budget,
    SrsTiming timing = SrsTiming::optimized, const DiscardSink& on_discard = null_discard_sink()) {
  if (teams.empty()) throw group_size_error("reduce-scatter with no teams");
  const int m = static_cast<int>(teams[0].workers.size());
  for (const SrsTeam& t : teams)
    if (static_cast<int>(t.workers.size()) != m)
      throw group_size_error("reduce-scatter teams must share one size");
  const int l = ceil_log2(m);
  // held[t][i][b]: what member i of team t holds of position b
  std::vector<std::vector<std::vector<std::optional<SparseBlock>>>> held(teams.size());
  std::vector<BagSchedule> bags;
  for (int i = 0; i < m; ++i) bags.push_back(build_bags(m, i));
  for (size_t t = 0; t < teams.size(); ++t) {
    held[t].resize(size_t(m));
    for (int i = 0; i < m; ++i) {
      auto& mine = teams[t].blocks[size_t(i)];
      if (static_cast<int>(mine.size()) != m)
        throw config_error("reduce-scatter: member needs one block per position");
      held[t][size_t(i)].resize(size_t(m));
      for (int b = 0; b < m; ++b) {
        if (mine[size_t(b)].nnz() > budget)
          throw config_error(
              "reduce-scatter: initial block exceeds budget; sparsify during dividing first");
        held[t][size_t(i)][size_t(b)] = std::move(mine[size_t(b)]);
      }
    }
  }
  for (int s = 1; s <= l; ++s) {
    const int dist = 1 << (l - s);
    const int bag = l - s;   // index of B_{l-s+1}
    Fabric::RoundPlan plan(size_t(fabric.worker_count()));
    for (size_t t = 0; t < teams.size(); ++t)
      for (int i = 0; i < m; ++i) {
        Fabric::Send snd;
        snd.target = teams[t].workers[size_t((i + dist) % m)];
        for (int pos : bags[size_t(i)].sending_bags[size_t(bag)]) {
          auto& slot = held[t][size_t(i)][size_t(pos)];
          if (!slot) throw theorem_violation_error("sending a block already given up");
          if (slot->nnz() > budget) throw error("budget discipline violated before send");
          snd.payload.push_back(std::move(*slot));
          slot.reset();
        }
        plan[size_t(teams[t].workers[size_t(i)])] = std::move(snd);
      }
    auto inbox = fabric.exchange(std::move(plan));
    for (size_t t = 0; t < teams.size(); ++t)
      for (int i = 0; i < m; ++i) {
        const WorkerId self = teams[t].workers[size_t(i)];
        auto& row = held[t][size_t(i)];
        for (SparseBlock& got : inbox[size_t(self)]) {
          if (got.block_id < 0 || got.block_id >= m)
            throw theorem_violation_error("received block id out of range");
          auto& slot = row[size_t(got.block_id)];
          if (!slot)
            throw theorem_violation_error("received block " + std::to_string(got.block_id) +
                                          " not held by worker " + std::to_string(self));
          *slot = merge_add(*slot, got);
        }
        if (timing == SrsTiming::naive) {
          for (auto& slot : row) b200::srs_sparsify(slot, budget, self, on_discard);
        } else if (s < l) {   // only the next bag must be back in budget
          for (int pos : bags[size_t(i)].sending_bags[size_t(bag - 1)])
            b200::srs_sparsify(row[size_t(pos)], budget, self, on_discard);
        }
      }
  }
  std::vector<std::vector<SparseBlock>> out(teams.size());
  for (size_t t = 0; t < teams.size(); ++t)
    for (int i = 0; i < m; ++i) {
      auto& kept = held[t][size_t(i)][size_t(bags[size_t(i)].preservation)];
      if (!kept) throw error("preservation block missing after reduce-scatter");
      b200::srs_sparsify(kept, budget, teams[t].workers[size_t(i)], on_discard);
      out[t].push_back(std::move(*kept));
    }
  return out;
}

inline std::vector<SparseBlock> run_srs(Fabric& fabric, std::vector<WorkerId> workers,
                                        std::vector<std::vector<SparseBlock>> blocks,
                                        Index budget, SrsTiming timing = SrsTiming::optimized,
                                        const DiscardSink& on_discard = null_discard_sink()) {
  std::vector<SrsTeam> teams{{std::move(workers), std::move(blocks)}};
  return run_srs_teams(fabric, std::move(teams), budget, timing, on_discard)[0];
}

// ---------------------------------------------------------------- inc/sag.hpp
class HController {
 public:
  HController(std::int64_t workers, std::int64_t k, std::int64_t teams) {
    b200::check(spardl_hctrl_init(&s_, workers, k, teams));
  }
  double h() const { return s_.h; }
  double step() const { return s_.step; }
  bool flag() const { return s_.flag != 0; }
  std::int64_t target() const { return s_.target; }
  Index budget() const {
    std::int64_t b = 0;
    b200::check(spardl_hctrl_budget(&s_, &b));
    return b;
  }
  void observe(std::int64_t n_t) { b200::check(spardl_hctrl_observe(&s_, n_t)); }
  const spardl_hctrl& raw() const { return s_; }
  spardl_hctrl& raw() { return s_; }

 private:
  spardl_hctrl s_{};
};

inline void controller_update(HController& c, std::int64_t n_t) { c.observe(n_t); }

inline std::vector<double> dyadic_shares(int count) {
  std::vector<double> s(static_cast<size_t>(std::max(count, 1)));
  b200::check(spardl_dyadic_shares(count, s.data()));
  s.resize(static_cast<size_t>(std::max(count, 0)));
  return s;
}

enum class SagMode { none, rsag, bsag };

struct CostRange {
  std::int64_t rounds = 0;
  std::int64_t scalars_low = 0;
  std::int64_t scalars_high = 0;
  bool exact() const { return scalars_low == scalars_high; }
};

inline CostRange expected_cost_sag(std::int64_t workers, std::int64_t k, std::int64_t teams,
                                   SagMode mode) {
  CostRange c;
  b200::check(spardl_expected_cost_sag(workers, k, teams, static_cast<std::int32_t>(mode),
                                       &c.rounds, &c.scalars_low, &c.scalars_high));
  return c;
}
inline CostRange bsag_phase_cost(std::int64_t workers, std::int64_t k, std::int64_t teams) {
  CostRange c;
  b200::check(spardl_bsag_phase_cost(workers, k, teams, &c.rounds, &c.scalars_low,
                                     &c.scalars_high));
  return c;
}
inline CostRange topka_cost(std::int64_t workers, std::int64_t k) {
  CostRange c;
  b200::check(spardl_topka_cost(workers, k, &c.rounds, &c.scalars_low, &c.scalars_high));
  return c;
}

// inc/sag.hpp:98-270: the team synchronisations as components (host
// Fabric, GPU merges and selections; see run_srs_teams).
struct PositionGroup {
  std::vector<WorkerId> workers;
  std::vector<SparseBlock> blocks;   // blocks[i] belongs to workers[i]
};

// R-SAG: log2 d rounds of XOR-partner swaps; each side merges the partner's
// block into its own and selects back to the budget, the discard shared
// 1/(2 dist) ways (inc/sag.hpp:125-173).
inline std::vector<std::vector<SparseBlock>> rsag_groups(
    Fabric& fabric, std::vector<PositionGroup> groups, Index budget,
    const DiscardSink& on_discard = null_discard_sink()) {
  if (groups.empty()) throw group_size_error("rsag with no groups");
  const int d = static_cast<int>(groups[0].workers.size());
  if (d < 2 || !is_power_of_two(d))
    throw group_size_error("rsag requires a power-of-two team count >= 2");
  for (const PositionGroup& g : groups)
    if (static_cast<int>(g.workers.size()) != d || g.blocks.size() != g.workers.size())
      throw group_size_error("rsag groups must share one size");
  for (int dist = 1; dist < d; dist <<= 1) {
    Fabric::RoundPlan plan(size_t(fabric.worker_count()));
    for (const PositionGroup& g : groups)
      for (int i = 0; i < d; ++i) {
        Fabric::Send snd;
        snd.target = g.workers[size_t(i ^ dist)];
        snd.payload = {g.blocks[size_t(i)]};
        plan[size_t(g.workers[size_t(i)])] = std::move(snd);
      }
    auto inbox = fabric.exchange(std::move(plan));
    const double share = 1.0 / static_cast<double>(2 * dist);
    for (PositionGroup& g : groups)
      for (int i = 0; i < d; ++i) {
        const WorkerId self = g.workers[size_t(i)];
        SparseBlock merged = merge_add(g.blocks[size_t(i)], inbox[size_t(self)].at(0));
        if (merged.nnz() > budget) {
          TopKResult r = top_k_select(merged, budget);
          on_discard(self, r.discarded.block_id, r.discarded, share);
          merged = std::move(r.selected);
        }
        g.blocks[size_t(i)] = std::move(merged);
      }
  }
  std::vector<std::vector<SparseBlock>> out;
  for (PositionGroup& g : groups) out.push_back(std::move(g.blocks));
  return out;
}

struct BsagGroupResult {
  std::vector<SparseBlock> blocks;   // identical on every member
  std::int64_t union_size = 0;       // N_t before the final selection
};

// B-SAG: every member pre-selects its block to h (the rest its own
// discard), the h-blocks are Bruck-gathered unmerged, every member folds
// them in source order and selects the identical union to the budget with
// its dyadic share of the discard (inc/sag.hpp:189-249).
inline std::vector<BsagGroupResult> bsag_groups(
    Fabric& fabric, std::vector<PositionGroup> groups, const std::vector<Index>& pre_budgets,
    Index budget, const DiscardSink& on_discard = null_discard_sink()) {
  if (groups.empty()) throw group_size_error("bsag with no groups");
  if (pre_budgets.size() != groups.size())
    throw config_error("bsag: one pre-selection budget per group");
  const int d = static_cast<int>(groups[0].workers.size());
  if (d < 2) throw group_size_error("bsag requires >= 2 teams");
  for (const PositionGroup& g : groups)
    if (static_cast<int>(g.workers.size()) != d || g.blocks.size() != g.workers.size())
      throw group_size_error("bsag groups must share one size");
  std::vector<GroupGather> gathers;
  for (size_t q = 0; q < groups.size(); ++q) {
    GroupGather gg;
    gg.workers = groups[q].workers;
    for (int i = 0; i < d; ++i) {
      SparseBlock& blk = groups[q].blocks[size_t(i)];
      if (blk.nnz() > pre_budgets[q]) {
        TopKResult r = top_k_select(blk, pre_budgets[q]);
        on_discard(groups[q].workers[size_t(i)], r.discarded.block_id, r.discarded, 1.0);
        blk = std::move(r.selected);
      }
      gg.blocks.push_back(std::move(blk));
    }
    gathers.push_back(std::move(gg));
  }
  auto got = detail::bruck_all_gather_multi(fabric, gathers);
  const std::vector<double> shares = dyadic_shares(d);
  std::vector<BsagGroupResult> out(groups.size());
  for (size_t q = 0; q < groups.size(); ++q)
    for (int i = 0; i < d; ++i) {
      SparseBlock acc = got[q][size_t(i)][0];
      for (int src = 1; src < d; ++src) acc = merge_add(acc, got[q][size_t(i)][size_t(src)]);
      out[q].union_size = acc.nnz();
      if (acc.nnz() > budget) {
        TopKResult r = top_k_select(acc, budget);
        on_discard(groups[q].workers[size_t(i)], r.discarded.block_id, r.discarded,
                   shares[size_t(i)]);
        acc = std::move(r.selected);
      }
      out[q].blocks.push_back(std::move(acc));
    }
  return out;
}

inline std::vector<SparseBlock> rsag(Fabric& fabric, std::vector<WorkerId> workers,
                                     std::vector<SparseBlock> blocks, Index budget,
                                     const DiscardSink& on_discard = null_discard_sink()) {
  std::vector<PositionGroup> groups{{std::move(workers), std::move(blocks)}};
  return rsag_groups(fabric, std::move(groups), budget, on_discard)[0];
}

inline BsagGroupResult bsag(Fabric& fabric, std::vector<WorkerId> workers,
                            std::vector<SparseBlock> blocks, Index pre_budget, Index budget,
                            const DiscardSink& on_discard = null_discard_sink()) {
  std::vector<PositionGroup> groups{{std::move(workers), std::move(blocks)}};
  return bsag_groups(fabric, std::move(groups), {pre_budget}, budget, on_discard)[0];
}

// ---------------------------------------------------------------- inc/residual.hpp
enum class ResidualMode { gres, pres, lres };

// inc/residual.hpp:52-177: a worker's residual state.  The pipeline keeps
// the authoritative carry on the GPU (in place: the carry buffer is G_copy)
// and mirrors it here after every spardl_all_reduce; the member functions
// are the reference's per-iteration protocol for callers that run the
// phases themselves (merges on the GPU in double, spardl_merge_add_f64).
class ResidualStore {
 public:
  ResidualStore(ResidualMode mode, Index n) : mode_(mode), n_(n), carry_(n) {}
  ResidualMode mode() const { return mode_; }
  Index dimension() const { return n_; }
  const GradientVector& carry() const { return carry_; }
  GradientVector& mutable_carry() { return carry_; }

  // combined = g + carry; the carry is consumed (inc/residual.hpp:63-71)
  GradientVector apply(const GradientVector& gradients) {
    if (gradients.size() != n_) throw config_error("apply_residual: dimension mismatch");
    GradientVector combined = gradients;
    for (Index i = 0; i < n_; ++i) combined[i] += carry_[i];
    carry_ = GradientVector(n_);
    return combined;
  }

  // G_copy := combined, per-block discard accumulators reset (:75-92)
  void begin_iteration(const GradientVector& combined, const BlockPartition& part) {
    if (in_iteration_) throw state_error("begin_iteration called twice without finalize");
    if (combined.size() != n_ || part.n != n_)
      throw config_error("begin_iteration: dimension mismatch");
    g_copy_ = combined;
    part_ = part;
    xi_.assign(size_t(part.block_count), SparseBlock{});
    for (int b = 0; b < part.block_count; ++b) {
      xi_[size_t(b)].block_id = b;
      xi_[size_t(b)].range = part.range_of(b);
    }
    remainder_ = GradientVector(n_);
    in_iteration_ = true;
  }

  // the dividing selection's leftovers, the lres carry (:96-99)
  void record_dividing_remainder(const SparseBlock& remainder) {
    require("record_dividing_remainder");
    for (const Entry& e : remainder.entries) remainder_[e.index] = e.value;
  }

  // xi[b] += weight * discarded (:104-124)
  void record_inproc(int block_id, const SparseBlock& discarded, double weight) {
    require("record_inproc");
    if (block_id < 0 || block_id >= part_.block_count)
      throw config_error("record_inproc: unknown block id");
    if (weight <= 0.0 || weight > 1.0)
      throw config_error("record_inproc: weight must be in (0, 1]");
    SparseBlock& acc = xi_[size_t(block_id)];
    for (const Entry& e : discarded.entries)
      if (!acc.range.contains(e.index))
        throw config_error("record_inproc: index " + std::to_string(e.index) +
                           " outside block range");
    SparseBlock w = scale(discarded, weight);
    w.block_id = block_id;
    w.range = acc.range;
    acc = merge_add(acc, w);
  }

  // the carry of the next iteration (:128-150)
  const GradientVector& finalize(const GlobalSparseGradient& final_global) {
    require("finalize");
    if (mode_ == ResidualMode::lres) {
      carry_ = remainder_;
    } else {
      carry_ = g_copy_;
      for (const Entry& e : final_global.entries)
        carry_[e.index] = mode_ == ResidualMode::gres ? xi_value(e.index) : 0.0;
    }
    in_iteration_ = false;
    return carry_;
  }

  // the in-procedure accumulator at one index, 0 when absent (:153-160)
  double xi_value(Index index) const {
    const SparseBlock& acc = xi_[size_t(part_.block_of(index))];
    auto it = std::lower_bound(acc.entries.begin(), acc.entries.end(), index,
                               [](const Entry& e, Index i) { return e.index < i; });
    return it != acc.entries.end() && it->index == index ? it->value : 0.0;
  }

 private:
  void require(const char* op) const {
    if (!in_iteration_) throw state_error(std::string(op) + " outside an iteration");
  }
  ResidualMode mode_;
  Index n_;
  GradientVector carry_;
  GradientVector g_copy_;
  GradientVector remainder_;
  std::vector<SparseBlock> xi_;
  BlockPartition part_;
  bool in_iteration_ = false;
};

inline GradientVector apply_residual(const GradientVector& gradients, ResidualStore& store) {
  return store.apply(gradients);
}
inline void record_inproc(ResidualStore& store, int block_id, const SparseBlock& discarded,
                          double weight) {
  store.record_inproc(block_id, discarded, weight);
}
inline const GradientVector& finalize(ResidualStore& store,
                                      const GlobalSparseGradient& final_global) {
  return store.finalize(final_global);
}

// ---------------------------------------------------------------- inc/pipeline.hpp
struct ClusterConfig {
  std::int64_t workers = 1;
  std::int64_t dimension = 1;
  std::int64_t k = 1;
  std::int64_t teams = 1;
  SagMode sag = SagMode::none;
  ResidualMode residual = ResidualMode::gres;
  SrsTiming timing = SrsTiming::optimized;
  std::uint64_t seed = 0;
  std::int64_t team_size() const { return workers / teams; }
  std::int64_t block_budget() const { return teams * k / workers; }
};

namespace b200 {
inline spardl_config to_c(const ClusterConfig& c) {
  spardl_config o{};
  o.workers = c.workers;
  o.dimension = c.dimension;
  o.k = c.k;
  o.teams = c.teams;
  o.sag = static_cast<std::int32_t>(c.sag);
  o.residual = static_cast<std::int32_t>(c.residual);
  o.timing = static_cast<std::int32_t>(c.timing);
  o.seed = c.seed;
  return o;
}

// The devices a drop-in spardl_all_reduce spreads its P workers over: the
// SPARDL_DEVICES list (e.g. "0,1,2,3") or every visible GPU, trimmed to the
// largest count that divides P.
inline std::vector<std::int32_t> dropin_devices(std::int64_t workers) {
  std::vector<std::int32_t> d;
  if (const char* e = std::getenv("SPARDL_DEVICES")) {
    std::string s(e);
    size_t p = 0;
    while (p < s.size()) {
      const size_t q = s.find(',', p);
      d.push_back(std::stoi(s.substr(p, q == std::string::npos ? std::string::npos : q - p)));
      if (q == std::string::npos) break;
      p = q + 1;
    }
  } else {
    std::int32_t n = 0;
    if (spardl_device_count(&n) != SPARDL_OK || n < 1) n = 1;
    for (int i = 0; i < n; ++i) d.push_back(i);
  }
  while (d.size() > 1 && workers % static_cast<std::int64_t>(d.size()) != 0) d.pop_back();
  if (d.empty()) d.push_back(0);
  return d;
}

struct DeviceState {   // one engine per device, all driven from this thread
  spardl_config cfg{};
  spardl_mctx* ctx = nullptr;
  std::vector<std::int64_t> last_scalars, last_rounds;
  ~DeviceState() {
    if (ctx) spardl_mctx_destroy(ctx);
  }
};
}  // namespace b200

inline void validate(const ClusterConfig& cfg) {
  const spardl_config c = b200::to_c(cfg);
  b200::check(spardl_validate(&c));
}

struct WorkerState {
  ResidualStore residual;
  std::optional<HController> controller;
};

inline std::vector<WorkerState> make_worker_states(const ClusterConfig& cfg) {
  validate(cfg);
  std::vector<WorkerState> s;
  for (std::int64_t w = 0; w < cfg.workers; ++w) {
    WorkerState ws{ResidualStore(cfg.residual, cfg.dimension), std::nullopt};
    if (cfg.sag == SagMode::bsag) ws.controller.emplace(cfg.workers, cfg.k, cfg.teams);
    s.push_back(std::move(ws));
  }
  return s;
}

inline bool verify_consistency(const std::vector<GlobalSparseGradient>& per_worker) {
  for (size_t w = 1; w < per_worker.size(); ++w)
    if (!(per_worker[w] == per_worker[0])) return false;
  return true;
}

struct PhaseCost {
  std::int64_t rounds = 0;
  std::int64_t scalars = 0;
};

struct RunResult {
  GlobalSparseGradient global;
  std::vector<GlobalSparseGradient> per_worker;
  bool consistent = false;
  bool conservation_applicable = false;
  double conservation_error = 0.0;
  LedgerReport ledger;
  PhaseCost srs_phase;
  PhaseCost sag_phase;
  PhaseCost gather_phase;
  CostRange predicted;
  std::vector<std::int64_t> union_sizes;
};

inline CostRange expected_cost(const ClusterConfig& cfg) {
  validate(cfg);
  return expected_cost_sag(cfg.workers, cfg.k, cfg.teams, cfg.sag);
}

// The sparse All-Reduce on the GPU(s): the P workers spread over the local
// devices (b200::dropin_devices), one host thread driving all of them --
// the reference's call shape.  Process-per-GPU callers use spardl_ctx_create
// with world_size > 1 (paper_2304_00737_b200.SparDL.from_process_group).
inline RunResult spardl_all_reduce(Fabric& fabric, const ClusterConfig& cfg,
                                   const std::vector<GradientVector>& grads,
                                   std::vector<WorkerState>& states) {
  validate(cfg);
  const int p = static_cast<int>(cfg.workers);
  if (fabric.worker_count() != p || grads.size() != size_t(p) || states.size() != size_t(p))
    throw config_error("worker count mismatch between fabric/inputs/states");
  const spardl_config c = b200::to_c(cfg);
  auto& dev = fabric.device;
  if (!dev || std::memcmp(&dev->cfg, &c, sizeof(c)) != 0) {
    dev = std::make_shared<b200::DeviceState>();
    dev->cfg = c;
    const std::vector<std::int32_t> devs = b200::dropin_devices(cfg.workers);
    b200::check(spardl_mctx_create(&c, static_cast<std::int32_t>(devs.size()), devs.data(),
                                   &dev->ctx));
    dev->last_scalars.assign(size_t(p), 0);
    dev->last_rounds.assign(size_t(p), 0);
  }
  const size_t n = static_cast<size_t>(cfg.dimension);
  // WorkerState in (value semantics): residual carries and controllers
  const size_t np = static_cast<size_t>(p);
  std::vector<std::vector<float>> g32(np, std::vector<float>(n));
  std::vector<std::vector<float>> comb(np, std::vector<float>(n));
  std::vector<const float*> gp(np);
  for (int w = 0; w < p; ++w) {
    if (states[size_t(w)].residual.mode() != cfg.residual)
      throw config_error("residual store mode differs from configuration");
    if (grads[size_t(w)].size() != cfg.dimension)
      throw config_error("apply_residual: dimension mismatch");
    std::vector<float> carry(n);
    for (size_t i = 0; i < n; ++i) {
      g32[size_t(w)][i] = static_cast<float>(grads[size_t(w)].values[i]);
      carry[i] = static_cast<float>(states[size_t(w)].residual.carry().values[i]);
      comb[size_t(w)][i] = g32[size_t(w)][i] + carry[i];
    }
    b200::check(spardl_mctx_carry_from_host(dev->ctx, w, carry.data()));
    if (cfg.sag == SagMode::bsag) {
      if (!states[size_t(w)].controller)
        throw config_error("bsag requires controller state per worker");
      b200::check(spardl_mctx_set_controller(dev->ctx, w, &states[size_t(w)].controller->raw()));
    }
    gp[size_t(w)] = g32[size_t(w)].data();
  }
  std::vector<std::int64_t> gi(size_t(cfg.k) + 1);
  std::vector<float> gv(size_t(cfg.k) + 1);
  std::int64_t nnz = 0;
  b200::check(spardl_mctx_allreduce_host(dev->ctx, gp.data(), gi.data(), gv.data(), cfg.k, &nnz));
  spardl_run_info info{};
  b200::check(spardl_mctx_get_run_info(dev->ctx, &info));

  RunResult r;
  r.global.n = cfg.dimension;
  for (std::int64_t e = 0; e < nnz; ++e) r.global.entries.push_back({gi[size_t(e)], gv[size_t(e)]});
  // every worker's own copy (each team assembles its own; on every device)
  r.per_worker.resize(size_t(p));
  for (int w = 0; w < p; ++w) {
    std::int64_t wn = 0;
    b200::check(spardl_mctx_get_global(dev->ctx, w, gi.data(), gv.data(), cfg.k, &wn));
    r.per_worker[size_t(w)].n = cfg.dimension;
    for (std::int64_t e = 0; e < wn; ++e)
      r.per_worker[size_t(w)].entries.push_back({gi[size_t(e)], gv[size_t(e)]});
  }
  r.consistent = info.consistent != 0 && verify_consistency(r.per_worker);
  // WorkerState out
  std::vector<float> carry(n);
  for (int w = 0; w < p; ++w) {
    b200::check(spardl_mctx_carry_to_host(dev->ctx, w, carry.data()));
    auto& dst = states[size_t(w)].residual.mutable_carry().values;
    for (size_t i = 0; i < n; ++i) dst[i] = carry[i];
    if (cfg.sag == SagMode::bsag)
      b200::check(spardl_mctx_get_controller(dev->ctx, w, &states[size_t(w)].controller->raw()));
  }
  // ledger: the device ledger is cumulative per context; fold its delta in
  std::vector<std::int64_t> rounds(np), scalars(np);
  b200::check(spardl_mctx_get_ledger(dev->ctx, rounds.data(), scalars.data()));
  for (int w = 0; w < p; ++w) {
    auto& l = fabric.mutable_ledger()[size_t(w)];
    l.scalars_received += scalars[size_t(w)] - dev->last_scalars[size_t(w)];
    l.rounds += rounds[size_t(w)] - dev->last_rounds[size_t(w)];
    dev->last_scalars[size_t(w)] = scalars[size_t(w)];
    dev->last_rounds[size_t(w)] = rounds[size_t(w)];
  }
  r.ledger = fabric.report();
  r.srs_phase = {info.srs_rounds, info.srs_scalars};
  r.sag_phase = {info.sag_rounds, info.sag_scalars};
  r.gather_phase = {info.gather_rounds, info.gather_scalars};
  r.predicted = {info.pred_rounds, info.pred_low, info.pred_high};
  if (info.n_union > 0) {
    r.union_sizes.resize(size_t(info.n_union));
    std::vector<std::int64_t> u(size_t(p), 0);
    b200::check(spardl_mctx_get_union_sizes(dev->ctx, u.data()));
    std::copy(u.begin(), u.begin() + std::ptrdiff_t(info.n_union), r.union_sizes.begin());
  }
  // conservation audit as the reference states it (inc/pipeline.hpp:305-334)
  r.conservation_applicable = cfg.residual == ResidualMode::gres;
  double worst = 0.0;
  {
    std::vector<double> lhs(n, 0.0), rhs(n, 0.0);
    for (int w = 0; w < p; ++w)
      for (size_t i = 0; i < n; ++i) lhs[i] += comb[size_t(w)][i];
    for (const Entry& e : r.global.entries) rhs[size_t(e.index)] += e.value;
    for (int w = 0; w < p; ++w)
      for (size_t i = 0; i < n; ++i) rhs[i] += states[size_t(w)].residual.carry().values[i];
    for (size_t i = 0; i < n; ++i) {
      const double den = std::max(1.0, lhs[i] < 0 ? -lhs[i] : lhs[i]);
      const double d = lhs[i] - rhs[i];
      worst = std::max(worst, (d < 0 ? -d : d) / den);
    }
  }
  r.conservation_error = worst;
  return r;
}

// ---------------------------------------------------------------- reporting
inline const char* to_string(SagMode m) {
  return m == SagMode::none ? "none" : (m == SagMode::rsag ? "rsag" : "bsag");
}
inline const char* to_string(ResidualMode m) {
  return m == ResidualMode::gres ? "gres" : (m == ResidualMode::pres ? "pres" : "lres");
}
inline const char* to_string(SrsTiming t) { return t == SrsTiming::optimized ? "optimized" : "naive"; }

// inc/pipeline.hpp:344-361
inline void write_run_report_header(std::ostream& os) {
  os << "P,N,k,d,sag,residual,timing,seed,max_rounds,max_scalars,"
        "predicted_rounds,predicted_scalars_low,predicted_scalars_high,"
        "consistent,conservation_error\n";
}
inline void write_run_report_row(std::ostream& os, const ClusterConfig& cfg, const RunResult& r) {
  os << cfg.workers << ',' << cfg.dimension << ',' << cfg.k << ',' << cfg.teams << ','
     << to_string(cfg.sag) << ',' << to_string(cfg.residual) << ',' << to_string(cfg.timing)
     << ',' << cfg.seed << ',' << r.ledger.max_rounds << ',' << r.ledger.max_scalars_received
     << ',' << r.predicted.rounds << ',' << r.predicted.scalars_low << ','
     << r.predicted.scalars_high << ',' << (r.consistent ? 1 : 0) << ',' << r.conservation_error
     << '\n';
}

// inc/sag.hpp:349-358
inline void write_controller_trace_header(std::ostream& os) { os << "iteration,h,step,flag,N_t,L\n"; }
inline void write_controller_trace_row(std::ostream& os, std::int64_t iter, const HController& c,
                                       std::int64_t n_t) {
  os << iter << ',' << c.h() << ',' << c.step() << ',' << (c.flag() ? 1 : 0) << ',' << n_t << ','
     << c.target() << '\n';
}

// inc/collectives.hpp:185-216: the Top-k All-Gather baseline -- local top-k
// on the GPU, Bruck all-gather over the Fabric, source-ordered merge fold on
// the GPU (a worker receives 2(P-1)k scalars in ceil(log2 P) rounds).  The
// GPU-resident form for real gradients is paper_2304_00737_b200.topka.
inline std::vector<GlobalSparseGradient> topka_baseline(Fabric& fabric,
                                                        const std::vector<GradientVector>& gradients,
                                                        Index k) {
  const int p = fabric.worker_count();
  if (static_cast<size_t>(p) != gradients.size())
    throw config_error("topka: gradient count != worker count");
  const Index n = gradients[0].size();
  if (k > n) throw config_error("topka: k must satisfy k <= N");
  std::vector<WorkerId> group;
  std::vector<SparseBlock> locals;
  for (int w = 0; w < p; ++w) {
    group.push_back(w);
    locals.push_back(top_k_select_slice(gradients[size_t(w)], 0, {0, n}, k).selected);
  }
  const GatherResult got = bruck_all_gather(fabric, group, locals);
  std::vector<GlobalSparseGradient> out(static_cast<size_t>(p));
  for (int w = 0; w < p; ++w) {
    SparseBlock acc;
    acc.block_id = 0;
    acc.range = {0, n};
    for (int s = 0; s < p; ++s) acc = merge_add(acc, got[size_t(w)][size_t(s)]);
    out[size_t(w)].n = n;
    out[size_t(w)].entries = std::move(acc.entries);
  }
  return out;
}

// inc/collectives.hpp:221-234: the dense element-wise sum in worker order,
// the reference's correctness oracle and dense baseline (no Fabric cost).
// A test utility: the dense all-reduce on B200 is NCCL's (bench.py context).
inline GradientVector dense_all_reduce_reference(const std::vector<GradientVector>& gradients) {
  if (gradients.empty()) throw group_size_error("all-reduce on empty group");
  GradientVector sum(gradients[0].size());
  for (const GradientVector& g : gradients) {
    if (g.size() != sum.size()) throw config_error("dense all-reduce: dimension mismatch");
    for (Index i = 0; i < sum.size(); ++i) sum[i] += g[i];
  }
  return sum;
}

}  // namespace spardl
