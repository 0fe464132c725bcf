// SparDL iteration planner / executor.  See engine.hpp for the overview.
//
// Reference mapping of the plan (inc/pipeline.hpp:140-342):
//   dividing           pipeline.hpp:162-184  -> div_stage_ (launch_divide + select)
//   Spar-Reduce-Scatter reduce_scatter.hpp:120-236 -> steps with phase 0
//   R-SAG / B-SAG      sag.hpp:125-249        -> steps with phase 1
//   final all-gather   pipeline.hpp:262-274  -> the gather step (phase 2)
//   assemble/finalize  pipeline.hpp:276-303  -> launch_assemble / launch_finalize
// The Fabric ledger (fabric.hpp:74-134) is reproduced exactly: rounds are
// counted on the host from the schedule, scalars on the device from the
// counts of the blocks each worker receives.
#include "engine.hpp"

#include "divplan.hpp"

#include <algorithm>
#include <cstddef>
#include <array>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <set>

#include <unistd.h>

namespace sdle {

#define CK(x)                                                                            \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess)                                                               \
      sdlh::fail(SPARDL_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));        \
  } while (0)
#define NK(x)                                                                            \
  do {                                                                                   \
    ncclResult_t r_ = (x);                                                               \
    if (r_ != ncclSuccess)                                                               \
      sdlh::fail(SPARDL_E_NCCL, std::string(#x) + ": " + ncclGetErrorString(r_));        \
  } while (0)

namespace {
constexpr int kMergeSmemEntries = 12800;
}  // namespace

// ---------------------------------------------------------------------------
Arena::~Arena() {
  for (void* p : chunks_) cudaFree(p);
}

void* Arena::alloc(size_t bytes) {
  bytes = (bytes + 255) & ~static_cast<size_t>(255);
  if (dry) {   // plan-only: distinct, aligned, never dereferenced addresses
    total_ += bytes;
    return reinterpret_cast<void*>(static_cast<uintptr_t>(0x1000) + total_ - bytes);
  }
  if (bytes > left_) {
    const size_t sz = std::max<size_t>(bytes, static_cast<size_t>(64) << 20);
    void* p = nullptr;
    CK(cudaMalloc(&p, sz));
    CK(cudaMemset(p, 0, sz));
    chunks_.push_back(p);
    cur_ = static_cast<unsigned char*>(p);
    left_ = sz;
    total_ += sz;
  }
  void* r = cur_;
  cur_ += bytes;
  left_ -= bytes;
  return r;
}

// ---------------------------------------------------------------------------
Engine::Engine(const spardl_config& cfg, int device, int world, int rank, const void* nccl_id,
               cudaStream_t stream, bool plan_only)
    : cfg_(cfg), device_(device), world_(world), rank_(rank) {
  dry_ = plan_only;
  arena_.dry = plan_only;
  sdlh::validate(cfg);
  P_ = static_cast<int>(cfg.workers);
  d_ = static_cast<int>(cfg.teams);
  m_ = P_ / d_;
  l_ = sdlh::ceil_log2(m_);
  L_ = cfg.teams * cfg.k / cfg.workers;                 // inc/pipeline.hpp:51
  Lcap_ = (L_ + 3) & ~static_cast<int64_t>(3);
  if (cfg.dimension >= (int64_t(1) << 31) - 1)
    sdlh::fail(SPARDL_E_UNSUPPORTED, "device path supports N < 2^31 - 1");
  if (world < 1 || rank < 0 || rank >= world || P_ % world != 0)
    sdlh::fail(SPARDL_E_UNSUPPORTED, "P must be a positive multiple of the process count");
  if (const char* we = std::getenv("SPARDL_WSEL")) {
    wide_on_ = we[0] != '0';
    wsel_force_ = we[0] == '1';
  }
  if (const char* wn = std::getenv("SPARDL_WSEL_MINENTRIES")) wsel_min_entries_ = std::atoll(wn);
  if (const char* wm = std::getenv("SPARDL_WSEL_MAXTASKS")) wsel_max_tasks_ = std::atoi(wm);
  if (const char* wf = std::getenv("SPARDL_WSEL_FUSE")) wsel_fuse_ = wf[0] == '1';
  if (const char* wc = std::getenv("SPARDL_WSEL_COOP")) {
    wsel_coop_ = wc[0] != '0';
    wsel_coop_force_ = wc[0] == '2';   // (tests: also where the overflow scratch carries entries)
  }
  // the cooperative select wherever a stage fits on chip, with <= 4 workers
  // per GPU (measured on B200, C4: 4 GPUs 1.212 -> 1.120 ms per step, 2 GPUs
  // 1.936 -> 1.916; with 8 workers per GPU it does not pay, C2 SRS 0.236 ->
  // 0.244 ms); SPARDL_WSEL_FIT=0/1/2 overrides
  wsel_fit_ = (P_ / world) <= 4 ? 1 : 0;
  if (const char* wf2 = std::getenv("SPARDL_WSEL_FIT")) wsel_fit_ = std::atoi(wf2);
  if (cfg.sag == SPARDL_SAG_BSAG && d_ > sdl::kMaxR)
    sdlh::fail(SPARDL_E_UNSUPPORTED, "bsag on the device supports d <= 16");
  wloc_ = P_ / world;
  first_ = rank * wloc_;
  part_ = sdlh::partition(cfg.dimension, m_);
  if (plan_only) {   // schedule inspection only: no device, no communicator
    for (int i = 0; i < wloc_; ++i) {
      carry_.push_back(static_cast<float*>(arena_.alloc(sizeof(float) * cfg.dimension)));
      ledger_total_.push_back(static_cast<int64_t*>(arena_.alloc(sizeof(int64_t))));
    }
    ledger_phase_ = static_cast<int64_t*>(arena_.alloc(sizeof(int64_t) * 3 * wloc_));
    ntot_ = static_cast<int64_t*>(arena_.alloc(sizeof(int64_t) * wloc_));
    budget_dev_ = static_cast<int64_t*>(arena_.alloc(sizeof(int64_t) * wloc_));
    ctl_dev_ = static_cast<sdl::HCtl*>(arena_.alloc(sizeof(sdl::HCtl) * wloc_));
    gtab_dev_ = static_cast<const float**>(arena_.alloc(sizeof(float*) * wloc_));
    err_dev_ = static_cast<int32_t*>(arena_.alloc(sizeof(int32_t)));
    hash_dev_ = static_cast<int64_t*>(arena_.alloc(sizeof(int64_t) * d_));
    rounds_.assign(static_cast<size_t>(P_), 0);
    phase_rounds_.assign(static_cast<size_t>(P_), {0, 0, 0});
    plan();
    carry_.clear();
    return;
  }

  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    sdlh::fail(SPARDL_E_CUDA, "no CUDA device: the SparDL device path has no CPU fallback");
  CK(cudaSetDevice(device));
  cudaDeviceProp prop{};
  CK(cudaGetDeviceProperties(&prop, device));
  if (prop.major != 10)
    sdlh::fail(SPARDL_E_CUDA, std::string("built for sm_100a (B200); device is ") + prop.name);
  if (stream) {
    stream_ = stream;
  } else {
    CK(cudaStreamCreateWithFlags(&stream_, cudaStreamNonBlocking));
    own_stream_ = true;
  }
  // a side stream for the work that may run beside the residual finalize
  CK(cudaStreamCreateWithFlags(&side_, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming));
  {
    int least = 0, greatest = 0;
    CK(cudaDeviceGetStreamPriorityRange(&least, &greatest));
    CK(cudaStreamCreateWithPriority(&hi_, cudaStreamNonBlocking, greatest));
    for (auto& e : ev_div_) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    const char* e = std::getenv("SPARDL_DIV_SPLIT");
    if (e) div_split_ = std::max(1, std::atoi(e));
  }
  if (world_ > 1) {
    if (!nccl_id) sdlh::fail(SPARDL_E_ARG, "world_size > 1 needs an NCCL unique id");
    ncclUniqueId id;
    std::memcpy(&id, nccl_id, sizeof(id));
    NK(ncclCommInitRank(&comm_, world_, id, rank_));
  }

  const size_t nbytes = static_cast<size_t>(cfg.dimension) * sizeof(float);
  for (int i = 0; i < wloc_; ++i) {
    float* c = nullptr;
    CK(cudaMalloc(&c, (nbytes + 255) & ~static_cast<size_t>(255)));
    CK(cudaMemset(c, 0, nbytes));
    carry_.push_back(c);
    ledger_total_.push_back(static_cast<int64_t*>(arena_.alloc(sizeof(int64_t))));
  }
  ledger_phase_ = static_cast<int64_t*>(arena_.alloc(sizeof(int64_t) * 3 * wloc_));
  ntot_ = static_cast<int64_t*>(arena_.alloc(sizeof(int64_t) * wloc_));
  budget_dev_ = static_cast<int64_t*>(arena_.alloc(sizeof(int64_t) * wloc_));
  ctl_dev_ = static_cast<sdl::HCtl*>(arena_.alloc(sizeof(sdl::HCtl) * wloc_));
  gtab_dev_ = static_cast<const float**>(arena_.alloc(sizeof(float*) * wloc_));
  CK(cudaMallocHost(reinterpret_cast<void**>(&gtab_host_), sizeof(float*) * wloc_ * kTabRing));
  std::memset(gtab_host_, 0, sizeof(float*) * wloc_ * kTabRing);
  gtab_cur_.assign(static_cast<size_t>(wloc_), nullptr);
  for (auto& e : tab_ev_) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  err_dev_ = static_cast<int32_t*>(arena_.alloc(sizeof(int32_t)));
  fallbacks_dev_ = static_cast<unsigned long long*>(arena_.alloc(sizeof(unsigned long long)));
  wide_back_dev_ = static_cast<unsigned long long*>(arena_.alloc(sizeof(unsigned long long)));
  retries_dev_ = static_cast<unsigned long long*>(arena_.alloc(sizeof(unsigned long long)));
  hash_dev_ = static_cast<int64_t*>(arena_.alloc(sizeof(int64_t) * d_));
  rb_dev_ = static_cast<int64_t*>(
      arena_.alloc(sizeof(int64_t) * (static_cast<size_t>(P_ + wloc_) + static_cast<size_t>(d_) * (world_ + 1))));
  rounds_.assign(static_cast<size_t>(P_), 0);
  phase_rounds_.assign(static_cast<size_t>(P_), {0, 0, 0});
  epoch_ = static_cast<long long*>(arena_.alloc(sizeof(long long)));
  peer_err_ = static_cast<int32_t*>(arena_.alloc(sizeof(int32_t)));
  if (const char* to = std::getenv("SPARDL_PEER_TIMEOUT_MS"))
    timeout_ns_ = static_cast<unsigned long long>(std::max(1, std::atoi(to))) * 1000000ull;
  setup_peer();
  plan();
  plan_peer();
  reset_state();
}

Engine::~Engine() {
  if (!dry_) cudaSetDevice(device_);
  if (graph_) cudaGraphExecDestroy(graph_);
  for (size_t q = 0; q < peer_base_.size(); ++q)
    if (peer_base_[q] && peer_base_[q] != sym_ && q < peer_ipc_.size() && peer_ipc_[q])
      cudaIpcCloseMemHandle(peer_base_[q]);
  if (sym_) cudaFree(sym_);
  if (comm_) ncclCommDestroy(comm_);
  for (float* c : carry_) cudaFree(c);
  if (gtab_host_) cudaFreeHost(gtab_host_);
  for (auto& e : tab_ev_)
    if (e) cudaEventDestroy(e);
  if (side_) cudaStreamDestroy(side_);
  if (ev_fork_) cudaEventDestroy(ev_fork_);
  if (ev_join_) cudaEventDestroy(ev_join_);
  if (hi_) cudaStreamDestroy(hi_);
  for (auto& e : ev_div_)
    if (e) cudaEventDestroy(e);
  if (own_stream_) cudaStreamDestroy(stream_);
}

std::vector<PlanOp> Engine::plan_ops() const {
  std::vector<PlanOp> ops;
  int round = 0;
  for (const Step& s : steps_) {
    if (s.xfers.empty()) continue;
    for (const Xfer& x : s.xfers) {
      if (x.src_rank == x.dst_rank) continue;
      const bool send = x.src_rank == rank_;
      ops.push_back({round, send ? x.dst_rank : x.src_rank, send ? 1 : 0, x.uid,
                     static_cast<int64_t>(16 + 8 * Lcap_)});
    }
    ++round;
  }
  return ops;
}

void Engine::drop_graph() {
  if (graph_) {
    cudaGraphExecDestroy(graph_);
    graph_ = nullptr;
  }
}

// ---------------------------------------------------------------------------
// planning helpers
int Engine::new_uid(int owner) {
  uid_owner_.push_back(owner);
  if (rank_slots_.size() != static_cast<size_t>(world_)) rank_slots_.assign(static_cast<size_t>(world_), 0);
  // every uid has its own buffer index on every rank (peer transport: a
  // producer may write a block straight into its consumer's copy)
  rank_slots_[static_cast<size_t>(rank_of(owner))]++;
  uid_slot_.push_back(next_uid_);
  return next_uid_++;
}

Slot& Engine::local_slot(int uid) {
  auto it = slots_.find(uid);
  if (it == slots_.end()) sdlh::fail(SPARDL_E_ERROR, "internal: block buffer not resident");
  return it->second;
}

Slot Engine::sym_slot(int uid) const {
  const int r = uid_owner_[static_cast<size_t>(uid)] / wloc_;
  Slot s;
  s.cap = Lcap_;
  s.bytes = 16 + 8 * static_cast<size_t>(Lcap_);
  s.base = peer_base_[static_cast<size_t>(r)] + slot_stride_ * static_cast<size_t>(uid_slot_[static_cast<size_t>(uid)]);
  s.cnt = reinterpret_cast<int32_t*>(s.base);
  s.idx = reinterpret_cast<int32_t*>(s.base + 16);
  s.val = reinterpret_cast<float*>(s.base + 16 + 4 * static_cast<size_t>(Lcap_));
  return s;
}

Slot Engine::own_slot(int uid) const {
  Slot s = sym_slot(uid);
  const size_t off = slot_stride_ * static_cast<size_t>(uid_slot_[static_cast<size_t>(uid)]);
  s.base = peer_base_[static_cast<size_t>(rank_)] + off;
  s.cnt = reinterpret_cast<int32_t*>(s.base);
  s.idx = reinterpret_cast<int32_t*>(s.base + 16);
  s.val = reinterpret_cast<float*>(s.base + 16 + 4 * static_cast<size_t>(Lcap_));
  return s;
}

// A block with remote consumer ranks: its producing select also writes the
// selection into each consumer's copy (the same place in its region).
void Engine::wire_push(sdl::SelTask& t, int uid) {
  if (!peer_) return;
  auto pd = push_dst_.find(uid);
  if (pd == push_dst_.end()) return;
  std::vector<unsigned char*> bases;
  for (int r : pd->second)
    bases.push_back(peer_base_[static_cast<size_t>(r)] +
                    slot_stride_ * static_cast<size_t>(uid_slot_[static_cast<size_t>(uid)]));
  auto* d = static_cast<unsigned char**>(arena_.alloc(sizeof(unsigned char*) * bases.size()));
  CK(mcpy(d, bases.data(), sizeof(unsigned char*) * bases.size(), cudaMemcpyHostToDevice));
  t.push_base = d;
  t.npush = static_cast<int32_t>(bases.size());
  t.push_cap = static_cast<int32_t>(Lcap_);
}

// A block buffer.  Peer transport: the buffer lives at a fixed place of its
// owner's symmetric region (the same numbering on every rank), so a consumer
// on another GPU addresses it directly; otherwise a private buffer that a
// transport round fills.
Slot Engine::make_slot(int uid) {
  if (peer_) return sym_slot(uid);
  Slot s;
  s.cap = Lcap_;
  s.bytes = 16 + 8 * static_cast<size_t>(Lcap_);
  s.base = static_cast<unsigned char*>(arena_.alloc(s.bytes));
  s.cnt = reinterpret_cast<int32_t*>(s.base);
  s.idx = reinterpret_cast<int32_t*>(s.base + 16);
  s.val = reinterpret_cast<float*>(s.base + 16 + 4 * static_cast<size_t>(Lcap_));
  return s;
}

void Engine::add_select(Stage& st, const sdl::SelTask& t0, int out_uid, int in_uid) {
  st.sel_uid.push_back(out_uid);
  st.sel_in.push_back(in_uid);
  sdl::SelTask t = t0;
  // t.stride carries the longest possible input segment (see callers)
  sdl::sel_prepare(t, t.stride);
  if (t.nseg > sdl::kMaxSegPerTask || t.dnseg > sdl::kMaxSegPerTask)
    sdlh::fail(SPARDL_E_UNSUPPORTED, "selection larger than the device work-item bound");
  t.scr = static_cast<sdl::SelScratch*>(arena_.alloc(sizeof(sdl::SelScratch)));
  const int nck = std::max(1, sdl::sel_chunk_capacity(t));
  int32_t* segs = static_cast<int32_t*>(arena_.alloc(sizeof(int32_t) * 6 * nck));
  t.seg_gt = segs;
  t.seg_eq = segs + nck;
  t.seg_sel_off = segs + 2 * nck;
  t.seg_dis_off = segs + 3 * nck;
  t.seg_take = segs + 4 * nck;
  t.seg_valid = segs + 5 * nck;
  // the select's per-CTA segment table is sized for a whole task's segments
  st.max_nseg = std::max(st.max_nseg, sdl::sel_scratch_segments(t));
  st.sels.push_back(t);
}

sdl::WScratch* Engine::make_wide(Stage& st, sdl::SelTask& t, const int32_t* idx, const float* val,
                                  const int32_t* seg_off, const int32_t* seg_cnt,
                                  const int32_t* count, int stride, int nseg, int group, int mode,
                                  int is_div, int64_t bin_cap, int64_t typical) {
  sdl::WScratch w{};
  w.idx = idx;
  w.val = val;
  w.seg_off = seg_off;
  w.seg_cnt = seg_cnt;
  w.count = count;
  w.stride = stride;
  w.nseg = nseg;
  w.group = std::max(1, std::min(group, 64));
  w.max_tiles = (nseg + w.group - 1) / w.group;
  w.mode = mode;
  w.is_div = is_div;
  w.handed_back = wide_back_dev_;
  bin_cap = std::max<int64_t>(1, std::min<int64_t>(bin_cap, int64_t(1) << 30));
  w.bin_cap = static_cast<int32_t>(bin_cap);
  w.bin_c = static_cast<unsigned long long*>(arena_.alloc(sizeof(unsigned long long) * bin_cap));
  w.bin_tile = static_cast<int32_t*>(arena_.alloc(sizeof(int32_t) * bin_cap));
  const size_t nt = static_cast<size_t>(std::max(1, w.max_tiles));
  w.tile_n = static_cast<int32_t*>(arena_.alloc(sizeof(int32_t) * nt));
  w.tile_sel = static_cast<int32_t*>(arena_.alloc(sizeof(int32_t) * nt));
  w.tile_sel_off = static_cast<int32_t*>(arena_.alloc(sizeof(int32_t) * nt));
  w.tile_dis_off = static_cast<int32_t*>(arena_.alloc(sizeof(int32_t) * nt));
  // the cooperative form's overflow scratch (entries past the CTAs' shared
  // copies, at their flat position): the task's input capacity
  w.ov_cap = std::max<int64_t>(1, typical);
  w.ov_val = static_cast<float*>(arena_.alloc(sizeof(float) * static_cast<size_t>(w.ov_cap)));
  w.ov_idx = static_cast<int32_t*>(arena_.alloc(sizeof(int32_t) * static_cast<size_t>(w.ov_cap)));
  auto* d = static_cast<sdl::WScratch*>(arena_.alloc(sizeof(sdl::WScratch)));
  CK(mcpy(d, &w, sizeof(w), cudaMemcpyHostToDevice));
  t.ws = d;
  st.w_max_tiles = std::max(st.w_max_tiles, w.max_tiles);
  st.w_max_nseg = std::max(st.w_max_nseg, nseg);
  st.w_max_entries = std::max<int64_t>(st.w_max_entries, typical);
  st.ws.push_back(d);
  return d;
}

sdl::SelTask Engine::select_from_slot(const Slot& in) {
  sdl::SelTask t{};
  t.mode = 0;
  t.idx = in.idx;
  t.val = in.val;
  t.count = in.cnt;
  int64_t stride = sdl::kTile;
  while ((in.cap + stride - 1) / stride > sdl::kMaxSegPerTask) stride += sdl::kTile;
  t.stride = static_cast<int32_t>(stride);
  t.nseg = static_cast<int32_t>((in.cap + stride - 1) / stride);
  t.weight = 1.f;
  return t;
}

sdl::SelTask Engine::select_from_merge(Stage& st, const std::vector<int>& pieces) {
  const int r = static_cast<int>(pieces.size());
  if (r > sdl::kMaxR) sdlh::fail(SPARDL_E_UNSUPPORTED, "merge fan-in above 16 lists");
  sdl::MergeTask mt{};
  mt.r = r;
  int64_t capsum = 0;
  for (int q = 0; q < r; ++q) {
    const Slot& s = local_slot(pieces[static_cast<size_t>(q)]);
    mt.in_idx[q] = s.idx;
    mt.in_val[q] = s.val;
    mt.in_cnt[q] = s.cnt;
    capsum += s.cap;
  }
  static const int64_t tnum = [] {
    const char* e = std::getenv("SPARDL_MERGE_TNUM");   // tuning experiments only
    return static_cast<int64_t>(e ? std::atoi(e) : 2048);
  }();
  int64_t T = std::max<int64_t>(tnum / r, (capsum + sdl::kMaxSamples - 1) / sdl::kMaxSamples);
  T = (std::max<int64_t>(T, 32) + 3) & ~int64_t(3);   // windows start 16-byte aligned
  if (static_cast<int64_t>(r) * T > kMergeSmemEntries)
    sdlh::fail(SPARDL_E_UNSUPPORTED, "merge of this size exceeds the shared-memory envelope");
  mt.T = static_cast<int32_t>(T);
  int64_t parts = 0;
  for (int q = 0; q < r; ++q) parts += (Lcap_ + T - 1) / T;
  mt.max_parts = static_cast<int32_t>(parts);
  mt.splitters = static_cast<int32_t*>(arena_.alloc(sizeof(int32_t) * (parts + 1)));
  mt.windows = static_cast<int32_t*>(arena_.alloc(sizeof(int32_t) * parts * r));
  mt.nparts = static_cast<int32_t*>(arena_.alloc(sizeof(int32_t)));
  mt.out_idx = static_cast<int32_t*>(arena_.alloc(sizeof(int32_t) * capsum));
  mt.out_val = static_cast<float*>(arena_.alloc(sizeof(float) * capsum));
  mt.out_cap = capsum;
  mt.seg_off = static_cast<int32_t*>(arena_.alloc(sizeof(int32_t) * parts));
  mt.seg_cnt = static_cast<int32_t*>(arena_.alloc(sizeof(int32_t) * parts));
  st.merges.push_back(mt);
  st.merge_cap.push_back(capsum);
  st.merge_in.push_back(pieces);
  st.max_parts = std::max<int>(st.max_parts, static_cast<int>(parts));
  st.max_rT = std::max<int>(st.max_rT, static_cast<int>(r * T));
  st.max_r = std::max<int>(st.max_r, r);

  sdl::SelTask t{};
  t.mode = 0;
  t.idx = mt.out_idx;
  t.val = mt.out_val;
  t.seg_off = mt.seg_off;
  t.seg_cnt = mt.seg_cnt;
  t.nseg = static_cast<int32_t>(parts);
  t.stride = static_cast<int32_t>(r * T);   // longest partition (offsets come from seg_off)
  t.weight = 1.f;
  t.merge_slot = static_cast<int32_t>(st.merges.size());
  return t;
}

// Merge `pieces` (fold order) and select `budget` of them; the result is a
// new block owned by worker w.  Discards go to worker w's residual list for
// block `xi_block` (inc/reduce_scatter.hpp:102-110 / sag.hpp:160-164 /
// sag.hpp:213-218 / sag.hpp:238-244 -> ResidualStore::record_inproc).
int Engine::materialize(int w, int pos, std::vector<int> pieces, int64_t budget, float weight,
                        const int64_t* budget_dev, int64_t* total_out, Stage& st,
                        int xi_block) {
  (void)pos;
  const int uid = new_uid(w);
  for (int u : pieces)
    if (st.produced.count(u))
      sdlh::fail(SPARDL_E_ERROR, "internal: stage reads a block produced in the same stage");
  st.produced.insert(uid);
  if (!is_local(w)) return uid;
  const int li = w - first_;
  Slot out = make_slot(uid);
  slots_[uid] = out;
  sdl::SelTask t = pieces.size() == 1 ? select_from_slot(local_slot(pieces[0]))
                                      : select_from_merge(st, pieces);
  t.budget = budget;
  t.budget_dev = budget_dev;
  t.weight = weight;
  t.total_out = total_out;
  t.sel_idx = out.idx;
  t.sel_val = out.val;
  t.sel_cnt = out.cnt;
  wire_push(t, uid);
  int64_t capsum = 0;
  for (int u : pieces) capsum += local_slot(u).cap;
  t.dis_idx = static_cast<int32_t*>(arena_.alloc(sizeof(int32_t) * capsum));
  t.dis_val = static_cast<float*>(arena_.alloc(sizeof(float) * capsum));
  t.sel_cap = static_cast<int32_t>(out.cap);
  t.dis_cap = static_cast<int32_t>(capsum);
  t.dis_cnt = static_cast<int32_t*>(arena_.alloc(sizeof(int32_t)));
  xi_[static_cast<size_t>(li)][static_cast<size_t>(xi_block)].push_back(
      {t.dis_idx, t.dis_val, t.dis_cnt});
  if (wide_on_) {
    if (pieces.size() == 1) {   // a single block buffer: one compact list
      const Slot& in = local_slot(pieces[0]);
      constexpr int kStride = 8192;
      make_wide(st, t, in.idx, in.val, nullptr, nullptr, in.cnt, kStride,
                static_cast<int>((in.cap + kStride - 1) / kStride), 1, sdl::kWAuto, 0,
                std::max<int64_t>(16384, in.cap / 8), in.cap);
    } else {                    // the merge's partitions
      const sdl::MergeTask& mt = st.merges.back();
      make_wide(st, t, mt.out_idx, mt.out_val, mt.seg_off, mt.seg_cnt, nullptr, t.stride, t.nseg,
                std::max(1, 8192 / std::max(1, static_cast<int>(mt.T))), sdl::kWAuto, 0,
                std::max<int64_t>(16384, capsum / 8), capsum);
    }
  }
  add_select(st, t, uid, pieces.size() == 1 ? pieces[0] : -1);
  if (t.merge_slot)   // diagnostics: the merge stamps its phases into the select's scratch
    st.merges[static_cast<size_t>(t.merge_slot - 1)].dbg = st.sels.back().scr->merge_ts;
  return uid;
}

// Moves block `uid` from worker src to worker dst in the current round.
// Physical transfers are deduplicated per (block, destination rank): workers
// co-resident on a device read the same buffer.  The ledger still charges
// every receiving worker (inc/fabric.hpp:95-106).
void Engine::transfer(std::vector<Xfer>& xs, int uid, int src, int dst, int phase,
                      std::vector<std::vector<int>>* recv_into) {
  (void)recv_into;
  const int sr = rank_of(src), dr = rank_of(dst);
  deliveries_.push_back({uid, dr});
  if (dr == rank_) {
    if (!has_local(uid)) {
      // a pushed block arrives in this rank's own copy of the buffer
      slots_[uid] = peer_ && push_dst_.count(uid) ? own_slot(uid) : make_slot(uid);
      xs.push_back({uid, src, sr, dr});
    }
    const int li = dst - first_;
    const Slot& s = local_slot(uid);
    ledger_adds_.push_back({ledger_total_[static_cast<size_t>(li)], s.cnt});
    ledger_adds_.push_back({ledger_phase_ + 3 * li + phase, s.cnt});
  } else if (sr == rank_) {
    bool dup = false;
    for (const Xfer& x : xs)
      if (x.uid == uid && x.dst_rank == dr) dup = true;
    if (!dup) xs.push_back({uid, src, sr, dr});
  }
}

// Fused merge+select for a stage: the widest cluster whose per-CTA window
// fits shared memory and whose clusters are all resident at once.
void Engine::plan_fused(Stage& st) {
  // opt-in: on B200 the separate merge kernels (every SM busy) beat the
  // fused prologue (one cluster per task) -- see DESIGN.md
  const char* env = std::getenv("SPARDL_FUSED_MERGE");
  if (dry_ || st.merges.empty() || !env || std::strcmp(env, "1") != 0) return;
  int64_t capmax = 0;
  int rmax = 0, tab = 1;
  for (size_t i = 0; i < st.merges.size(); ++i) {
    capmax = std::max(capmax, st.merge_cap[i]);
    rmax = std::max(rmax, static_cast<int>(st.merges[i].r));
  }
  for (const auto& t : st.sels)
    if (!t.merge_slot) tab = std::max(tab, sdl::sel_scratch_segments(t));
  const int64_t Ts = (std::max<int64_t>(32, (capmax + sdl::kMergeSamples - 1) / sdl::kMergeSamples) + 3) & ~int64_t(3);
  const int maxwin = sdl::select_max_window();
  const int ntask = static_cast<int>(st.sels.size());
  for (int cl : {16, 8, 4, 2}) {
    const int64_t win = (capmax + cl - 1) / cl + (2 * rmax + 2) * Ts;
    if (win > maxwin) continue;
    if (sdl::select_resident_clusters(cl, tab, static_cast<int>(win)) < ntask) continue;
    st.fused = true;
    st.cl = cl;
    st.win_cap = static_cast<int>(win);
    st.max_nseg = tab;
    for (auto& mt : st.merges) mt.T = static_cast<int32_t>(Ts);
    return;
  }
}

void Engine::finish_stage(Stage& st) {
  plan_fused(st);
  // the wide select where the cluster select cannot fill the GPU: one worker
  // per GPU (the north-star split), few selections (<= SPARDL_WSEL_MAXTASKS)
  // of large inputs (>= 200k entries).  Measured on B200 (C4, 4 GPUs): one
  // worker per GPU 0.873 -> 0.771 ms per step; two per GPU 1.349 -> 1.370
  // (the cluster selects of 4-16 tasks already fill the GPU); C2's 64k-128k
  // entry selects favour the cluster select's single kernel (0.415 vs 0.507).
  // SPARDL_WSEL=1: every stage, =0: none.
  const bool fits = wsel_fit_ && !dry_ &&
                   st.w_max_entries <= sdl::wsel_coop_capacity(static_cast<int>(st.sels.size()), st.w_max_nseg) &&
                   (wsel_fit_ == 2 || &st != &div_stage_);
  st.wide = !st.fused && !st.sels.empty() && st.ws.size() == st.sels.size() &&
            (wsel_force_ || st.need_wide || fits ||
             (wloc_ == 1 && static_cast<int>(st.sels.size()) <= wsel_max_tasks_ &&
              st.w_max_entries >= wsel_min_entries_));
  if (!st.wide)
    for (auto& t : st.sels) t.ws = nullptr;   // (cluster selects only)
  // the single-kernel form when every task's segment table and entries fit
  // (the tiled form otherwise; producer-fused dividing histograms need it)
  // (where a stage's typical entries fit the CTAs' shared copies: the
  // overflow scratch is measured slower than the tiled form when it carries a
  // large share -- C4 with 8 workers per GPU: SRS 0.955 vs 0.755 ms -- and
  // only catches runs past the typical size)
  st.coop = st.wide && wsel_coop_ && !dry_ && st.w_max_nseg <= sdl::wsel_coop_max_seg() &&
            !(&st == &div_stage_ && wsel_fuse_) &&
            (wsel_coop_force_ ||
             st.w_max_entries <= sdl::wsel_coop_capacity(static_cast<int>(st.sels.size()), st.w_max_nseg));
  if (!st.sels.empty())
    st.sels_dev =
        static_cast<sdl::SelTask*>(arena_.alloc(sizeof(sdl::SelTask) * st.sels.size()));
  if (!st.merges.empty())
    st.merges_dev = static_cast<sdl::MergeTask*>(
        arena_.alloc(sizeof(sdl::MergeTask) * st.merges.size()));
  // a wide select fed by a merge: the merge histograms its output and
  // decides (no histogram pass for that select; opt-in SPARDL_WSEL_FUSE=1:
  // measured slower on B200, every small merge CTA flushes a 2048-bin
  // histogram)
  if (st.wide && wsel_fuse_ && !st.merges.empty())
    for (size_t i = 0; i < st.sels.size(); ++i) {
      sdl::SelTask& t = st.sels[i];
      if (!t.merge_slot) continue;
      sdl::MergeTask& mt = st.merges[static_cast<size_t>(t.merge_slot - 1)];
      mt.ws = t.ws;
      mt.sel = st.sels_dev + i;
      const int32_t one = 1;
      CK(mcpy(reinterpret_cast<unsigned char*>(t.ws) + offsetof(sdl::WScratch, by_merge), &one,
              sizeof(one), cudaMemcpyHostToDevice));
    }
  if (!st.merges.empty()) {
    CK(mcpy(st.merges_dev, st.merges.data(), sizeof(sdl::MergeTask) * st.merges.size(),
                  cudaMemcpyHostToDevice));
    if (!st.fused) launches_ += 2;
  }
  if (st.fused)
    for (auto& t : st.sels)
      if (t.merge_slot) {
        t.merge = st.merges_dev + (t.merge_slot - 1);
        t.nseg = 1;
      }
  if (!st.sels.empty()) {
    CK(mcpy(st.sels_dev, st.sels.data(), sizeof(sdl::SelTask) * st.sels.size(),
                  cudaMemcpyHostToDevice));
    launches_ += 9;
  }
  if (std::getenv("SPARDL_PLAN_DEBUG") && rank_ == 0) {   // the stage's shape (diagnostics)
    std::string line = "stage: " + std::to_string(st.merges.size()) + " merges r/T/out_cap:";
    for (const auto& mt : st.merges)
      line += " " + std::to_string(mt.r) + "/" + std::to_string(mt.T) + "/" +
              std::to_string(mt.out_cap);
    line += " | " + std::to_string(st.sels.size()) + " selects budget/nseg:";
    for (const auto& t : st.sels)
      line += " " + std::to_string(t.budget) + "/" + std::to_string(t.nseg);
    line += st.wide ? " (wide)" : (st.fused ? " (fused)" : "");
    std::fprintf(stderr, "%s\n", line.c_str());
  }
}

// the wide scratch of every task of a stage back to its idle state
void Engine::reset_wide(const Stage& st) {
  for (sdl::WScratch* w : st.ws) {
    // hist .. ntiles (the run state); the input descriptor and buffers stay
    const size_t a = offsetof(sdl::WScratch, hist), b = offsetof(sdl::WScratch, total);
    CK(cudaMemset(reinterpret_cast<unsigned char*>(w) + a, 0, b - a));
    // the cooperative form's histograms, barrier and counts (in the bin buffer)
    unsigned long long* bc = nullptr;
    CK(mcpy(&bc, reinterpret_cast<unsigned char*>(w) + offsetof(sdl::WScratch, bin_c), sizeof(bc),
            cudaMemcpyDeviceToHost));
    if (bc) CK(cudaMemset(bc, 0, sizeof(uint32_t) * sdl::wsel_coop_words()));
  }
}

// ---------------------------------------------------------------------------
void Engine::plan() {
  const int64_t N = cfg_.dimension;
  div_uid_.assign(static_cast<size_t>(wloc_), std::vector<int>(static_cast<size_t>(m_), -1));
  div_scr_.assign(static_cast<size_t>(wloc_),
                  std::vector<const sdl::SelScratch*>(static_cast<size_t>(m_), nullptr));
  xi_.assign(static_cast<size_t>(wloc_),
             std::vector<std::vector<sdl::XiList>>(static_cast<size_t>(m_)));
  std::vector<std::vector<std::vector<int>>> held(
      static_cast<size_t>(P_), std::vector<std::vector<int>>(static_cast<size_t>(m_)));
  std::vector<std::vector<char>> has(static_cast<size_t>(P_),
                                     std::vector<char>(static_cast<size_t>(m_), 1));

  // ---- dividing (inc/pipeline.hpp:162-184)
  int max_chunks = 0;
  for (int w = 0; w < P_; ++w) {
    for (int b = 0; b < m_; ++b) {
      const int uid = new_uid(w);
      held[static_cast<size_t>(w)][static_cast<size_t>(b)] = {uid};
      div_stage_.produced.insert(uid);
      if (!is_local(w)) continue;
      const int li = w - first_;
      div_uid_[static_cast<size_t>(li)][static_cast<size_t>(b)] = uid;
      Slot out = make_slot(uid);
      slots_[uid] = out;
      const int64_t lo = part_.lo[static_cast<size_t>(b)], hi = part_.hi[static_cast<size_t>(b)];
      sdl::DivTask dt{};
      sdl::SelTask t{};
      sdl::div_plan(dt, t, lo, hi, L_, [&](size_t n) { return arena_.alloc(n); });
      dt.g_tab = gtab_dev_;
      dt.g_id = li;
      dt.carry = carry_[static_cast<size_t>(li)];
      dt.err = err_dev_;
      div_tasks_.push_back(dt);
      max_chunks = std::max(max_chunks, dt.nchunks);
      t.dval = dt.carry + lo;
      t.fallbacks = fallbacks_dev_;
      t.sel_cap = static_cast<int32_t>(out.cap);
      if (dt.huge) div_stage_.need_wide = true;   // (the cluster select would go dense)
      if (dt.use_cand && div_split_ <= 1 && (wide_on_ || dt.huge)) {
        div_tasks_.back().ws_fused = wsel_fuse_ ? 1 : 0;
        div_tasks_.back().ws = make_wide(div_stage_, t, dt.cand_idx, dt.cand_val, nullptr,
                                         dt.cand_cnt, nullptr, dt.cap, dt.nchunks, 64,
                                         sdl::kWWindow, 1, std::max<int64_t>(16384, L_ / 8),
                                         L_ + L_ / 3);
      }
      t.sel_idx = out.idx;
      t.sel_val = out.val;
      t.sel_cnt = out.cnt;
      wire_push(t, uid);
      add_select(div_stage_, t, uid, -1);
      div_scr_[static_cast<size_t>(li)][static_cast<size_t>(b)] = div_stage_.sels.back().scr;
    }
  }
  // one sample_every for the whole batch (the launcher sizes its grid with it)
  // ~8 sampled chunks (65k elements) per block: ~650 expected top-L samples
  // at 1% density whatever the block size (the 4-sigma margin is ~15%)
  div_sample_every_ = std::max(1, max_chunks / 8);
  for (auto& dt : div_tasks_) {
    dt.sample_every = div_sample_every_;
    dt.retries = retries_dev_;
  }
  div_max_chunks_ = max_chunks;
  if (!div_tasks_.empty()) {
    div_dev_ = static_cast<sdl::DivTask*>(arena_.alloc(sizeof(sdl::DivTask) * div_tasks_.size()));
    CK(mcpy(div_dev_, div_tasks_.data(), sizeof(sdl::DivTask) * div_tasks_.size(),
                  cudaMemcpyHostToDevice));
    launches_ += 3;
  }
  finish_stage(div_stage_);

  auto team_of = [&](int w) { return w / m_; };
  auto pos_in_team = [&](int w) { return w % m_; };
  std::vector<sdlh::Bags> bags;
  for (int i = 0; i < m_; ++i) bags.push_back(sdlh::build_bags(m_, i));
  const bool naive = cfg_.timing == SPARDL_TIMING_NAIVE;

  auto materialize_pending = [&](Stage& st) {
    for (int w = 0; w < P_; ++w)
      for (int b = 0; b < m_; ++b) {
        auto& h = held[static_cast<size_t>(w)][static_cast<size_t>(b)];
        if (h.size() > 1) h = {materialize(w, b, h, L_, 1.f, nullptr, nullptr, st, b)};
      }
  };

  // ---- Spar-Reduce-Scatter (inc/reduce_scatter.hpp:120-236)
  for (int s = 1; s <= l_; ++s) {
    Step step;
    const int dist = 1 << (l_ - s);
    const int bi = l_ - s + 1;
    if (naive) materialize_pending(step.stage);   // blocks merged at step s-1
    for (int w = 0; w < P_; ++w) {
      const int i = pos_in_team(w);
      for (int pos : bags[static_cast<size_t>(i)].bags[static_cast<size_t>(bi - 1)]) {
        if (!has[static_cast<size_t>(w)][static_cast<size_t>(pos)])
          sdlh::fail(SPARDL_E_THEOREM, "sending a block already given up");
        auto& h = held[static_cast<size_t>(w)][static_cast<size_t>(pos)];
        // optimized timing: the blocks of the bag about to leave are
        // sparsified now (inc/reduce_scatter.hpp:207-215)
        if (h.size() > 1) h = {materialize(w, pos, h, L_, 1.f, nullptr, nullptr, step.stage, pos)};
      }
    }
    for (int w = 0; w < P_; ++w) {
      const int t = team_of(w), i = pos_in_team(w);
      const int target = t * m_ + (i + dist) % m_;
      for (int pos : bags[static_cast<size_t>(i)].bags[static_cast<size_t>(bi - 1)]) {
        auto& h = held[static_cast<size_t>(w)][static_cast<size_t>(pos)];
        const int uid = h[0];
        h.clear();
        has[static_cast<size_t>(w)][static_cast<size_t>(pos)] = 0;
        if (!has[static_cast<size_t>(target)][static_cast<size_t>(pos)])
          sdlh::fail(SPARDL_E_THEOREM, "received block " + std::to_string(pos) +
                                           " not held by worker " + std::to_string(target));
        transfer(step.xfers, uid, w, target, 0);
        held[static_cast<size_t>(target)][static_cast<size_t>(pos)].push_back(uid);
      }
      phase_rounds_[static_cast<size_t>(w)][0] += 1;
    }
    finish_stage(step.stage);
    steps_.push_back(std::move(step));
  }
  // reserved block: sparsified once after the last merge (reduce_scatter.hpp:220-234)
  Step res;
  if (naive) materialize_pending(res.stage);
  std::vector<int> R(static_cast<size_t>(P_));
  for (int w = 0; w < P_; ++w) {
    const int i = pos_in_team(w);
    auto& h = held[static_cast<size_t>(w)][static_cast<size_t>(i)];
    if (h.empty()) sdlh::fail(SPARDL_E_ERROR, "preservation block missing after reduce-scatter");
    if (h.size() > 1) h = {materialize(w, i, h, L_, 1.f, nullptr, nullptr, res.stage, i)};
    R[static_cast<size_t>(w)] = h[0];
  }

  // ---- Spar-All-Gather across teams (inc/sag.hpp:125-249)
  Step* open = &res;        // stage that runs before the next transport round
  std::vector<Step> sag_steps;
  union_group_owner_.clear();
  if (d_ > 1 && cfg_.sag == SPARDL_SAG_RSAG) {
    const int steps = sdlh::exact_log2(d_);
    for (int ts = 0; ts < steps; ++ts) {
      const int dist = 1 << ts;
      // round: every member swaps its block with the partner at XOR distance
      std::vector<int> recv(static_cast<size_t>(P_), -1);
      for (int g = 0; g < m_; ++g)
        for (int t = 0; t < d_; ++t) {
          const int w = t * m_ + g, partner = (t ^ dist) * m_ + g;
          transfer(open->xfers, R[static_cast<size_t>(w)], w, partner, 1);
          recv[static_cast<size_t>(partner)] = R[static_cast<size_t>(w)];
          phase_rounds_[static_cast<size_t>(w)][1] += 1;
        }
      finish_stage(open->stage);
      steps_.push_back(std::move(*open));
      Step next;
      const float share = 1.f / static_cast<float>(2 * dist);   // sag.hpp:153
      for (int g = 0; g < m_; ++g)
        for (int t = 0; t < d_; ++t) {
          const int w = t * m_ + g;
          R[static_cast<size_t>(w)] =
              materialize(w, g, {R[static_cast<size_t>(w)], recv[static_cast<size_t>(w)]}, L_,
                          share, nullptr, nullptr, next.stage, g);
        }
      sag_steps.push_back(std::move(next));
      open = &sag_steps.back();
    }
  } else if (d_ > 1) {
    // B-SAG: pre-select h (weight 1), gather unmerged, fold in source order,
    // select L with dyadic shares, observe N_t (inc/sag.hpp:189-249,
    // inc/pipeline.hpp:224-257)
    const std::vector<double> shares = sdlh::dyadic_shares(d_);
    std::vector<int> Q(static_cast<size_t>(P_));
    // the pre-selection reads the reserved blocks: it needs its own stage
    finish_stage(open->stage);
    steps_.push_back(std::move(*open));
    sag_steps.emplace_back();
    open = &sag_steps.back();
    for (int g = 0; g < m_; ++g)
      for (int t = 0; t < d_; ++t) {
        const int w = t * m_ + g;
        const int li = w - first_;
        Q[static_cast<size_t>(w)] =
            materialize(w, g, {R[static_cast<size_t>(w)]}, L_, 1.f,
                        is_local(w) ? budget_dev_ + li : nullptr, nullptr, open->stage, g);
      }
    for (int g = 0; g < m_; ++g)
      for (int s = 0; s < d_; ++s) {
        const int ws = s * m_ + g;
        for (int i = 0; i < d_; ++i) {
          if (i == s) continue;
          transfer(open->xfers, Q[static_cast<size_t>(ws)], ws, i * m_ + g, 1);
        }
        phase_rounds_[static_cast<size_t>(ws)][1] += sdlh::ceil_log2(d_);
      }
    finish_stage(open->stage);
    steps_.push_back(std::move(*open));
    Step post;
    for (int g = 0; g < m_; ++g) {
      union_group_owner_.push_back(g);   // worker t=0 of group g reports N_t
      for (int i = 0; i < d_; ++i) {
        const int w = i * m_ + g;
        std::vector<int> pieces;
        for (int s = 0; s < d_; ++s) pieces.push_back(Q[static_cast<size_t>(s * m_ + g)]);
        const int li = w - first_;
        R[static_cast<size_t>(w)] =
            materialize(w, g, pieces, L_, static_cast<float>(shares[static_cast<size_t>(i)]),
                        nullptr, is_local(w) ? ntot_ + li : nullptr, post.stage, g);
      }
    }
    post.controller_after = true;
    sag_steps.push_back(std::move(post));
    open = &sag_steps.back();
  }

  // ---- final all-gather inside each team (inc/pipeline.hpp:262-274)
  std::vector<std::vector<int>> team_blocks(static_cast<size_t>(d_));
  for (int t = 0; t < d_; ++t) {
    for (int j = 0; j < m_; ++j) {
      const int wj = t * m_ + j;
      team_blocks[static_cast<size_t>(t)].push_back(R[static_cast<size_t>(wj)]);
      for (int i = 0; i < m_; ++i) {
        if (i == j) continue;
        transfer(open->xfers, R[static_cast<size_t>(wj)], wj, t * m_ + i, 2);
      }
      phase_rounds_[static_cast<size_t>(wj)][2] += sdlh::ceil_log2(m_);
    }
  }
  finish_stage(open->stage);
  steps_.push_back(std::move(*open));

  // ---- assemble per (team, device) and finalize per worker (pipeline.hpp:276-303)
  team_of_local_global_.assign(static_cast<size_t>(wloc_), -1);
  int64_t max_m = m_;
  for (int t = 0; t < d_; ++t) {
    bool any = false;
    for (int j = 0; j < m_; ++j) any |= is_local(t * m_ + j);
    if (!any) continue;
    std::vector<sdl::GatherSrc> src;
    for (int j = 0; j < m_; ++j) {
      const Slot& s = local_slot(team_blocks[static_cast<size_t>(t)][static_cast<size_t>(j)]);
      src.push_back({s.idx, s.val, s.cnt});
    }
    auto* src_dev = static_cast<sdl::GatherSrc*>(arena_.alloc(sizeof(sdl::GatherSrc) * m_));
    CK(mcpy(src_dev, src.data(), sizeof(sdl::GatherSrc) * m_, cudaMemcpyHostToDevice));
    team_src_host_.push_back(src);
    Slot gs;
    gs.cap = cfg_.k;
    gs.bytes = 16 + 8 * static_cast<size_t>((cfg_.k + 3) & ~3);
    gs.base = static_cast<unsigned char*>(arena_.alloc(gs.bytes));
    gs.cnt = reinterpret_cast<int32_t*>(gs.base);
    gs.idx = reinterpret_cast<int32_t*>(gs.base + 16);
    gs.val = reinterpret_cast<float*>(gs.base + 16 + 4 * static_cast<size_t>((cfg_.k + 3) & ~3));
    sdl::AssembleTask at{};
    at.m = m_;
    at.src = src_dev;
    at.out_idx = gs.idx;
    at.out_val = gs.val;
    at.out_cnt = gs.cnt;
    at.out_hash = hash_dev_ + t;
    asm_tasks_.push_back(at);
    asm_in_.push_back(team_blocks[static_cast<size_t>(t)]);
    for (int j = 0; j < m_; ++j)
      if (is_local(t * m_ + j))
        team_of_local_global_[static_cast<size_t>(t * m_ + j - first_)] =
            static_cast<int>(global_.size());
    global_.push_back(gs);
    global_team_.push_back(t);
    team_src_.push_back(src_dev);
  }
  (void)max_m;
  asm_dev_ = static_cast<sdl::AssembleTask*>(
      arena_.alloc(sizeof(sdl::AssembleTask) * std::max<size_t>(1, asm_tasks_.size())));
  CK(mcpy(asm_dev_, asm_tasks_.data(), sizeof(sdl::AssembleTask) * asm_tasks_.size(),
                cudaMemcpyHostToDevice));
  launches_ += 1;

  for (int li = 0; li < wloc_; ++li) {
    sdl::FinalizeTask ft{};
    ft.mode = cfg_.residual;
    ft.m = m_;
    ft.n = N;
    ft.carry = carry_[static_cast<size_t>(li)];
    ft.gblk = team_src_[static_cast<size_t>(team_of_local_global_[static_cast<size_t>(li)])];
    auto* sc_dev = static_cast<const sdl::SelScratch**>(
        arena_.alloc(sizeof(sdl::SelScratch*) * m_));
    CK(mcpy(sc_dev, div_scr_[static_cast<size_t>(li)].data(), sizeof(sdl::SelScratch*) * m_,
                  cudaMemcpyHostToDevice));
    ft.div_sc = sc_dev;
    std::vector<sdl::GatherSrc> div;
    std::vector<int32_t> xoff;
    std::vector<sdl::XiList> xl;
    for (int b = 0; b < m_; ++b) {
      const Slot& s = local_slot(div_uid_[static_cast<size_t>(li)][static_cast<size_t>(b)]);
      div.push_back({s.idx, s.val, s.cnt});
      xoff.push_back(static_cast<int32_t>(xl.size()));
      for (const auto& x : xi_[static_cast<size_t>(li)][static_cast<size_t>(b)]) xl.push_back(x);
    }
    xoff.push_back(static_cast<int32_t>(xl.size()));
    auto* div_dev = static_cast<sdl::GatherSrc*>(arena_.alloc(sizeof(sdl::GatherSrc) * m_));
    CK(mcpy(div_dev, div.data(), sizeof(sdl::GatherSrc) * m_, cudaMemcpyHostToDevice));
    auto* xoff_dev = static_cast<int32_t*>(arena_.alloc(sizeof(int32_t) * xoff.size()));
    CK(mcpy(xoff_dev, xoff.data(), sizeof(int32_t) * xoff.size(), cudaMemcpyHostToDevice));
    auto* xl_dev = static_cast<sdl::XiList*>(
        arena_.alloc(sizeof(sdl::XiList) * std::max<size_t>(1, xl.size())));
    if (!xl.empty())
      CK(mcpy(xl_dev, xl.data(), sizeof(sdl::XiList) * xl.size(), cudaMemcpyHostToDevice));
    ft.div = div_dev;
    ft.xi_off = xoff_dev;
    ft.xi = xl_dev;
    fin_tasks_.push_back(ft);
  }
  // deferred finalize records (gres, <= 2 discard lists per block; the
  // split dividing pass launches per group and keeps the plain finalize)
  {
    bool ok = cfg_.residual == SPARDL_RES_GRES && div_split_ <= 1 &&
              static_cast<int>(div_tasks_.size()) == wloc_ * m_;
    for (int li = 0; li < wloc_ && ok; ++li)
      for (int b = 0; b < m_; ++b)
        ok &= xi_[static_cast<size_t>(li)][static_cast<size_t>(b)].size() <= 2;
    // SPARDL_FIN_DEFER: 1 = records applied by the next candidate pass,
    // 2 = records applied right away by k_fin_apply (no carry access in the
    // join), 0 (default) = k_finalize (join and carry read-modify-write)
    const char* fe = std::getenv("SPARDL_FIN_DEFER");
    fin_mode_ = fe ? std::atoi(fe) : 0;
    if (fin_mode_ <= 0) ok = false;
    fin_defer_ok_ = ok;
    fin_apply_ = static_cast<int32_t*>(arena_.alloc(sizeof(int32_t)));
    if (ok) {
      for (int li = 0; li < wloc_; ++li)
        for (int b = 0; b < m_; ++b) {
          sdl::DivTask& dt = div_tasks_[static_cast<size_t>(li * m_ + b)];
          const sdl::GatherSrc& gs_ = team_src_host_[static_cast<size_t>(
              team_of_local_global_[static_cast<size_t>(li)])][static_cast<size_t>(b)];
          sdl::FinRecTask r{};
          r.g_idx = gs_.idx;
          r.g_cnt = gs_.cnt;
          const auto& xl = xi_[static_cast<size_t>(li)][static_cast<size_t>(b)];
          r.nxl = static_cast<int32_t>(xl.size());
          for (size_t q = 0; q < xl.size(); ++q) r.xl[q] = xl[q];
          r.nchunks = dt.nchunks;
          r.origin = static_cast<int64_t>(dt.lo) & ~int64_t(3);
          r.rec_idx = static_cast<int32_t*>(arena_.alloc(sizeof(int32_t) * Lcap_));
          r.rec_v1 = static_cast<float*>(arena_.alloc(sizeof(float) * Lcap_));
          r.rec_v2 = static_cast<float*>(arena_.alloc(sizeof(float) * Lcap_));
          r.chunk_off = static_cast<int32_t*>(arena_.alloc(sizeof(int32_t) * (dt.nchunks + 1)));
          r.rec_n = static_cast<int32_t*>(arena_.alloc(sizeof(int32_t)));
          r.carry = carry_[static_cast<size_t>(li)];
          r.div_sc = div_scr_[static_cast<size_t>(li)][static_cast<size_t>(b)];
          fin_rec_.push_back(r);
          dt.rec_idx = r.rec_idx;
          dt.rec_v1 = r.rec_v1;
          dt.rec_v2 = r.rec_v2;
          dt.chunk_off = r.chunk_off;
          dt.fin_apply = fin_apply_;
          dt.prev_sel = r.div_sc;
        }
      fin_rec_dev_ = static_cast<sdl::FinRecTask*>(
          arena_.alloc(sizeof(sdl::FinRecTask) * fin_rec_.size()));
      CK(mcpy(fin_rec_dev_, fin_rec_.data(), sizeof(sdl::FinRecTask) * fin_rec_.size(),
              cudaMemcpyHostToDevice));
      CK(mcpy(div_dev_, div_tasks_.data(), sizeof(sdl::DivTask) * div_tasks_.size(),
              cudaMemcpyHostToDevice));
    }
    fin_defer_ = ok;
  }
  fin_max_div_ = cfg_.residual == SPARDL_RES_LRES ? Lcap_ : 0;
  fin_dev_ = static_cast<sdl::FinalizeTask*>(
      arena_.alloc(sizeof(sdl::FinalizeTask) * fin_tasks_.size()));
  CK(mcpy(fin_dev_, fin_tasks_.data(), sizeof(sdl::FinalizeTask) * fin_tasks_.size(),
                cudaMemcpyHostToDevice));
  launches_ += fin_max_div_ > 0 ? 2 : 1;

  if (!ledger_adds_.empty()) {
    ledger_dev_ = static_cast<sdl::LedgerAdd*>(
        arena_.alloc(sizeof(sdl::LedgerAdd) * ledger_adds_.size()));
    CK(mcpy(ledger_dev_, ledger_adds_.data(), sizeof(sdl::LedgerAdd) * ledger_adds_.size(),
                  cudaMemcpyHostToDevice));
    launches_ += 1;
  }
  if (cfg_.sag == SPARDL_SAG_BSAG) {
    for (int li = 0; li < wloc_; ++li)
      ctl_tasks_.push_back({ctl_dev_ + li, ntot_ + li, budget_dev_ + li});
    ctl_tasks_dev_ =
        static_cast<sdl::CtlTask*>(arena_.alloc(sizeof(sdl::CtlTask) * ctl_tasks_.size()));
    CK(mcpy(ctl_tasks_dev_, ctl_tasks_.data(), sizeof(sdl::CtlTask) * ctl_tasks_.size(),
                  cudaMemcpyHostToDevice));
    launches_ += 1;
  }
}

// ---------------------------------------------------------------------------
// deferred finalize
void Engine::flush_finalize() {
  if (dry_ || !fin_defer_ || fin_rec_.empty()) return;
  CK(cudaSetDevice(device_));
  sdl::launch_fin_apply(fin_rec_dev_, static_cast<int>(fin_rec_.size()), Lcap_, fin_apply_,
                        stream_);
  CK(cudaMemsetAsync(fin_apply_, 0, sizeof(int32_t), stream_));
  CK(sdl::take_launch_error());
  CK(cudaStreamSynchronize(stream_));
}

void Engine::set_defer(bool on) {
  on = on && fin_defer_ok_;
  if (on == fin_defer_) return;
  flush_finalize();   // pending records applied before the mode changes
  fin_defer_ = on;
  drop_graph();
}

// ---------------------------------------------------------------------------
// sparse conservation audit
void Engine::set_audit(bool on) {
  audit_ = on;
  if (dry_) return;
  CK(cudaSetDevice(device_));
  sync();
  // the audit reads the finalized carry at the global positions: plain finalize
  set_defer(!on);
  const size_t k = static_cast<size_t>(std::max<int64_t>(1, cfg_.k));
  if (on && aud_comb_.empty()) {
    for (int li = 0; li < wloc_; ++li) {
      aud_comb_.push_back(static_cast<float*>(arena_.alloc(sizeof(float) * k)));
      aud_carry_.push_back(static_cast<float*>(arena_.alloc(sizeof(float) * k)));
    }
    if (world_ > 1)
      aud_gather_ = static_cast<float*>(
          arena_.alloc(sizeof(float) * k * 2 * static_cast<size_t>(wloc_) * (world_ + 1)));
  }
  for (int li = 0; li < wloc_; ++li) {
    fin_tasks_[static_cast<size_t>(li)].aud_comb = on ? aud_comb_[static_cast<size_t>(li)] : nullptr;
    fin_tasks_[static_cast<size_t>(li)].aud_carry = on ? aud_carry_[static_cast<size_t>(li)] : nullptr;
  }
  CK(mcpy(fin_dev_, fin_tasks_.data(), sizeof(sdl::FinalizeTask) * fin_tasks_.size(),
          cudaMemcpyHostToDevice));
}

// max over the global positions of |sum_w combined_w - (global + sum_w carry_w)|
// / max(1, |sum_w combined_w|), sums in double in worker order (collective)
double Engine::conservation_audit() {
  const size_t k = static_cast<size_t>(std::max<int64_t>(1, cfg_.k));
  const Slot& gs = global_[static_cast<size_t>(team_of_local_global_[0])];
  int32_t n = 0;
  CK(mcpy(&n, gs.cnt, sizeof(int32_t), cudaMemcpyDeviceToHost));
  std::vector<float> gval(static_cast<size_t>(n));
  if (n) CK(mcpy(gval.data(), gs.val, sizeof(float) * n, cudaMemcpyDeviceToHost));
  // all workers' (combined, carry) at the global positions, worker order
  std::vector<float> all(k * 2 * static_cast<size_t>(P_));
  if (world_ > 1) {
    float* send = aud_gather_;
    for (int li = 0; li < wloc_; ++li) {
      CK(cudaMemcpy(send + k * 2 * li, aud_comb_[static_cast<size_t>(li)], sizeof(float) * k,
                    cudaMemcpyDeviceToDevice));
      CK(cudaMemcpy(send + k * (2 * li + 1), aud_carry_[static_cast<size_t>(li)],
                    sizeof(float) * k, cudaMemcpyDeviceToDevice));
    }
    float* recv = send + k * 2 * wloc_;
    NK(ncclAllGather(send, recv, k * 2 * wloc_, ncclFloat, comm_, stream_));
    CK(cudaStreamSynchronize(stream_));
    CK(cudaMemcpy(all.data(), recv, sizeof(float) * all.size(), cudaMemcpyDeviceToHost));
  } else {
    for (int li = 0; li < wloc_; ++li) {
      CK(cudaMemcpy(all.data() + k * 2 * li, aud_comb_[static_cast<size_t>(li)],
                    sizeof(float) * k, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(all.data() + k * (2 * li + 1), aud_carry_[static_cast<size_t>(li)],
                    sizeof(float) * k, cudaMemcpyDeviceToHost));
    }
  }
  double worst = 0.0;
  for (int32_t p = 0; p < n; ++p) {
    double lhs = 0.0, rhs = 0.0;
    for (int w = 0; w < P_; ++w) lhs += all[k * 2 * w + static_cast<size_t>(p)];
    rhs += gval[static_cast<size_t>(p)];
    for (int w = 0; w < P_; ++w) rhs += all[k * (2 * w + 1) + static_cast<size_t>(p)];
    const double den = std::max(1.0, lhs < 0 ? -lhs : lhs);
    const double d = lhs - rhs;
    worst = std::max(worst, (d < 0 ? -d : d) / den);
  }
  return worst;
}

// ---------------------------------------------------------------------------
// peer-memory transport setup
void Engine::setup_peer() {
  if (world_ == 1) return;
  const char* env = std::getenv("SPARDL_TRANSPORT");
  if (env && std::strcmp(env, "nccl") == 0) return;
  // the plan numbers every rank's buffers identically: a plan-only replay
  // gives the region size each rank needs
  int max_slots = 0, nuid = 0;
  {
    Engine dry(cfg_, 0, world_, rank_, nullptr, nullptr, true);
    nuid = dry.next_uid_;
    max_slots = nuid;   // global buffer numbering
    // blocks delivered to other ranks are pushed by their producing select
    // into every consumer rank's copy (consumers then read local memory)
    const char* pe = std::getenv("SPARDL_PUSH");
    if (!(pe && pe[0] == '0')) {
      std::map<int, std::set<int>> dst;
      for (const auto& dl : dry.deliveries_) {
        const int o = rank_of(dry.uid_owner_[static_cast<size_t>(dl.first)]);
        if (dl.second != o) dst[dl.first].insert(dl.second);
      }
      for (const auto& kv : dst)
        if (kv.second.size() <= static_cast<size_t>(sdl::kMaxPush))
          push_dst_[kv.first] = std::vector<int>(kv.second.begin(), kv.second.end());
    }
  }
  auto align = [](size_t x) { return (x + 255) & ~static_cast<size_t>(255); };
  slot_stride_ = align(16 + 8 * static_cast<size_t>(Lcap_));
  flags_off_ = slot_stride_ * static_cast<size_t>(max_slots);
  done_off_ = flags_off_ + align(sizeof(long long) * static_cast<size_t>(nuid));
  const size_t bytes = done_off_ + align(sizeof(long long) * static_cast<size_t>(world_));
  CK(cudaMalloc(&sym_, bytes));
  CK(cudaMemset(sym_, 0, bytes));
  // what every rank learns about every other: its IPC handle, and -- for
  // ranks in this same process (spardl_mctx: one host thread, several
  // GPUs), where IPC handles cannot be opened -- its raw pointer and device
  struct PeerInfo {
    cudaIpcMemHandle_t h;
    long long pid;
    unsigned long long ptr;
    int32_t dev;
    int32_t pad;
  };
  PeerInfo mine{};
  int32_t ok = cudaIpcGetMemHandle(&mine.h, sym_) == cudaSuccess ? 1 : 0;
  cudaGetLastError();
  mine.pid = static_cast<long long>(getpid());
  mine.ptr = reinterpret_cast<unsigned long long>(sym_);
  mine.dev = device_;
  const size_t hb = sizeof(PeerInfo);
  unsigned char* dbuf = nullptr;
  CK(cudaMalloc(&dbuf, hb * static_cast<size_t>(world_ + 1) + 16));
  CK(cudaMemcpy(dbuf, &mine, hb, cudaMemcpyHostToDevice));
  NK(ncclAllGather(dbuf, dbuf + hb, hb, ncclChar, comm_, stream_));
  std::vector<PeerInfo> hs(static_cast<size_t>(world_));
  CK(cudaStreamSynchronize(stream_));
  CK(cudaMemcpy(hs.data(), dbuf + hb, hb * static_cast<size_t>(world_), cudaMemcpyDeviceToHost));
  peer_base_.assign(static_cast<size_t>(world_), nullptr);
  peer_ipc_.assign(static_cast<size_t>(world_), 0);
  peer_base_[static_cast<size_t>(rank_)] = sym_;
  for (int q = 0; q < world_ && ok; ++q) {
    if (q == rank_) continue;
    const PeerInfo& pi = hs[static_cast<size_t>(q)];
    if (pi.pid == mine.pid) {   // same process: direct peer access (UVA)
      int can = 0;
      if (cudaDeviceCanAccessPeer(&can, device_, pi.dev) != cudaSuccess || !can) {
        cudaGetLastError();
        ok = 0;
        continue;
      }
      const cudaError_t pe = cudaDeviceEnablePeerAccess(pi.dev, 0);
      if (pe != cudaSuccess && pe != cudaErrorPeerAccessAlreadyEnabled) ok = 0;
      cudaGetLastError();
      peer_base_[static_cast<size_t>(q)] = reinterpret_cast<unsigned char*>(pi.ptr);
      continue;
    }
    void* p = nullptr;
    if (cudaIpcOpenMemHandle(&p, pi.h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      ok = 0;
    } else {
      peer_base_[static_cast<size_t>(q)] = static_cast<unsigned char*>(p);
      peer_ipc_[static_cast<size_t>(q)] = 1;
    }
  }
  // every rank must agree, or all use NCCL
  int32_t* dok = reinterpret_cast<int32_t*>(dbuf + hb * static_cast<size_t>(world_ + 1));
  CK(cudaMemcpy(dok, &ok, sizeof(ok), cudaMemcpyHostToDevice));
  NK(ncclAllReduce(dok, dok, 1, ncclInt32, ncclMin, comm_, stream_));
  CK(cudaStreamSynchronize(stream_));
  CK(cudaMemcpy(&ok, dok, sizeof(ok), cudaMemcpyDeviceToHost));
  CK(cudaFree(dbuf));
  if (!ok) {
    for (int q = 0; q < world_; ++q)
      if (q != rank_ && peer_base_[static_cast<size_t>(q)] && peer_ipc_[static_cast<size_t>(q)])
        cudaIpcCloseMemHandle(peer_base_[static_cast<size_t>(q)]);
    peer_base_.clear();
    cudaFree(sym_);
    sym_ = nullptr;
    return;
  }
  peer_ = true;
}

// Readiness flags: the owner of a block publishes it to every rank it is
// delivered to right after the stage that produces it; a consumer waits at the
// round of the schedule that delivers it.
void Engine::plan_peer() {
  if (!peer_) return;
  auto flag_at = [&](int rank, int uid) {
    return reinterpret_cast<long long*>(peer_base_[static_cast<size_t>(rank)] + flags_off_) + uid;
  };
  auto upload = [&](const auto& v) {
    using T = typename std::decay_t<decltype(v)>::value_type;
    T* d = static_cast<T*>(arena_.alloc(sizeof(T) * std::max<size_t>(1, v.size())));
    if (!v.empty()) CK(cudaMemcpy(d, v.data(), sizeof(T) * v.size(), cudaMemcpyHostToDevice));
    return d;
  };
  // every block delivered to another rank must come out of a planned stage
  for (const auto& dl : deliveries_) {
    const int uid = dl.first;
    if (rank_of(uid_owner_[static_cast<size_t>(uid)]) != rank_ || dl.second == rank_) continue;
    bool found = div_stage_.produced.count(uid) != 0;
    for (size_t i = 0; i < steps_.size() && !found; ++i) found = steps_[i].stage.produced.count(uid) != 0;
    if (!found) sdlh::fail(SPARDL_E_ERROR, "internal: delivered block has no producing stage");
  }
  // per-task synchronisation: a select publishes its block as soon as it is
  // complete; a merge, a single-block select and an assembly wait for their
  // own remote inputs (no stage-wide publish / wait kernels)
  std::map<int, std::set<int>> dsts;   // uid -> ranks it is delivered to
  for (const auto& dl : deliveries_)
    if (dl.second != rank_ && rank_of(uid_owner_[static_cast<size_t>(dl.first)]) == rank_)
      dsts[dl.first].insert(dl.second);
  auto pubs_of = [&](int uid) {
    std::vector<long long*> v;
    auto it = dsts.find(uid);
    if (it != dsts.end())
      for (int d : it->second) v.push_back(flag_at(d, uid));
    return v;
  };
  auto waits_of = [&](const std::vector<int>& uids) {
    std::vector<const long long*> v;
    for (int u : uids)
      if (u >= 0 && rank_of(uid_owner_[static_cast<size_t>(u)]) != rank_) v.push_back(flag_at(rank_, u));
    return v;
  };
  auto sync_of = [&](const std::vector<const long long*>& w, const std::vector<long long*>& p) {
    sdl::PeerSync ps{};
    ps.wait = w.empty() ? nullptr : upload(w);
    ps.nwait = static_cast<int32_t>(w.size());
    ps.pub = p.empty() ? nullptr : upload(p);
    ps.npub = static_cast<int32_t>(p.size());
    ps.epoch = epoch_;
    ps.err = peer_err_;
    ps.timeout_ns = timeout_ns_;
    return ps;
  };
  auto wire_stage = [&](Stage& st) {
    for (size_t j = 0; j < st.merges.size(); ++j) st.merges[j].ps = sync_of(waits_of(st.merge_in[j]), {});
    for (size_t i = 0; i < st.sels.size(); ++i) {
      sdl::SelTask& t = st.sels[i];
      std::vector<int> in;
      if (st.sel_in[i] >= 0) in.push_back(st.sel_in[i]);
      if (st.fused && t.merge_slot) in = st.merge_in[static_cast<size_t>(t.merge_slot - 1)];
      t.ps = sync_of(waits_of(in), pubs_of(st.sel_uid[i]));
    }
    if (!st.merges.empty())
      CK(cudaMemcpy(st.merges_dev, st.merges.data(), sizeof(sdl::MergeTask) * st.merges.size(),
                    cudaMemcpyHostToDevice));
    if (!st.sels.empty())
      CK(cudaMemcpy(st.sels_dev, st.sels.data(), sizeof(sdl::SelTask) * st.sels.size(),
                    cudaMemcpyHostToDevice));
  };
  wire_stage(div_stage_);
  for (Step& stp : steps_) wire_stage(stp.stage);
  for (size_t q = 0; q < asm_tasks_.size(); ++q) asm_tasks_[q].ps = sync_of(waits_of(asm_in_[q]), {});
  // the residual finalize (or its records) reads the global gradient's blocks
  for (int li = 0; li < wloc_; ++li) {
    const size_t q = static_cast<size_t>(team_of_local_global_[static_cast<size_t>(li)]);
    fin_tasks_[static_cast<size_t>(li)].ps = sync_of(waits_of(asm_in_[q]), {});
  }
  if (!fin_tasks_.empty())
    CK(cudaMemcpy(fin_dev_, fin_tasks_.data(), sizeof(sdl::FinalizeTask) * fin_tasks_.size(),
                  cudaMemcpyHostToDevice));
  for (size_t i = 0; i < fin_rec_.size(); ++i) {
    const size_t li = i / static_cast<size_t>(m_), b = i % static_cast<size_t>(m_);
    const size_t q = static_cast<size_t>(team_of_local_global_[li]);
    fin_rec_[i].ps = sync_of(waits_of({asm_in_[q][b]}), {});
  }
  if (!fin_rec_.empty())
    CK(cudaMemcpy(fin_rec_dev_, fin_rec_.data(), sizeof(sdl::FinRecTask) * fin_rec_.size(),
                  cudaMemcpyHostToDevice));
  if (!asm_tasks_.empty())
    CK(cudaMemcpy(asm_dev_, asm_tasks_.data(), sizeof(sdl::AssembleTask) * asm_tasks_.size(),
                  cudaMemcpyHostToDevice));

  std::vector<const long long*> begin;
  std::vector<long long*> done;
  for (int q = 0; q < world_; ++q) {
    if (q == rank_) continue;
    begin.push_back(reinterpret_cast<const long long*>(sym_ + done_off_) + q);
    done.push_back(reinterpret_cast<long long*>(peer_base_[static_cast<size_t>(q)] + done_off_) + rank_);
  }
  begin_dev_ = upload(begin);
  done_dev_ = upload(done);
  npeer_ = static_cast<int>(begin.size());
}

// ---------------------------------------------------------------------------
// execution
int Engine::exec_stage(const Stage& st, bool dividing, cudaEvent_t after_merge) {
  int n = 0;
  if (!st.merges.empty() && !st.fused)
    n += sdl::launch_merge(st.merges_dev, static_cast<int>(st.merges.size()), st.max_parts,
                           st.max_rT, st.max_r, stream_);
  if (after_merge) CK(cudaEventRecord(after_merge, stream_));
  // wide path first (with SPARDL_WSEL_FUSE=1 the dividing histogram and
  // decision come from the candidate pass); the cluster select then runs
  // only the tasks handed back
  if (st.wide && st.coop)
    n += sdl::launch_wselect_coop(st.sels_dev, static_cast<int>(st.sels.size()), st.w_max_nseg,
                                  stream_);
  else if (st.wide)
    n += sdl::launch_wselect(st.sels_dev, static_cast<int>(st.sels.size()), st.w_max_tiles,
                             !(dividing && wsel_fuse_), stream_);
  if (!st.sels.empty())
    n += sdl::launch_select(st.sels_dev, static_cast<int>(st.sels.size()), st.max_nseg, stream_,
                            st.fused ? st.cl : 0, st.fused ? st.win_cap : 0);
  return n;
}

void Engine::exec_round(const std::vector<Xfer>& xs) {
  if (world_ == 1 || peer_) return;
  bool any = false;
  for (const Xfer& x : xs) any |= x.src_rank != x.dst_rank;
  if (!any) return;
  NK(ncclGroupStart());
  for (const Xfer& x : xs) {
    if (x.src_rank == x.dst_rank) continue;
    Slot& s = local_slot(x.uid);
    if (x.src_rank == rank_)
      NK(ncclSend(s.base, s.bytes, ncclChar, x.dst_rank, comm_, stream_));
    else
      NK(ncclRecv(s.base, s.bytes, ncclChar, x.src_rank, comm_, stream_));
  }
  NK(ncclGroupEnd());
}

// One iteration.  When `ev` is given (profiling, never inside a graph), an
// event is recorded at each phase boundary:
//   ev[0] | sample+pre-threshold | ev[1] | candidate pass | ev[2] | dividing
//   select | ev[3] | SRS + SAG stages and rounds | ev[4] | final gather,
//   assemble, finalize, ledger | ev[5]
void Engine::enqueue_iteration(cudaEvent_t* ev) {
  int n = 0;
  auto mark = [&](int i) {
    if (ev) CK(cudaEventRecord(ev[i], stream_));
  };
  const int32_t* abort = peer_ ? peer_err_ : nullptr;   // peer timeout: state untouched
  CK(cudaMemsetAsync(ledger_phase_, 0, sizeof(int64_t) * 3 * wloc_, stream_));
  CK(cudaMemsetAsync(hash_dev_, 0, sizeof(int64_t) * d_, stream_));
  // peers may read our block buffers until they finish the previous iteration
  if (peer_) n += sdl::launch_begin(epoch_, begin_dev_, npeer_, peer_err_, timeout_ns_, stream_);
  mark(0);
  n += sdl::launch_divide(div_dev_, static_cast<int>(div_tasks_.size()), div_max_chunks_,
                          div_sample_every_, 1, stream_, 1);
  mark(1);
  // Tasks are worker-major (m_ blocks per local worker).  With a split the
  // candidate passes of the worker groups run back to back on stream_ and
  // each group's select runs on the high-priority stream as soon as its own
  // pass is done, beside the next group's pass.
  const int ndt = static_cast<int>(div_tasks_.size());
  const int G = std::min(div_split_, wloc_);
  if (G <= 1 || div_stage_.sels.size() != div_tasks_.size()) {
    n += sdl::launch_divide(div_dev_, ndt, div_max_chunks_, div_sample_every_,
                            fin_defer_ && fin_mode_ == 1 ? 2 : 1, stream_, 2);
    mark(2);
    n += exec_stage(div_stage_, true);   // (peer transport: each select publishes its block)
  } else {
    for (int g = 0; g < G; ++g) {
      const int t0 = (g * wloc_ / G) * m_, t1 = ((g + 1) * wloc_ / G) * m_;
      n += sdl::launch_divide(div_dev_ + t0, t1 - t0, div_max_chunks_, div_sample_every_, 1,
                              stream_, 2);
      const bool last = g + 1 == G;
      cudaStream_t ss = last ? stream_ : hi_;
      if (!last) {
        CK(cudaEventRecord(ev_div_[0], stream_));
        CK(cudaStreamWaitEvent(hi_, ev_div_[0], 0));
      } else {
        mark(2);
      }
      n += sdl::launch_select(div_stage_.sels_dev + t0, t1 - t0, div_stage_.max_nseg, ss);
    }
    CK(cudaEventRecord(ev_div_[1], hi_));
    CK(cudaStreamWaitEvent(stream_, ev_div_[1], 0));
  }
  mark(3);
  // optional per-step events (profiling diagnostics, SPARDL_STEP_EVENTS=1)
  const bool sev = ev && !step_ev_.empty();
  auto step_mark = [&](size_t i, int what) {
    if (sev) CK(cudaEventRecord(step_ev_[4 * i + what], stream_));
  };
  for (size_t i = 0; i < steps_.size(); ++i) {
    const Step& s = steps_[i];
    n += exec_stage(s.stage, false, sev ? step_ev_[4 * i] : nullptr);
    step_mark(i, 1);
    if (s.controller_after)
      n += sdl::launch_controller(ctl_tasks_dev_, static_cast<int>(ctl_tasks_.size()), 1, abort,
                                  stream_);
    step_mark(i, 2);
    if (i + 1 == steps_.size()) mark(4);
    exec_round(s.xfers);   // NCCL transport only: peers wait per task
    step_mark(i, 3);
  }
  if (steps_.empty()) mark(4);
  // the assembled global gradient and the ledger only read the gathered
  // blocks: they run on a side stream beside the residual finalize
  CK(cudaEventRecord(ev_fork_, stream_));
  CK(cudaStreamWaitEvent(side_, ev_fork_, 0));
  n += sdl::launch_assemble(asm_dev_, static_cast<int>(asm_tasks_.size()), m_, cfg_.k, side_);
  n += sdl::launch_ledger(ledger_dev_, static_cast<int>(ledger_adds_.size()), abort, side_);
  if (fin_defer_) {   // records for the next candidate pass (no carry access here)
    n += sdl::launch_fin_records(fin_rec_dev_, static_cast<int>(fin_rec_.size()), Lcap_,
                                 fin_apply_, stream_);
    if (fin_mode_ == 2) {   // ... or applied at once
      n += sdl::launch_fin_apply(fin_rec_dev_, static_cast<int>(fin_rec_.size()), Lcap_,
                                 fin_apply_, stream_);
      CK(cudaMemsetAsync(fin_apply_, 0, sizeof(int32_t), stream_));
    }
  } else
    n += sdl::launch_finalize(fin_dev_, static_cast<int>(fin_tasks_.size()), Lcap_, m_,
                              static_cast<int>(fin_max_div_), abort, stream_);
  CK(cudaEventRecord(ev_join_, side_));
  CK(cudaStreamWaitEvent(stream_, ev_join_, 0));
  // last remote read of the iteration done: peers may overwrite their buffers
  if (peer_) n += sdl::launch_publish(done_dev_, npeer_, epoch_, stream_);
  mark(5);
  CK(sdl::take_launch_error());
  CK(cudaGetLastError());
  launches_ = n;
}

void Engine::profile(const float* const* grads, int iters, double* phase_ms) {
  // the pointer table only: every profiled iteration is a fresh one on these
  // gradients (no extra warm iteration re-adding the same gradient)
  set_grads(grads);
  const char* se = std::getenv("SPARDL_STEP_EVENTS");
  if (se && se[0] == '1' && step_ev_.empty()) {
    step_ev_.resize(4 * steps_.size());
    for (auto& e : step_ev_) CK(cudaEventCreate(&e));
  }
  std::vector<double> step_acc(4 * steps_.size(), 0.0);
  cudaEvent_t ev[6];
  for (auto& e : ev) CK(cudaEventCreate(&e));
  double acc[5] = {0, 0, 0, 0, 0};
  for (int it = 0; it < iters; ++it) {
    for (int w = 0; w < P_; ++w)
      for (int p = 0; p < 3; ++p)
        rounds_[static_cast<size_t>(w)] +=
            phase_rounds_[static_cast<size_t>(w)][static_cast<size_t>(p)];
    enqueue_iteration(ev);
    CK(cudaEventSynchronize(ev[5]));
    for (int p = 0; p < 5; ++p) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, ev[p], ev[p + 1]));
      acc[p] += ms;
    }
    for (size_t q = 0; q < step_ev_.size(); ++q) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, q == 0 ? ev[3] : step_ev_[q - 1], step_ev_[q]));
      step_acc[q] += ms;
    }
  }
  if (!step_ev_.empty()) {   // stage / publish / wait of every step, us
    std::string line =
        "rank " + std::to_string(rank_) + " steps (merge, select, controller, round us):";
    char buf[48];
    for (size_t q = 0; q < step_acc.size(); ++q) {
      std::snprintf(buf, sizeof(buf), "%s%.1f", q % 4 == 0 ? " | " : " ",
                    1e3 * step_acc[q] / std::max(iters, 1));
      line += buf;
    }
    std::fprintf(stderr, "%s\n", line.c_str());   // one write per rank
  }
  for (auto& e : ev) cudaEventDestroy(e);
  for (int p = 0; p < 5; ++p) phase_ms[p] = acc[p] / std::max(iters, 1);
}

void Engine::set_grads(const float* const* grads) {
  CK(cudaSetDevice(device_));
  if (poisoned_)
    sdlh::fail(SPARDL_E_STATE, "peer transport: an earlier iteration timed out waiting for a "
                               "peer; the residual state is void until reset_state()");
  bool changed = false;
  for (int i = 0; i < wloc_; ++i) {
    if (!grads[i]) sdlh::fail(SPARDL_E_ARG, "null gradient pointer");
    if (reinterpret_cast<uintptr_t>(grads[i]) % 16 != 0)
      sdlh::fail(SPARDL_E_ARG, "gradient pointers must be 16-byte aligned");
    changed |= gtab_cur_[static_cast<size_t>(i)] != grads[i];
  }
  if (changed) {
    // the graph reads the pointer table from device memory: a new table is
    // uploaded in stream order from a ring of pinned host slots (no host
    // synchronisation; a slot is reused only after its upload has run)
    float const** slot = gtab_host_ + static_cast<size_t>(tab_next_) * wloc_;
    if (tab_used_[tab_next_]) CK(cudaEventSynchronize(tab_ev_[tab_next_]));
    for (int i = 0; i < wloc_; ++i) {
      slot[i] = grads[i];
      gtab_cur_[static_cast<size_t>(i)] = grads[i];
    }
    CK(cudaMemcpyAsync(gtab_dev_, slot, sizeof(float*) * wloc_, cudaMemcpyHostToDevice, stream_));
    CK(cudaEventRecord(tab_ev_[tab_next_], stream_));
    tab_used_[tab_next_] = true;
    tab_next_ = (tab_next_ + 1) % kTabRing;
  }
}

void Engine::run(const float* const* grads) {
  set_grads(grads);
  for (int w = 0; w < P_; ++w)
    for (int p = 0; p < 3; ++p)
      rounds_[static_cast<size_t>(w)] += phase_rounds_[static_cast<size_t>(w)][static_cast<size_t>(p)];
  if (use_graph_) {
    if (!graph_) {
      cudaGraph_t g = nullptr;
      CK(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
      try {
        enqueue_iteration();
      } catch (...) {
        cudaStreamEndCapture(stream_, &g);
        if (g) cudaGraphDestroy(g);
        throw;
      }
      CK(cudaStreamEndCapture(stream_, &g));
      CK(cudaGraphInstantiate(&graph_, g, cudaGraphInstantiateFlagUseNodePriority));
      cudaGraphDestroy(g);
    }
    CK(cudaGraphLaunch(graph_, stream_));
  } else {
    enqueue_iteration();
  }
  ran_ = true;
}

void Engine::sync() {
  CK(cudaSetDevice(device_));
  CK(cudaStreamSynchronize(stream_));
  int32_t err = 0;
  if (peer_) {
    CK(cudaMemcpy(&err, peer_err_, sizeof(err), cudaMemcpyDeviceToHost));
    if (err) {
      poisoned_ = true;   // carry / controller / ledger of that iteration are void
      sdlh::fail(SPARDL_E_CUDA, "peer transport: a peer did not arrive within the timeout (" +
                                    std::to_string(timeout_ns_ / 1000000) + " ms)");
    }
  }
  CK(mcpy(&err, err_dev_, sizeof(err), cudaMemcpyDeviceToHost));
  if (err) {
    CK(cudaMemset(err_dev_, 0, sizeof(int32_t)));
    sdlh::fail(SPARDL_E_ARG, "gradient contains NaN (selection order undefined)");
  }
}

void Engine::reset_state() {
  CK(cudaSetDevice(device_));
  CK(cudaStreamSynchronize(stream_));
  if (peer_) CK(cudaMemset(peer_err_, 0, sizeof(int32_t)));
  poisoned_ = false;
  for (int i = 0; i < wloc_; ++i) {
    CK(cudaMemset(carry_[static_cast<size_t>(i)], 0, sizeof(float) * cfg_.dimension));
    CK(cudaMemset(ledger_total_[static_cast<size_t>(i)], 0, sizeof(int64_t)));
  }
  std::fill(rounds_.begin(), rounds_.end(), 0);
  CK(cudaMemset(fallbacks_dev_, 0, sizeof(unsigned long long)));
  if (fin_apply_) CK(cudaMemset(fin_apply_, 0, sizeof(int32_t)));
  CK(cudaMemset(wide_back_dev_, 0, sizeof(unsigned long long)));
  CK(cudaMemset(retries_dev_, 0, sizeof(unsigned long long)));
  reset_wide(div_stage_);
  for (const Step& stp : steps_) reset_wide(stp.stage);
  for (const auto& dt : div_tasks_) CK(cudaMemset(dt.hist, 0, sizeof(sdl::DivHistory)));
  if (cfg_.sag == SPARDL_SAG_BSAG) {
    std::vector<sdl::HCtl> c(static_cast<size_t>(wloc_));
    std::vector<int64_t> b(static_cast<size_t>(wloc_));
    for (int i = 0; i < wloc_; ++i) {
      spardl_hctrl h;
      sdlh::hctrl_init(&h, cfg_.workers, cfg_.k, cfg_.teams);
      c[static_cast<size_t>(i)] = {h.lower, h.upper, h.target, h.h, h.step, h.flag, 0};
      b[static_cast<size_t>(i)] = sdlh::hctrl_budget(&h);
    }
    CK(mcpy(ctl_dev_, c.data(), sizeof(sdl::HCtl) * wloc_, cudaMemcpyHostToDevice));
    CK(mcpy(budget_dev_, b.data(), sizeof(int64_t) * wloc_, cudaMemcpyHostToDevice));
  }
  ran_ = false;
}

// Gathers one int64 per local worker from every rank into out[P].
static void allgather_i64(ncclComm_t comm, cudaStream_t st, int world, const int64_t* local_dev,
                          int wloc, int64_t* out_host, int64_t* scratch_dev) {
  if (world == 1) {
    if (cudaMemcpy(out_host, local_dev, sizeof(int64_t) * wloc, cudaMemcpyDeviceToHost) !=
        cudaSuccess)
      sdlh::fail(SPARDL_E_CUDA, "readback failed");
    return;
  }
  NK(ncclAllGather(local_dev, scratch_dev, static_cast<size_t>(wloc), ncclInt64, comm, st));
  if (cudaStreamSynchronize(st) != cudaSuccess) sdlh::fail(SPARDL_E_CUDA, "allgather sync failed");
  if (cudaMemcpy(out_host, scratch_dev, sizeof(int64_t) * wloc * world, cudaMemcpyDeviceToHost) !=
      cudaSuccess)
    sdlh::fail(SPARDL_E_CUDA, "readback failed");
}

void Engine::ledger(int64_t* rounds, int64_t* scalars) {
  sync();
  std::vector<int64_t> loc(static_cast<size_t>(wloc_));
  for (int i = 0; i < wloc_; ++i)
    CK(mcpy(&loc[static_cast<size_t>(i)], ledger_total_[static_cast<size_t>(i)],
                  sizeof(int64_t), cudaMemcpyDeviceToHost));
  int64_t* tmp = rb_dev_;
  CK(mcpy(tmp, loc.data(), sizeof(int64_t) * wloc_, cudaMemcpyHostToDevice));
  allgather_i64(comm_, stream_, world_, tmp, wloc_, scalars, tmp + wloc_);
  for (int w = 0; w < P_; ++w) rounds[w] = rounds_[static_cast<size_t>(w)];
}

spardl_run_info Engine::run_info() {
  sync();
  spardl_run_info ri{};
  std::vector<int64_t> rounds(static_cast<size_t>(P_)), scalars(static_cast<size_t>(P_));
  ledger(rounds.data(), scalars.data());
  for (int w = 0; w < P_; ++w) {
    ri.max_rounds = std::max(ri.max_rounds, rounds[static_cast<size_t>(w)]);
    ri.max_scalars = std::max(ri.max_scalars, scalars[static_cast<size_t>(w)]);
  }
  // per-phase deltas: max over workers (fabric.hpp:124-134)
  std::vector<int64_t> ph(static_cast<size_t>(3 * P_));
  {
    int64_t* tmp = rb_dev_;
    // gather phase p of all workers
    for (int p = 0; p < 3; ++p) {
      std::vector<int64_t> loc(static_cast<size_t>(wloc_));
      std::vector<int64_t> all(static_cast<size_t>(P_));
      std::vector<int64_t> buf(static_cast<size_t>(3 * wloc_));
      CK(mcpy(buf.data(), ledger_phase_, sizeof(int64_t) * 3 * wloc_, cudaMemcpyDeviceToHost));
      for (int i = 0; i < wloc_; ++i) loc[static_cast<size_t>(i)] = buf[static_cast<size_t>(3 * i + p)];
      CK(mcpy(tmp, loc.data(), sizeof(int64_t) * wloc_, cudaMemcpyHostToDevice));
      allgather_i64(comm_, stream_, world_, tmp, wloc_, all.data(), tmp + wloc_);
      for (int w = 0; w < P_; ++w) ph[static_cast<size_t>(3 * w + p)] = all[static_cast<size_t>(w)];
    }
  }
  for (int w = 0; w < P_; ++w) {
    ri.srs_scalars = std::max(ri.srs_scalars, ph[static_cast<size_t>(3 * w)]);
    ri.sag_scalars = std::max(ri.sag_scalars, ph[static_cast<size_t>(3 * w + 1)]);
    ri.gather_scalars = std::max(ri.gather_scalars, ph[static_cast<size_t>(3 * w + 2)]);
    ri.srs_rounds = std::max<int64_t>(ri.srs_rounds, phase_rounds_[static_cast<size_t>(w)][0]);
    ri.sag_rounds = std::max<int64_t>(ri.sag_rounds, phase_rounds_[static_cast<size_t>(w)][1]);
    ri.gather_rounds = std::max<int64_t>(ri.gather_rounds, phase_rounds_[static_cast<size_t>(w)][2]);
  }
  sdlh::expected_cost_sag(cfg_.workers, cfg_.k, cfg_.teams, cfg_.sag, &ri.pred_rounds,
                          &ri.pred_low, &ri.pred_high);
  // consistency: every assembled global gradient hashes identically
  {
    std::vector<int64_t> h(static_cast<size_t>(d_), 0);
    CK(mcpy(h.data(), hash_dev_, sizeof(int64_t) * d_, cudaMemcpyDeviceToHost));
    if (world_ > 1) {
      int64_t* tmp = rb_dev_;
      CK(mcpy(tmp, h.data(), sizeof(int64_t) * d_, cudaMemcpyHostToDevice));
      NK(ncclAllGather(tmp, tmp + d_, static_cast<size_t>(d_), ncclInt64, comm_, stream_));
      CK(cudaStreamSynchronize(stream_));
      h.resize(static_cast<size_t>(d_ * world_));
      CK(mcpy(h.data(), tmp + d_, sizeof(int64_t) * d_ * world_, cudaMemcpyDeviceToHost));
    }
    bool ok = true;
    int64_t ref = 0;
    bool have = false;
    std::vector<int32_t> nnz(global_.size());
    for (size_t q = 0; q < global_.size(); ++q)
      CK(mcpy(&nnz[q], global_[q].cnt, sizeof(int32_t), cudaMemcpyDeviceToHost));
    for (int64_t v : h) {
      if (v == 0) continue;   // team not hosted there (an empty gradient hashes to 0 too)
      if (!have) {
        ref = v;
        have = true;
      } else if (v != ref) {
        ok = false;
      }
    }
    ri.consistent = ok ? 1 : 0;
    ri.global_nnz = global_.empty() ? 0 : nnz[0];
  }
  ri.conservation_applicable = cfg_.residual == SPARDL_RES_GRES ? 1 : 0;
  ri.conservation_error = -1.0;
  if (audit_ && !aud_comb_.empty() && cfg_.residual != SPARDL_RES_LRES)
    ri.conservation_error = conservation_audit();
  ri.n_union = cfg_.sag == SPARDL_SAG_BSAG ? m_ : 0;
  return ri;
}

void Engine::div_diag(int task, int64_t* out) {
  sync();
  const sdl::DivTask& dt = div_tasks_.at(static_cast<size_t>(task));
  int32_t bad = 0, cnt = 0, mode = 0;
  int64_t tot = 0;
  uint32_t pre = 0;
  CK(mcpy(&bad, dt.cand_bad, sizeof(bad), cudaMemcpyDeviceToHost));
  cnt = dt.max_tiles;
  CK(mcpy(&tot, dt.cand_total, sizeof(tot), cudaMemcpyDeviceToHost));
  CK(mcpy(&pre, dt.pre_key, sizeof(pre), cudaMemcpyDeviceToHost));
  const int li = task / m_, b = task % m_;
  CK(mcpy(&mode, &div_scr_[static_cast<size_t>(li)][static_cast<size_t>(b)]->mode,
                sizeof(mode), cudaMemcpyDeviceToHost));
  out[0] = mode;
  out[1] = bad;
  out[2] = tot;
  out[3] = cnt;
  out[4] = pre;
  out[5] = dt.cap;
  sdl::DivHistory h{};
  CK(mcpy(&h, dt.hist, sizeof(h), cudaMemcpyDeviceToHost));
  uint32_t T = 0;
  CK(mcpy(&T, &div_scr_[static_cast<size_t>(li)][static_cast<size_t>(b)]->prefix, sizeof(T),
          cudaMemcpyDeviceToHost));
  out[6] = T;
  out[7] = h.valid ? static_cast<int64_t>(h.next_pre) : -1;
  out[8] = h.delta;
}

void Engine::select_timestamps(int step, int task, int64_t* out12) {
  sync();
  const Stage& st = step < 0 ? div_stage_ : steps_.at(static_cast<size_t>(step)).stage;
  const sdl::SelScratch* sc = st.sels.at(static_cast<size_t>(task)).scr;
  CK(mcpy(out12, sc->tstamp, sizeof(long long) * 116, cudaMemcpyDeviceToHost));
}

int64_t Engine::wide_handed_back() {
  sync();
  unsigned long long n = 0;
  if (wide_back_dev_) CK(mcpy(&n, wide_back_dev_, sizeof(n), cudaMemcpyDeviceToHost));
  return static_cast<int64_t>(n);
}

int64_t Engine::candidate_retries() {
  sync();
  unsigned long long n = 0;
  CK(mcpy(&n, retries_dev_, sizeof(n), cudaMemcpyDeviceToHost));
  return static_cast<int64_t>(n);
}

int64_t Engine::dense_fallbacks_total() {
  sync();
  unsigned long long n = 0;
  CK(mcpy(&n, fallbacks_dev_, sizeof(n), cudaMemcpyDeviceToHost));
  return static_cast<int64_t>(n);
}

int64_t Engine::dense_fallbacks() {
  sync();
  int64_t n = 0;
  for (const auto& row : div_scr_)
    for (const sdl::SelScratch* sc : row) {
      int32_t mode = 0;
      CK(mcpy(&mode, &sc->mode, sizeof(mode), cudaMemcpyDeviceToHost));
      n += mode == 1;
    }
  return n;
}

void Engine::union_sizes(int64_t* out) {
  if (cfg_.sag != SPARDL_SAG_BSAG) return;
  sync();
  std::vector<int64_t> all(static_cast<size_t>(P_));
  int64_t* tmp = rb_dev_;
  CK(mcpy(tmp, ntot_, sizeof(int64_t) * wloc_, cudaMemcpyDeviceToDevice));
  allgather_i64(comm_, stream_, world_, tmp, wloc_, all.data(), tmp + wloc_);
  for (int g = 0; g < m_; ++g) out[g] = all[static_cast<size_t>(g)];   // team 0 member g
}

void Engine::controller(int local, spardl_hctrl* out) {
  if (cfg_.sag != SPARDL_SAG_BSAG) sdlh::fail(SPARDL_E_CONFIG, "no controller: sag != bsag");
  sync();
  sdl::HCtl c;
  CK(mcpy(&c, ctl_dev_ + local, sizeof(c), cudaMemcpyDeviceToHost));
  *out = {c.lower, c.upper, c.target, c.h, c.step, c.flag, 0};
}

void Engine::set_controller(int local, const spardl_hctrl& h) {
  if (cfg_.sag != SPARDL_SAG_BSAG) sdlh::fail(SPARDL_E_CONFIG, "no controller: sag != bsag");
  if (local < 0 || local >= wloc_) sdlh::fail(SPARDL_E_ARG, "local worker out of range");
  sync();
  const sdl::HCtl c{h.lower, h.upper, h.target, h.h, h.step, h.flag, 0};
  const int64_t b = sdlh::hctrl_budget(&h);
  CK(mcpy(ctl_dev_ + local, &c, sizeof(c), cudaMemcpyHostToDevice));
  CK(mcpy(budget_dev_ + local, &b, sizeof(b), cudaMemcpyHostToDevice));
}

void Engine::global(int local, const int32_t** idx, const float** val, int64_t* nnz) {
  sync();
  const Slot& gs = global_[static_cast<size_t>(team_of_local_global_[static_cast<size_t>(local)])];
  int32_t n = 0;
  CK(mcpy(&n, gs.cnt, sizeof(n), cudaMemcpyDeviceToHost));
  *idx = gs.idx;
  *val = gs.val;
  *nnz = n;
}

}  // namespace sdle
