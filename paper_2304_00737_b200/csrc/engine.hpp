// The SparDL iteration planner/executor (host C++).
//
// At context creation the whole iteration of spardl_all_reduce
// (inc/pipeline.hpp:140-342) is planned once, for every one of the P
// workers, by replaying the reference schedule symbolically: which block
// buffers exist, which worker merges which pieces in which order, which
// buffer moves to which worker in which round.  The plan is identical on
// every rank (it depends only on the config), so NCCL point-to-point ops
// match without any runtime negotiation.  Only the tasks of this rank's
// workers become device work; their descriptors are uploaded once, so an
// iteration is a fixed sequence of kernel launches and NCCL group calls
// (CUDA-graph capturable).
#pragma once

#include <cuda_runtime.h>
#include <nccl.h>

#include <array>
#include <cstdint>
#include <map>
#include <memory>
#include <set>
#include <string>
#include <vector>

#include "host.hpp"
#include "kernels.cuh"

namespace sdle {

// A block buffer: [int32 cnt | pad to 16 B][int32 idx[cap]][float val[cap]],
// contiguous so one NCCL op moves it.
struct Slot {
  unsigned char* base = nullptr;
  int32_t* cnt = nullptr;
  int32_t* idx = nullptr;
  float* val = nullptr;
  int64_t cap = 0;
  size_t bytes = 0;
};

class Arena {
 public:
  ~Arena();
  void* alloc(size_t bytes);
  size_t total() const { return total_; }
  bool dry = false;   // plan-only mode: hand out fake addresses, touch no device

 private:
  std::vector<void*> chunks_;
  unsigned char* cur_ = nullptr;
  size_t left_ = 0;
  size_t total_ = 0;
};

struct Xfer {            // one block moved from a worker to another rank
  int uid;
  int src_worker;
  int src_rank;
  int dst_rank;
};

struct Stage {           // one batch of merge + select tasks
  std::vector<sdl::MergeTask> merges;
  std::vector<sdl::SelTask> sels;
  sdl::MergeTask* merges_dev = nullptr;
  sdl::SelTask* sels_dev = nullptr;
  int max_parts = 0;
  int max_rT = 0;
  int max_r = 0;
  int max_nseg = 0;
  std::set<int> produced;    // uids written by this stage (dependency guard)
  std::vector<int64_t> merge_cap;   // input capacity of each merge task
  std::vector<std::vector<int>> merge_in;   // input block uids of each merge task
  std::vector<int> sel_uid;         // output block uid of each select task
  std::vector<int> sel_in;          // input block uid of a single-block select, else -1
  bool fused = false;        // merges run inside the select kernel (no merge launches)
  int cl = 0;                // fused: cluster width
  int win_cap = 0;           // fused: window entries per CTA
  bool wide = false;         // every select runs the wide path first (wselect.cu)
  int w_max_tiles = 0;       // wide: largest tile count of a task
  int64_t w_max_entries = 0; // wide: largest input capacity of a task
  bool need_wide = false;    // a dividing block too large for the cluster select's work list
  bool coop = false;         // wide: the single-kernel cooperative form (k_wsel_coop)
  int w_max_nseg = 0;        // wide: most input segments of a task
  std::vector<sdl::WScratch*> ws;   // wide: per select task
};

struct Step {            // a stage followed by a transport round
  Stage stage;
  std::vector<Xfer> xfers;   // empty: no round
  bool controller_after = false;
};

// One NCCL point-to-point op of a rank's iteration (plan-only inspection).
struct PlanOp {
  int32_t round;
  int32_t peer;       // other rank
  int32_t is_send;
  int32_t uid;        // block buffer id (identical numbering on every rank)
  int64_t bytes;
};

class Engine {
 public:
  Engine(const spardl_config& cfg, int device, int world, int rank, const void* nccl_id,
         cudaStream_t stream, bool plan_only = false);
  // the NCCL ops this rank issues per iteration, in issue order
  std::vector<PlanOp> plan_ops() const;
  ~Engine();

  void run(const float* const* grads_dev);
  // upload a new gradient pointer table in stream order when it changed
  void set_grads(const float* const* grads);
  // per-phase device time of `iters` profiled (non-graph) iterations, ms:
  // [sample+prethr, candidate pass, dividing select, SRS/SAG, gather+finalize]
  void profile(const float* const* grads_dev, int iters, double* phase_ms);
  void sync();
  void reset_state();
  spardl_run_info run_info();
  void ledger(int64_t* rounds, int64_t* scalars);
  void union_sizes(int64_t* out);
  // dividing selects of the last iteration that fell back to the dense path
  int64_t dense_fallbacks();
  // dividing selects that fell back to the dense path since reset_state()
  int64_t dense_fallbacks_total();
  // dividing blocks whose carried pre-threshold missed and whose candidates
  // were redone from a fresh sample (k_div_recand) since reset_state()
  int64_t candidate_retries();
  // wide-path selects handed back to the cluster select since reset_state()
  int64_t wide_handed_back();
  // device timestamps (ns) of the phases of one select of the last run
  void select_timestamps(int step, int task, int64_t* out12);
  // [mode, cand_bad, cand_total, cand_count, pre_key, cap] of dividing task i
  void div_diag(int task, int64_t* out);
  void controller(int local, spardl_hctrl* out);
  void set_controller(int local, const spardl_hctrl& c);
  void global(int local, const int32_t** idx, const float** val, int64_t* nnz);
  // the residual of local worker `local` (pending deferred finalize applied)
  float* carry(int local) {
    flush_finalize();
    return carry_[static_cast<size_t>(local)];
  }
  // applies the last iteration's deferred finalize records to the carries
  // (no-op when none are pending); synchronises
  void flush_finalize();
  bool finalize_deferred() const { return fin_defer_; }
  int64_t dimension() const { return cfg_.dimension; }
  int first_worker() const { return first_; }
  int local_workers() const { return wloc_; }
  int64_t launches_per_iter() const { return launches_; }
  cudaStream_t stream() const { return stream_; }
  cudaStream_t side_stream() const { return side_; }
  void set_graph(bool on) {
    use_graph_ = on;
    drop_graph();
  }
  // the sparse conservation audit of inc/pipeline.hpp:304-332 (gres, pres):
  // off the global gradient both sides are the same values, so only the k
  // global positions are compared; reported by run_info()
  void set_audit(bool on);

 private:
  // --- planning
  struct Held {                   // symbolic held block: pending pieces
    std::vector<int> pieces;      // uids, in fold order
  };
  int new_uid(int owner_worker);
  Slot& local_slot(int uid);      // the local copy (must exist)
  bool has_local(int uid) const { return slots_.count(uid) != 0; }
  Slot make_slot(int uid);
  Slot sym_slot(int uid) const;   // uid's buffer in its owner's symmetric region
  int materialize(int w, int pos, std::vector<int> pieces, int64_t budget, float weight,
                  const int64_t* budget_dev, int64_t* total_out, Stage& st, int xi_block);
  void add_select(Stage& st, const sdl::SelTask& t, int out_uid, int in_uid);
  // wide-select scratch of a task over the given input segments
  sdl::WScratch* make_wide(Stage& st, sdl::SelTask& t, const int32_t* idx, const float* val,
                           const int32_t* seg_off, const int32_t* seg_cnt, const int32_t* count,
                           int stride, int nseg, int group, int mode, int is_div, int64_t bin_cap,
                           int64_t typical);   // typical: the input's expected size
  // the wide select (wselect.cu) for stages the cluster select cannot fill
  // (see finish_stage); SPARDL_WSEL=1: every stage, =0: never
  bool wide_on_ = true;
  bool wsel_force_ = false;
  int wsel_max_tasks_ = 12;            // stages of at most this many selections ...
  int64_t wsel_min_entries_ = 200000;  // ... with inputs of at least this many entries
  bool wsel_fuse_ = false;   // SPARDL_WSEL_FUSE=1: producers histogram for the wide select
  bool wsel_coop_ = true;    // SPARDL_WSEL_COOP=0: the tiled wide select (three kernels)
  bool wsel_coop_force_ = false;   // SPARDL_WSEL_COOP=2: cooperative even past the on-chip copies
  int wsel_fit_ = 0;         // SPARDL_WSEL_FIT=1: the cooperative select wherever a stage fits on chip (2: dividing too)
  sdl::SelTask select_from_slot(const Slot& in);
  sdl::SelTask select_from_merge(Stage& st, const std::vector<int>& pieces);
  void finish_stage(Stage& st);
  void plan_fused(Stage& st);
  double conservation_audit();
  std::vector<float*> aud_comb_, aud_carry_;   // per local worker, k entries each
  float* aud_gather_ = nullptr;                 // all workers' pairs (world > 1)
  void transfer(std::vector<Xfer>& xs, int uid, int src_worker, int dst_worker, int phase,
                std::vector<std::vector<int>>* recv_into = nullptr);
  void plan();
  bool is_local(int w) const { return w >= first_ && w < first_ + wloc_; }
  int rank_of(int w) const { return w / wloc_; }
  void exec_round(const std::vector<Xfer>& xs);
  int exec_stage(const Stage& st, bool dividing, cudaEvent_t after_merge = nullptr);
  void reset_wide(const Stage& st);
  cudaError_t mcpy(void* dst, const void* src, size_t bytes, cudaMemcpyKind kind) {
    return dry_ ? cudaSuccess : cudaMemcpy(dst, src, bytes, kind);
  }
  bool dry_ = false;
  void enqueue_iteration(cudaEvent_t* ev = nullptr);
  void drop_graph();

  // --- config
  spardl_config cfg_;
  int P_ = 1, m_ = 1, d_ = 1, l_ = 0;
  int64_t L_ = 1, Lcap_ = 4;
  sdlh::Partition part_;
  int device_ = 0, world_ = 1, rank_ = 0, wloc_ = 1, first_ = 0;
  cudaStream_t stream_ = nullptr;
  cudaStream_t side_ = nullptr;
  cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr;
  // dividing pass split into worker groups: group g's select (high-priority
  // stream hi_) overlaps the candidate pass of group g+1 (SPARDL_DIV_SPLIT)
  cudaStream_t hi_ = nullptr;
  cudaEvent_t ev_div_[2] = {nullptr, nullptr};
  int div_split_ = 1;
  bool own_stream_ = false;
  ncclComm_t comm_ = nullptr;
  bool use_graph_ = true;
  bool audit_ = false;
  cudaGraphExec_t graph_ = nullptr;
  std::vector<cudaEvent_t> step_ev_;   // profiling diagnostics (SPARDL_STEP_EVENTS)
  int64_t launches_ = 0;

  Arena arena_;
  // per local worker
  std::vector<float*> carry_;
  std::vector<int64_t*> ledger_total_;   // device [1] per worker (cumulative scalars)
  int64_t* ledger_phase_ = nullptr;      // device [wloc*3] per call
  int64_t* ntot_ = nullptr;              // device [wloc] B-SAG union sizes
  int64_t* budget_dev_ = nullptr;        // device [wloc] B-SAG pre-selection budgets
  sdl::HCtl* ctl_dev_ = nullptr;         // device [wloc]
  const float** gtab_dev_ = nullptr;     // device [wloc] gradient pointers
  const float** gtab_host_ = nullptr;    // pinned ring of kTabRing tables
  static constexpr int kTabRing = 32;
  std::vector<const float*> gtab_cur_;   // the table the device holds (last upload)
  cudaEvent_t tab_ev_[kTabRing] = {};
  bool tab_used_[kTabRing] = {};
  int tab_next_ = 0;
  int32_t* err_dev_ = nullptr;           // NaN flag
  unsigned long long* fallbacks_dev_ = nullptr;   // dense fallbacks since reset_state()
  unsigned long long* wide_back_dev_ = nullptr;   // wide selects handed back since reset_state()
  unsigned long long* retries_dev_ = nullptr;     // dividing candidate passes redone since reset_state()
  int64_t* hash_dev_ = nullptr;          // [d] consistency hashes
  int64_t* rb_dev_ = nullptr;            // readback scratch
  std::vector<int64_t> rounds_;          // host, per global worker (cumulative)
  std::vector<std::array<int64_t, 3>> phase_rounds_;  // per global worker per call

  // plan
  int next_uid_ = 0;
  std::vector<int> uid_owner_;
  std::map<int, Slot> slots_;            // uid -> local buffer
  std::vector<sdl::DivTask> div_tasks_;
  sdl::DivTask* div_dev_ = nullptr;
  int div_max_chunks_ = 0, div_sample_every_ = 1;
  Stage div_stage_;
  std::vector<Step> steps_;
  std::vector<sdl::LedgerAdd> ledger_adds_;
  sdl::LedgerAdd* ledger_dev_ = nullptr;
  std::vector<sdl::AssembleTask> asm_tasks_;
  std::vector<std::vector<int>> asm_in_;     // source block uids of each assembly
  sdl::AssembleTask* asm_dev_ = nullptr;
  std::vector<sdl::FinalizeTask> fin_tasks_;
  // deferred finalize (gres): records written at the end of an iteration,
  // applied by the next candidate pass (or flush_finalize)
  bool fin_defer_ = false;
  int fin_mode_ = 0;                     // SPARDL_FIN_DEFER (see plan())
  bool fin_defer_ok_ = false;            // the plan allows it (audit may switch it off)
  std::vector<sdl::FinRecTask> fin_rec_;
  sdl::FinRecTask* fin_rec_dev_ = nullptr;
  int32_t* fin_apply_ = nullptr;         // device flag: records pending
  void set_defer(bool on);
  sdl::FinalizeTask* fin_dev_ = nullptr;
  int64_t fin_max_div_ = 0;
  std::vector<sdl::CtlTask> ctl_tasks_;
  sdl::CtlTask* ctl_tasks_dev_ = nullptr;
  std::vector<int> team_of_local_global_;    // local worker -> index into global_ bufs
  std::vector<Slot> global_;                 // per local team: assembled global (cap k)
  std::vector<int> global_team_;             // team id of each global_ entry
  // per local worker, per block: dividing outputs and discard lists
  std::vector<std::vector<int>> div_uid_;
  std::vector<std::vector<const sdl::SelScratch*>> div_scr_;
  std::vector<const sdl::GatherSrc*> team_src_;   // per global_ entry: the m reserved blocks
  std::vector<std::vector<sdl::GatherSrc>> team_src_host_;   // (host copies)
  std::vector<std::vector<std::vector<sdl::XiList>>> xi_;
  std::vector<int> union_group_owner_;       // position group -> worker providing N_t
  bool ran_ = false;

  // --- peer-memory transport (transport.cu); NCCL send/recv when off
  void setup_peer();                    // before plan(): symmetric region + IPC mappings
  void plan_peer();                     // after plan(): publish / wait lists
  bool peer_ = false;
  unsigned char* sym_ = nullptr;
  std::vector<unsigned char*> peer_base_;   // per rank; own entry is sym_
  std::vector<char> peer_ipc_;              // per rank: mapped through CUDA IPC (to close)
  size_t slot_stride_ = 0, flags_off_ = 0, done_off_ = 0;
  std::vector<int> uid_slot_;               // buffer index of each uid (peer transport: global)
  std::map<int, std::vector<int>> push_dst_;   // uid -> remote ranks its producer writes into
  Slot own_slot(int uid) const;             // this rank's copy of a pushed block
  void wire_push(sdl::SelTask& t, int uid);
  std::vector<int> rank_slots_;             // buffers numbered so far, per rank
  std::vector<std::pair<int, int>> deliveries_;   // (uid, destination rank), whole plan
  long long* epoch_ = nullptr;
  int32_t* peer_err_ = nullptr;
  unsigned long long timeout_ns_ = 10ull * 1000 * 1000 * 1000;   // one peer wait
  bool poisoned_ = false;   // a peer wait timed out: state void until reset_state()
  const long long** begin_dev_ = nullptr;
  long long** done_dev_ = nullptr;
  int npeer_ = 0;

 public:
  bool peer_transport() const { return peer_; }
};

}  // namespace sdle
