/*
 * spardl_cuda.h -- the C ABI of the B200-native SparDL sparse All-Reduce.
 *
 * This is the drop-in boundary for the reference's hot path, the C++ API of
 * /root/reference/proj/include/spardl (abbreviated `inc/`).  Every entry
 * point names the reference interface it replaces.  Plain pointers and sizes
 * only; no C++ or torch types.  All functions return a status (SPARDL_OK or
 * one SPARDL_E_* per reference exception class, inc/error.hpp:23-75) and set
 * a thread-local message readable with spardl_last_error(); the message text
 * of every reference error is reproduced verbatim.
 *
 * Threading/ownership: a context (spardl_ctx) belongs to one process and one
 * CUDA device and hosts a contiguous range of the P logical workers
 * ("local workers").  P workers may live on 1..P devices (P % world_size == 0);
 * the reference's single-call-drives-all-workers semantics
 * (inc/pipeline.hpp:140-142) is the world_size == 1 case.  Workers on other
 * devices are reached over NVLink through NCCL point-to-point rounds.
 *
 * The hot path never falls back to the CPU: without a usable sm_100 device
 * spardl_ctx_create fails with SPARDL_E_CUDA.
 */
#ifndef SPARDL_CUDA_H_
#define SPARDL_CUDA_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define SPARDL_ABI_VERSION 1

/* status codes -- one per reference exception class (inc/error.hpp) */
#define SPARDL_OK 0
#define SPARDL_E_ERROR 1            /* spardl::error                 error.hpp:23 */
#define SPARDL_E_PARTITION 2        /* spardl::partition_error       error.hpp:29 */
#define SPARDL_E_BLOCK_MISMATCH 3   /* spardl::block_mismatch_error  error.hpp:35 */
#define SPARDL_E_SCHEDULE 4         /* spardl::schedule_violation_error error.hpp:41 */
#define SPARDL_E_THEOREM 5          /* spardl::theorem_violation_error  error.hpp:47 */
#define SPARDL_E_GROUP_SIZE 6       /* spardl::group_size_error      error.hpp:53 */
#define SPARDL_E_CONFIG 7           /* spardl::config_error          error.hpp:60 */
#define SPARDL_E_STATE 8            /* spardl::state_error           error.hpp:66 */
#define SPARDL_E_CONSISTENCY 9      /* spardl::consistency_error     error.hpp:72 */
#define SPARDL_E_CUDA 100           /* device / runtime failure (no reference analogue) */
#define SPARDL_E_NCCL 101           /* transport failure */
#define SPARDL_E_ARG 102            /* invalid pointer / size argument */
#define SPARDL_E_UNSUPPORTED 103    /* configuration outside the device envelope */

/* enums of inc/sag.hpp:272, inc/residual.hpp:37, inc/reduce_scatter.hpp:34 */
#define SPARDL_SAG_NONE 0
#define SPARDL_SAG_RSAG 1
#define SPARDL_SAG_BSAG 2
#define SPARDL_RES_GRES 0
#define SPARDL_RES_PRES 1
#define SPARDL_RES_LRES 2
#define SPARDL_TIMING_OPTIMIZED 0
#define SPARDL_TIMING_NAIVE 1

/* spardl::ClusterConfig, inc/pipeline.hpp:39-52 (field for field) */
typedef struct spardl_config {
  int64_t workers;   /* P */
  int64_t dimension; /* N */
  int64_t k;         /* total selection count */
  int64_t teams;     /* d */
  int32_t sag;       /* SPARDL_SAG_* */
  int32_t residual;  /* SPARDL_RES_* */
  int32_t timing;    /* SPARDL_TIMING_* */
  int32_t pad_;
  uint64_t seed;
} spardl_config;

/* spardl::RunResult scalars, inc/pipeline.hpp:115-127 */
typedef struct spardl_run_info {
  int32_t consistent;
  int32_t conservation_applicable;
  double conservation_error;   /* when the audit is enabled (gres, pres), else -1 */
  int64_t max_rounds, max_scalars;            /* LedgerReport, fabric.hpp:41-45 */
  int64_t srs_rounds, srs_scalars;            /* srs_phase */
  int64_t sag_rounds, sag_scalars;            /* sag_phase */
  int64_t gather_rounds, gather_scalars;      /* gather_phase */
  int64_t pred_rounds, pred_low, pred_high;   /* predicted, sag.hpp:283-289 */
  int64_t n_union;                            /* union_sizes.size() */
  int64_t global_nnz;
} spardl_run_info;

/* spardl::HController state, inc/sag.hpp:37-90 */
typedef struct spardl_hctrl {
  double lower, upper;
  int64_t target;
  double h, step;
  int32_t flag;
  int32_t pad_;
} spardl_hctrl;

typedef struct spardl_ctx spardl_ctx;

const char* spardl_last_error(void);
/* CUDA devices visible to this process (0 without a GPU) */
int spardl_device_count(int32_t* n);
int spardl_abi_version(void);

/* ------------------------------------------------------------------ */
/* host-side schedule logic (no GPU needed)                            */
/* ------------------------------------------------------------------ */
/* validate(ClusterConfig), inc/pipeline.hpp:54-78 */
int spardl_validate(const spardl_config* cfg);
/* partition(N, B), inc/sparse.hpp:98-117: lo[B], hi[B] */
int spardl_partition(int64_t n, int32_t count, int64_t* lo, int64_t* hi);
/* BlockPartition::block_of, inc/sparse.hpp:88-95 */
int spardl_block_of(int64_t n, int32_t count, int64_t i, int32_t* block);
/* build_bags(m, rank), inc/reduce_scatter.hpp:51-74.
 * bag_size[l] receives |B_1..B_l|, positions[m-1] the bags concatenated. */
int spardl_build_bags(int32_t m, int32_t rank, int32_t* l, int32_t* remainder,
                      int32_t* bag_size, int32_t* positions);
/* expected_cost_srs, inc/reduce_scatter.hpp:257-262 */
int spardl_expected_cost_srs(int64_t m, int64_t k, int64_t* rounds, int64_t* scalars);
/* expected_cost_sag, inc/sag.hpp:295-329 (mode = SPARDL_SAG_*) */
int spardl_expected_cost_sag(int64_t P, int64_t k, int64_t d, int32_t mode, int64_t* rounds,
                             int64_t* low, int64_t* high);
/* bsag_phase_cost, inc/sag.hpp:332-340 */
int spardl_bsag_phase_cost(int64_t P, int64_t k, int64_t d, int64_t* rounds, int64_t* low,
                           int64_t* high);
/* topka_cost, inc/sag.hpp:343-346 */
int spardl_topka_cost(int64_t P, int64_t k, int64_t* rounds, int64_t* low, int64_t* high);
/* dyadic_shares, inc/sag.hpp:108-118 */
int spardl_dyadic_shares(int32_t count, double* out);
/* HController ctor / observe / budget, inc/sag.hpp:40-81 */
int spardl_hctrl_init(spardl_hctrl* c, int64_t P, int64_t k, int64_t d);
int spardl_hctrl_observe(spardl_hctrl* c, int64_t n_t);
int spardl_hctrl_budget(const spardl_hctrl* c, int64_t* budget);

/* ------------------------------------------------------------------ */
/* device components (device pointers; enqueued on `stream`, then      */
/* synchronised because the output sizes are returned to the host)     */
/* ------------------------------------------------------------------ */
/* top_k_select, inc/sparse.hpp:136-162: n index-sorted entries in; the
 * selected and discarded entries out, each index-sorted.  Output arrays
 * must hold n entries; dis_* may be NULL. */
int spardl_topk_select(const int32_t* idx, const float* val, int64_t n, int64_t budget,
                       int32_t* sel_idx, float* sel_val, int64_t* n_sel, int32_t* dis_idx,
                       float* dis_val, int64_t* n_dis, void* stream);
/* top_k_select_slice, inc/sparse.hpp:167-177: dense values g[lo..hi) */
int spardl_topk_select_slice(const float* g, int64_t lo, int64_t hi, int64_t budget,
                             int32_t* sel_idx, float* sel_val, int64_t* n_sel, void* stream);
/* r-fold merge_add, inc/sparse.hpp:182-208: out = ((l0 + l1) + l2) ... ;
 * out arrays hold sum(n_t) entries. */
int spardl_merge_add(int32_t r, const int32_t* const* idx, const float* const* val,
                     const int64_t* n, int32_t* out_idx, float* out_val, int64_t* n_out,
                     void* stream);

/* The same three components on HOST buffers (staged through the device by
 * the library; synchronous).  Used by the C++ drop-in shim. */
/* fp64 forms (the C++ drop-in surface, include/spardl/): the reference's
 * double semantics.  top_k_select: flag[i] = 1 for the min(budget, n)
 * entries first in (|val| desc, idx asc), inc/sparse.hpp:136-162; merge_add
 * of two index-sorted lists, coinciding indices summed a + b,
 * inc/sparse.hpp:182-208.  Device pointers (stream-ordered, synchronising)
 * and host-buffer variants. */
int spardl_topk_select_f64(const int64_t* idx, const double* val, int64_t n, int64_t budget,
                           uint8_t* flag, void* stream);
int spardl_merge_add_f64(const int64_t* ai, const double* av, int64_t na, const int64_t* bi,
                         const double* bv, int64_t nb, int64_t* oi, double* ov, int64_t* n_out,
                         void* stream);
int spardl_topk_select_f64_hostbuf(const int64_t* idx, const double* val, int64_t n,
                                   int64_t budget, uint8_t* flag);
int spardl_merge_add_f64_hostbuf(const int64_t* ai, const double* av, int64_t na,
                                 const int64_t* bi, const double* bv, int64_t nb, int64_t* oi,
                                 double* ov, int64_t* n_out);
int spardl_topk_select_hostbuf(const int32_t* idx, const float* val, int64_t n, int64_t budget,
                               int32_t* sel_idx, float* sel_val, int64_t* n_sel,
                               int32_t* dis_idx, float* dis_val, int64_t* n_dis);
int spardl_topk_select_slice_hostbuf(const float* g, int64_t lo, int64_t hi, int64_t budget,
                                     int32_t* sel_idx, float* sel_val, int64_t* n_sel);
int spardl_merge_add_hostbuf(int32_t r, const int32_t* const* idx, const float* const* val,
                             const int64_t* n, int32_t* out_idx, float* out_val, int64_t* n_out);

/* ------------------------------------------------------------------ */
/* the pipeline: spardl_all_reduce, inc/pipeline.hpp:140-342           */
/* ------------------------------------------------------------------ */
/* NCCL rendezvous for multi-process contexts: rank 0 creates the id and
 * the caller broadcasts its 128 bytes (e.g. with torch.distributed). */
int spardl_nccl_unique_id(void* out128);

/* make_worker_states + Fabric(P), inc/pipeline.hpp:87-99 / fabric.hpp:54.
 * device: CUDA ordinal; world_size/rank: processes sharing the P workers
 * (world_size 1 => all workers local, nccl_id ignored); stream: cudaStream_t
 * the work is enqueued on (NULL: a context-owned stream). */
int spardl_ctx_create(const spardl_config* cfg, int32_t device, int32_t world_size,
                      int32_t rank, const void* nccl_id, void* stream, spardl_ctx** out);
int spardl_ctx_destroy(spardl_ctx* ctx);
/* Host-only schedule inspection (no GPU): the NCCL point-to-point ops rank
 * `rank` of `world_size` issues per iteration, in issue order, 5 int64 each:
 * (round, peer rank, is_send, block id, bytes).  ops may be NULL to query
 * the count.  Every rank derives the same plan, so sends and receives of a
 * rank pair match one to one in order (tested with a gloo process group). */
int spardl_plan_ops(const spardl_config* cfg, int32_t world_size, int32_t rank, int64_t* ops,
                    int64_t cap, int64_t* n_ops);
/* first global worker id and count of the workers hosted by this context */
int spardl_ctx_local_workers(const spardl_ctx* ctx, int32_t* first, int32_t* count);
/* *peer = 1 when blocks move by direct peer-memory reads over NVLink (CUDA
 * IPC mappings; all ranks on one node), 0 when by NCCL send/recv.  The
 * environment variable SPARDL_TRANSPORT=nccl forces NCCL at creation. */
int spardl_ctx_transport(const spardl_ctx* ctx, int32_t* peer);
/* enable (1) / disable (0) CUDA-graph replay of the whole iteration */
int spardl_ctx_set_graph(spardl_ctx* ctx, int32_t enable);
/* enable the conservation audit (inc/pipeline.hpp:305-334), computed exactly
 * on the k global positions (off them both sides are the same values); the
 * next spardl_get_run_info reports it (collective). */
int spardl_ctx_set_audit(spardl_ctx* ctx, int32_t enable);

/* One synchronisation: grads[i] is local worker i's dense fp32 gradient
 * (device pointer, N floats, 16-byte aligned).  Enqueued asynchronously. */
int spardl_allreduce(spardl_ctx* ctx, const float* const* grads_dev);
/* Same, with HOST gradients (pinned or pageable): the copies in and the
 * result copy out are part of the call (the reference's host signature). */
int spardl_allreduce_host(spardl_ctx* ctx, const float* const* grads_host, int64_t* g_idx,
                          float* g_val, int64_t cap, int64_t* nnz);
/* Measurement hook (bench.py): runs `iters` extra iterations outside any
 * CUDA graph with events on the context stream at the phase boundaries and
 * returns the mean device time per phase in ms: [0] sampling + pre-threshold,
 * [1] fused residual-add/candidate pass, [2] dividing select, [3] SRS/SAG
 * stages and rounds, [4] final gather + assemble + finalize + ledger.
 * The iterations advance the residual state like ordinary calls. */
int spardl_profile(spardl_ctx* ctx, const float* const* grads_dev, int32_t iters,
                   double* phase_ms);
/* wait for the enqueued work; reports device-side errors (NaN input) */
int spardl_sync(spardl_ctx* ctx);
/* RunResult scalars of the last call (synchronises; collective when
 * world_size > 1: every rank must call it) */
int spardl_get_run_info(spardl_ctx* ctx, spardl_run_info* out);
/* device view of local worker i's GlobalSparseGradient (valid until the
 * next call); *nnz needs a sync, so this synchronises */
int spardl_get_global(spardl_ctx* ctx, int32_t local_worker, const int32_t** idx,
                      const float** val, int64_t* nnz);
/* WorkerState::residual.carry() of local worker i (device, N floats) */
int spardl_get_carry(spardl_ctx* ctx, int32_t local_worker, float** carry_dev);
/* host copies of WorkerState::residual.carry() (N floats; synchronise) --
 * used by the C++ drop-in shim to keep the reference's value semantics */
int spardl_carry_to_host(spardl_ctx* ctx, int32_t local_worker, float* host);
int spardl_carry_from_host(spardl_ctx* ctx, int32_t local_worker, const float* host);
/* overwrite WorkerState::controller of local worker i (B-SAG only) */
int spardl_set_controller(spardl_ctx* ctx, int32_t local_worker, const spardl_hctrl* c);
/* reset residuals / controllers / ledger to the make_worker_states state */
int spardl_ctx_reset_state(spardl_ctx* ctx);
/* Fabric::ledger(), fabric.hpp:110: per GLOBAL worker (P entries); collective */
int spardl_get_ledger(spardl_ctx* ctx, int64_t* rounds, int64_t* scalars);
/* RunResult::union_sizes (B-SAG N_t per position group; n_union entries) */
int spardl_get_union_sizes(spardl_ctx* ctx, int64_t* out);
/* WorkerState::controller of local worker i (B-SAG only) */
int spardl_get_controller(spardl_ctx* ctx, int32_t local_worker, spardl_hctrl* out);
/* diagnostics: dividing selections of the last call that could not use the
 * candidate fast path and selected from the dense slice (synchronises) */
int spardl_dense_fallbacks(spardl_ctx* ctx, int64_t* count);
/* diagnostics: dividing selections that took the dense path, summed over every
 * call since creation / reset_state (synchronises) */
int spardl_dense_fallbacks_total(spardl_ctx* ctx, int64_t* count);
/* diagnostics: selections the wide (whole-GPU) select handed back to the
 * cluster select (threshold outside the dividing window, massive key ties),
 * summed since creation / reset_state (synchronises) */
int spardl_wide_handed_back(spardl_ctx* ctx, int64_t* count);
/* diagnostics: dividing blocks whose carried pre-threshold missed (too few
 * candidates, a chunk overflow) and whose candidates were redone from a fresh
 * sample instead of the dense path, summed since creation / reset_state
 * (synchronises) */
int spardl_candidate_retries(spardl_ctx* ctx, int64_t* count);
/* diagnostics of local dividing task i (= local_worker * m + block):
 * [resolved mode, candidate flags, candidate total, list length, pre-key, capacity,
 *  selection threshold key, carried next pre-key (-1: none), carried margin] */
int spardl_div_diag(spardl_ctx* ctx, int32_t task, int64_t* out9);
/* diagnostics: device timestamps (ns) of the phases of select `task` of
 * planner step `step` (-1: the dividing stage) in the last iteration:
 * out[0..12) CTA 0's phase stamps, [12..28) each cluster CTA's start,
 * [28..44) each CTA's end of the first histogram pass, [44..52) CTA 0's
 * fused-merge phases (and guess diagnostics), [52..116) the feeding merge's
 * phase stamps for its partitions 0..7 (8 each) */
int spardl_debug_select_timestamps(spardl_ctx* ctx, int32_t step, int32_t task, int64_t* out116);
/* number of kernels this context launches per iteration */
int spardl_kernel_launches(const spardl_ctx* ctx, int64_t* per_iteration);
/* the stream the context enqueues on (cudaStream_t) */
int spardl_ctx_stream(const spardl_ctx* ctx, void** stream);

/* ---------------------------------------------------------------------------
 * One process, one host thread, several local GPUs (the reference's call
 * shape: one spardl_all_reduce advances all P workers, inc/fabric.hpp:47-53,
 * inc/pipeline.hpp:140-142).  One engine per device (ranks of one NCCL
 * clique, peers read each other's buffers through direct peer access);
 * worker w lives on devs[w / (P / ndev)].  devs == NULL: devices 0..ndev-1.
 * The iteration is enqueued on every device from the calling thread;
 * run-info / ledger gathers run one internal host thread per device. */
typedef struct spardl_mctx spardl_mctx;
int spardl_mctx_create(const spardl_config* cfg, int32_t ndev, const int32_t* devs,
                       spardl_mctx** out);
int spardl_mctx_destroy(spardl_mctx* m);
int spardl_mctx_devices(const spardl_mctx* m, int32_t* ndev, int32_t* transport_peer);
int spardl_mctx_allreduce(spardl_mctx* m, const float* const* grads_dev);
int spardl_mctx_allreduce_host(spardl_mctx* m, const float* const* grads_host, int64_t* g_idx,
                               float* g_val, int64_t cap, int64_t* nnz);
int spardl_mctx_sync(spardl_mctx* m);
int spardl_mctx_get_run_info(spardl_mctx* m, spardl_run_info* out);
int spardl_mctx_get_ledger(spardl_mctx* m, int64_t* rounds, int64_t* scalars);
int spardl_mctx_get_union_sizes(spardl_mctx* m, int64_t* out);
int spardl_mctx_get_global(spardl_mctx* m, int32_t worker, int64_t* g_idx, float* g_val,
                           int64_t cap, int64_t* nnz);
int spardl_mctx_carry_to_host(spardl_mctx* m, int32_t worker, float* host);
int spardl_mctx_carry_from_host(spardl_mctx* m, int32_t worker, const float* host);
int spardl_mctx_set_controller(spardl_mctx* m, int32_t worker, const spardl_hctrl* c);
int spardl_mctx_get_controller(spardl_mctx* m, int32_t worker, spardl_hctrl* c);
int spardl_mctx_reset_state(spardl_mctx* m);

#ifdef __cplusplus
}
#endif

#endif /* SPARDL_CUDA_H_ */
