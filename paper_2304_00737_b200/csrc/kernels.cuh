// Device-side data model and kernel launchers of the SparDL B200 path.
//
// Everything on the device is SoA: a sparse block is (int32 idx[], float
// val[], int32 count) with a fixed capacity -- the reference's AoS
// {int64 index; double value} Entry (inc/sparse.hpp:57-62) re-laid for
// coalesced 128-bit traffic.  Indices are int32 (N < 2^31).
//
// Three kernel families:
//   select  -- deterministic top-L over a *segmented* list (|v| desc, index
//              asc; inc/sparse.hpp:122-162): 3 radix passes over the 31-bit
//              magnitude key, per-segment counts, ordered compaction of the
//              selected and discarded parts (both index-sorted).
//   merge   -- r-way index merge with a left fold of the values in list order
//              (inc/sparse.hpp:182-208 applied r-1 times), sample-splitter
//              partitioned so every CTA merges <= r*T entries in shared memory.
//   divide  -- the dividing pass (inc/pipeline.hpp:162-184): residual add fused
//              with candidate compaction above a sampled pre-threshold.
#pragma once
#ifndef SPARDL_STAMPS
#define SPARDL_STAMPS 0   // device phase timestamps (diagnostics; make EXTRA=-DSPARDL_STAMPS=1)
#endif

#include <cuda_runtime.h>
#include <stdint.h>

namespace sdl {

constexpr int kThreads = 256;
constexpr int kBins = 2048;            // radix digit width of passes 0 and 1 (11 bits)
constexpr int kMaxR = 16;              // max lists folded by one merge task
#ifndef SPARDL_DIV_CHUNK
#define SPARDL_DIV_CHUNK 8192
#endif
constexpr int kChunk = SPARDL_DIV_CHUNK;   // dividing chunk (elements per CTA)
constexpr int kMaxSamples = 8000;      // merge splitter samples per task (< kMaxSegPerTask)
constexpr int kTile = 256;             // select work item (entries per warp task)
constexpr int kCl = 16;                // CTAs per select cluster (one cluster per task)
constexpr int kMaxSegPerTask = 8192;   // select work items per task (smem bound)
constexpr int kSampShift = 18;         // dividing sample histogram: key >> 18
constexpr int kSampBins = 1 << (31 - kSampShift);   // 8192 bins (1/32 octave)

// Peer-transport synchronisation carried by a task (empty lists: none): the
// task first waits until the flags of its remote inputs reach the iteration
// epoch, and its producer publishes the epoch to the consumers' flags of its
// output as soon as the output is complete.
struct PeerSync {
  const long long* const* wait;   // local flags of remote inputs
  long long* const* pub;          // consumers' flags of this task's output
  int32_t nwait;
  int32_t npub;
  const long long* epoch;
  int32_t* err;                   // timeout flag (this GPU's; set: the iteration is void)
  unsigned long long timeout_ns;  // bound of one wait (SPARDL_PEER_TIMEOUT_MS, default 10 s)
};

struct SelTask;
struct WScratch;
// Host helper: fills the derived work-decomposition fields of a select task
// (tiles per input segment; dense tiles) given the largest possible length of
// one input segment.  Returns the number of work segments of the task.
int sel_prepare(SelTask& t, int max_seg_len);
int sel_scratch_segments(const SelTask& t);   // per-segment scratch entries needed
int sel_grid_segments(const SelTask& t);      // segments the launch grid is sized for
int sel_chunk_capacity(const SelTask& t);     // per-chunk scratch entries needed

// ---------------------------------------------------------------------------
// Select
// ---------------------------------------------------------------------------
// Per-task scratch, device resident.  `hist` is left zeroed by every kernel
// that consumes it, so a task can be re-run without host-side clears.
struct SelScratch {
  uint32_t hist[kBins];
  uint32_t prefix;       // key bits fixed so far
  uint32_t pmask;        // which key bits are fixed
  int64_t rank;          // 1-based rank still to find inside the prefix
  int64_t cnt_gt;        // entries with key strictly above the prefix range
  int64_t total;         // entries in the input
  int64_t budget;        // effective budget for this run
  int32_t all;           // 1: total <= budget, all selected; 2: budget 0; 0: threshold
  int32_t mode;          // resolved input mode for this run
  int32_t cut_idx;       // largest selected index among entries with key == T
  int32_t pad_;
  // (phase stamps are compiled in only with -DSPARDL_STAMPS=1; zero otherwise)
  long long tstamp[12];  // phase timestamps (globaltimer ns) of the last run, CTA 0
  long long cta_ts[2][16];   // per CTA: start, end of the pass-0 histogram
  long long pro_ts[8];       // CTA 0: fused-merge prologue phase ends
  long long merge_ts[64];    // the feeding merge: 8 phase stamps of its partitions 0..7
};

// Membership in a finished selection without searching its output:
// selected  <=>  key > T  or  (key == T and index <= cut_idx).
__device__ __forceinline__ bool sel_member(const SelScratch* sc, uint32_t key, int32_t idx) {
  if (sc->all == 1) return true;
  if (sc->all == 2) return false;
  return key > sc->prefix || (key == sc->prefix && idx <= sc->cut_idx);
}

// Input is a list of segments.  mode 0 (explicit): segment s holds entries
// idx[off+j], val[off+j] for j < cnt with off = seg_off ? seg_off[s] : s*stride
// and cnt = seg_cnt ? seg_cnt[s] : clamp(*count - off, 0, stride) (a compact
// list cut into strided segments).  mode 1 (dense slice): entries are
// (dbase + p, dval[p]) for p in [s*dstride, min((s+1)*dstride, dn)).
// When `mode_from_cand` is set (the dividing select), the mode is decided on
// the device: explicit candidates if they are complete, else dense fallback.
struct SelTask {
  int32_t nseg;          // input segments (explicit mode)
  int32_t mode;
  int32_t mode_from_cand;
  int32_t stride;
  int32_t pad1_;
  int32_t pad2_;
  const int32_t* nseg_dev;  // nullable: segments actually in use (device-decided)
  const int32_t* idx;
  const float* val;
  const int32_t* seg_off;
  const int32_t* seg_cnt;
  const int32_t* count;
  // dense slice
  const float* dval;
  int32_t dbase;
  int32_t dn;
  int32_t dstride;
  int32_t dnseg;
  // candidate-path verdict (dividing)
  const int64_t* cand_total;
  const int32_t* cand_bad;
  struct DivHistory* div_hist;   // nullable: dividing select -> next pre-threshold
  unsigned long long* fallbacks; // nullable: += 1 per run that took the dense path
  const uint32_t* pre_key_dev;   // the pre-threshold of this run (dividing select)
  // budget
  int64_t budget;
  const int64_t* budget_dev;
  // outputs
  int32_t* sel_idx;
  float* sel_val;
  int32_t* sel_cnt;
  int32_t* dis_idx;      // nullable: discards are not materialised
  float* dis_val;
  int32_t* dis_cnt;
  float weight;          // discard share (inc/residual.hpp:104-124)
  int32_t sel_cap;       // capacity of sel_idx/sel_val (bounds checks; 0: unchecked)
  int32_t dis_cap;       // capacity of dis_idx/dis_val
  int32_t pad0_;
  int64_t* total_out;    // nullable: B-SAG union size N_t
  // scratch
  SelScratch* scr;
  int32_t* seg_gt;       // [sel_chunk_capacity] per work chunk
  int32_t* seg_eq;
  int32_t* seg_sel_off;
  int32_t* seg_dis_off;
  int32_t* seg_take;
  int32_t* seg_valid;    // entries per work item that are not merge holes
  // fused merge (nullable): the select first merges the r lists of *merge
  // itself, each cluster CTA one index range, into merge->out_* (idx/val
  // above), leaving a hole (kHoleKey) where equal indices were folded
  const struct MergeTask* merge;
  int32_t merge_slot;    // host bookkeeping: 1 + index of the stage's merge task, 0 none
  int32_t pad3_;
  PeerSync ps;           // waits on remote inputs, publishes the output
  // wide path (wselect.cu; nullable): the select spread over the whole GPU;
  // this kernel then only runs the tasks the wide path hands back
  WScratch* ws;
  // peer transport: copies of the selection written straight into the
  // buffers of the consumer ranks (slot layout: count, idx[push_cap],
  // val[push_cap]); npush = 0: none
  unsigned char* const* push_base;
  int32_t npush;
  int32_t push_cap;
};
constexpr int kMaxPush = 8;   // remote consumer ranks a select writes into

// ---------------------------------------------------------------------------
// Wide select (wselect.cu): one select task spread over the whole GPU.
// The task's input is cut into tiles (groups of `group` consecutive input
// segments).  Level 1: a 2048-bin histogram of the magnitude keys -- the full
// key range (bin = key >> 20) or a window (bin = (key - base) >> shift, past
// the window: `above`, under it: `below`) -- for the dividing select above
// its pre-threshold, for the others around the previous threshold.
// The bin holding the L-th key is located by every gather CTA; the gather
// pass collects that bin's entries (key, index, tile) and per-tile counts;
// the last gather CTA of the task selects the exact boundary entry inside
// the bin (radix select on key desc / index asc), fixes per-tile output
// offsets and the selection state; the write pass compacts every tile in
// index order.  A task the wide path cannot finish (window miss, bin buffer
// overflow, dividing candidates incomplete) is handed to k_select (state
// kWFallback), which also covers every input with merge holes.
constexpr int kWBins = 2048;
constexpr int kWFull = 0, kWWindow = 1, kWAuto = 2;       // histogram modes
// kWAuto (Spar-Reduce-Scatter / SAG selects): a window of 2048 bins of
// 2^kWAutoShift keys centred on the task's previous threshold (its
// SelScratch prefix, whichever path selected it), the full key range when
// there is none yet.  The merged lists concentrate in a narrow magnitude
// range, so full-range bins (1/8 octave) would hold a large share of them.
constexpr int kWAutoShift = 12;   // window = previous T +- 1/2 octave
constexpr int kWOk = 0, kWAll = 1, kWNone = 2, kWFallback = 3;   // run states
struct WScratch {
  // input: segments of the task (conventions of SelTask mode 0)
  const int32_t* idx;
  const float* val;
  const int32_t* seg_off;     // nullable: segment s starts at s * stride
  const int32_t* seg_cnt;     // nullable: clamp(*count - off, 0, stride)
  const int32_t* count;
  const int32_t* nseg_dev;    // nullable: segments in use
  int32_t stride;
  int32_t nseg;
  int32_t group;              // segments per tile
  int32_t max_tiles;
  int32_t mode;               // kWWindow (dividing: window set by k_div_prethr) / kWAuto
  int32_t is_div;             // dividing select (candidates + history)
  int32_t by_merge;           // the feeding merge histograms and decides (no hist pass)
  int32_t pad2_;
  // level-1 histogram (zeroed by the decider after use)
  uint32_t hist[kWBins];
  uint32_t above;             // window mode: keys past the last bin
  uint32_t below;             // window mode: keys below bin 0 (kWAuto; dividing: none)
  uint32_t base;              // dividing: lowest key of bin 0 (= pre-threshold), set by k_div_prethr
  uint32_t shift;             // dividing: log2 of the bin width in key units
  uint32_t harrive;           // histogram CTAs done (reset by the decider)
  uint32_t arrive;            // gather CTAs done (reset by the finisher)
  uint32_t wdone;             // write CTAs done (reset by the last writer)
  uint32_t bin_n;             // entries collected into the bin buffer
  int32_t state;              // kWOk / kWAll / kWNone / kWFallback of this run (decider)
  int32_t run_mode;           // this run's histogram geometry (decider, read by the gather)
  uint32_t run_base, run_shift;
  int32_t bstar;              // the level-1 bin holding the L-th key
  uint32_t bin_expect;        // its count
  long long before;           // entries in higher bins (and above the window)
  long long total_in;         // entries of the input this run
  uint32_t T;                 // threshold key of this run (kWOk; finisher)
  int32_t cut;                // largest selected index among key == T
  int32_t ntiles;             // tiles in use this run
  int32_t pad1_;
  long long total, total_sel; // entries, selected entries of this run
  // the bin buffer
  unsigned long long* bin_c;  // (key << 32) | (0x7fffffff - index): larger = earlier
  int32_t* bin_tile;
  int32_t bin_cap;
  int32_t pad_;
  // per tile: entries, selected (gather: above the bin; finisher: + in-bin),
  // exclusive output offsets of the selected / discarded entries
  int32_t* tile_n;
  int32_t* tile_sel;
  int32_t* tile_sel_off;
  int32_t* tile_dis_off;
  unsigned long long* handed_back;   // nullable: += 1 per run handed to k_select
  // cooperative form: entries past a CTA's shared-memory copy live here, at
  // their flat position in the task (nullable: such tasks are handed back)
  float* ov_val;
  int32_t* ov_idx;
  long long ov_cap;
};

// value bits of a merge hole: its magnitude key is kHoleKey, never a real
// entry's (a NaN with every mantissa bit set)
constexpr uint32_t kHoleBits = 0xffffffffu;
constexpr uint32_t kHoleKey = 0x7fffffffu;
constexpr int kMergeSamples = 2048;   // fused merge: splitter samples per task

// ---------------------------------------------------------------------------
// Merge
// ---------------------------------------------------------------------------
struct MergeTask {
  int32_t r;
  int32_t T;                        // window (sample spacing) per list
  PeerSync ps;                      // waits on remote input lists
  const int32_t* in_idx[kMaxR];
  const float* in_val[kMaxR];
  const int32_t* in_cnt[kMaxR];
  // device scratch written by the splitter kernel
  int32_t* splitters;               // [max_parts + 1]
  int32_t* windows;                 // [max_parts * r]
  int32_t* nparts;                  // [1]
  int32_t max_parts;
  int32_t pad_;
  // output: segmented list
  int32_t* out_idx;                 // capacity sum of input capacities
  float* out_val;
  int64_t out_cap;                  // capacity of out_idx/out_val (bounds checks)
  int32_t* seg_off;                 // [max_parts]
 int32_t* seg_cnt;                 // [max_parts]
  long long* dbg;                   // diagnostics: phase stamps of partitions 0..7, or null
  // the wide select consuming this merge (nullable): every partition CTA
  // histograms its output, the last one decides (wsel_common.cuh)
  WScratch* ws;
  const SelTask* sel;
};

// ---------------------------------------------------------------------------
// Dividing
// ---------------------------------------------------------------------------
// Pre-threshold carried between iterations: after a successful candidate
// run the dividing select stores next_pre = key(T' ) - delta (T: the exact
// L-th key it found; T' = T extrapolated linearly in magnitude from the
// previous run's threshold, for residuals that keep growing) and the next
// iteration skips the sample.  delta is re-fitted every run from the two
// points it observed -- (pre-threshold, candidates) and (T, L) -- so that
// the next candidate count is ~1.5 L (a secant step in log-count over key
// space).  A fallback to the dense path clears `valid`: the next iteration
// samples again.  Only the amount of work depends on it, never the result.
struct DivHistory {
  uint32_t next_pre;
  uint32_t delta;
  int32_t valid;
  uint32_t last_T;       // threshold of the previous run (valid when has_T)
  int32_t has_T;
  int32_t pad_;
};

struct DivTask {
  const float* const* g_tab;  // gradient pointer table (updated per call)
  int32_t g_id;            // this worker's entry in g_tab
  int32_t pad_;
  float* carry;            // worker residual; becomes g + carry (= g_copy) in place
  int32_t lo, hi;          // block range
  int32_t nchunks;
  int32_t cap;             // candidate capacity per chunk segment
  int64_t budget;          // L
  // candidates: one index-ordered segment per chunk, then a tile work list
  int32_t* cand_idx;       // [nchunks * cap]
  float* cand_val;
  int32_t* cand_cnt;       // [nchunks]
  int32_t* tile_off;       // [max_tiles] work list for the select (k_div_tiles)
  int32_t* tile_cnt;       // [max_tiles]
  int32_t max_tiles;
  int32_t tile_len;        // candidates per work-list tile (multiple of kTile)
  int32_t* ntiles;         // tiles in use (written by k_div_tiles)
  int64_t* cand_total;
  int32_t* cand_bad;       // bit 0: candidate path off for this run, bit 1: chunk overflow,
                           // bit 2: select work-list overflow (the wide select still applies),
                           // bit 3: candidates being redone (second chance, k_div_recand)
  uint32_t* pre_key;       // candidate threshold (key >= pre_key)
  uint32_t* samp_hist;     // [kSampBins]
  struct DivHistory* hist;  // threshold carried over from the previous iteration
  int32_t sample_every;    // sample one chunk in `sample_every`
  int32_t use_cand;        // 0: candidate path disabled (dense select)
  int32_t* err;            // NaN flag
  WScratch* ws;            // nullable: the wide select of this block (window histogram)
  int32_t ws_fused;        // k_div_cand histograms the candidates and decides (opt-in)
  int32_t huge;            // more chunks than select work items (wide select only)
  // deferred finalize (nullable): the previous iteration's records of this
  // block, applied to the carry before the gradient is added when *fin_apply
  const int32_t* rec_idx;
  const float* rec_v1;
  const float* rec_v2;
  const int32_t* chunk_off;
  const int32_t* fin_apply;
  const SelScratch* prev_sel; // the previous iteration's dividing selection (membership)
  unsigned long long* retries;  // nullable: += 1 per block whose candidates were redone
};

// ---------------------------------------------------------------------------
// Launchers (stream-ordered; no host synchronisation inside)
// They return the number of kernels launched; a failed launch is recorded
// per host thread (note_launch) and reported by take_launch_error(), which
// the engine checks after enqueueing an iteration.
void note_launch(cudaError_t e);
cudaError_t take_launch_error();
// ---------------------------------------------------------------------------
// tasks_dev: device copy of the task array; ntask; max_nseg: grid extent.
int launch_select(const SelTask* tasks_dev, int ntask, int max_nseg, cudaStream_t s,
                  int cluster = 0, int win_cap = 0);
// the wide path of a batch of selects (all tasks must carry ws): level-1
// histogram (skipped for dividing selects: k_div_cand fills it), gather +
// finisher, write; then launch_select for the tasks handed back
// the single-kernel cooperative form of the wide select (one wave of CTAs,
// task barriers in global memory); tasks that do not fit are handed back
int launch_wselect_coop(const SelTask* tasks_dev, int ntask, int max_nseg, cudaStream_t s);
int wsel_coop_words();               // uint32 words of its scratch (in the bin buffer)
int wsel_coop_max_seg();             // most input segments of a task
long long wsel_coop_capacity(int ntask, int max_nseg);   // entries per task that fit on this device
int launch_wselect(const SelTask* tasks_dev, int ntask, int max_tiles, bool histogram,
                   cudaStream_t s);
// fused merge+select: smem window capacity (entries) available per CTA, and
// the clusters of width cl resident at once for a launch with that window
int select_max_window();
int select_resident_clusters(int cl, int tab_cap, int win_cap);
int launch_merge(const MergeTask* tasks_dev, int ntask, int max_parts, int max_r_T, int max_r,
                 cudaStream_t s);
// part: 0 = whole pass, 1 = sample + pre-threshold only, 2 = candidate pass only
int launch_divide(const DivTask* tasks_dev, int ntask, int max_chunks, int sample_every,
                  int apply_residual, cudaStream_t s, int part = 0);

// Finalize / assembly helpers
struct GatherSrc {            // one source block of an assembled global gradient
  const int32_t* idx;
  const float* val;
  const int32_t* cnt;
};
struct AssembleTask {
  int32_t m;
  int32_t pad_;
  const GatherSrc* src;       // [m] (device)
  int32_t* out_idx;
  float* out_val;
  int32_t* out_cnt;
  int64_t* out_hash;          // nullable: FNV-style hash for consistency checks
  PeerSync ps;                // waits on remote source blocks
};
int launch_assemble(const AssembleTask* tasks_dev, int ntask, int max_m, int64_t max_k,
                    cudaStream_t s);

constexpr int kMaxXi = 24;
struct XiList {               // one in-procedure discard list (already weight-scaled)
  const int32_t* idx;
  const float* val;
  const int32_t* cnt;
};
// residual finalize for one worker (inc/residual.hpp:128-150)
struct FinalizeTask {
  int32_t mode;               // 0 gres, 1 pres, 2 lres
  int32_t m;                  // blocks
  int64_t n;                  // dimension
  float* carry;               // in: g_copy (combined); out: residual
  const GatherSrc* gblk;      // [m] the global gradient, block by block
  const SelScratch* const* div_sc;  // [m] dividing-select state (membership test)
  // per block: dividing selection + discard lists in recording order
  const GatherSrc* div;       // [m]
  const int32_t* xi_off;      // [m+1] offsets into xi
  const XiList* xi;           // lists
  // conservation audit (nullable): per position of the assembled global
  // gradient, this worker's combined value and final residual
  float* aud_comb;
  float* aud_carry;
  PeerSync ps;                // waits on the remote blocks of the global gradient
};

// Deferred residual finalize (gres): instead of a random read-modify-write
// of the carry at the k global positions at the end of an iteration, the
// finalize is written as records -- per global index j of block b, the
// in-procedure discard values of j in recording order (<= 2 lists per
// block; absent = kNoRec bits) -- and the next iteration's candidate pass,
// which streams the carry anyway, applies them chunk by chunk before it adds
// the gradient (inc/residual.hpp:128-150 evaluated at the next apply,
// inc/residual.hpp:63-71; same fold, same rounding).  Reading the carry in
// between (spardl_get_carry & co.) applies them first (k_fin_apply).
constexpr uint32_t kNoRec = 0x7fffffffu;   // a NaN: never a discard value
struct FinRecTask {           // one (local worker, block b)
  const int32_t* g_idx;       // the global gradient's block b
  const int32_t* g_cnt;
  XiList xl[2];               // the worker's discard lists of block b, recording order
  int32_t nxl;
  int32_t nchunks;            // chunks of the worker's dividing task of block b
  int64_t origin;             // its chunk origin (lo rounded down to 4)
  int32_t* rec_idx;           // [L] records, in global-gradient order
  float* rec_v1;
  float* rec_v2;
  int32_t* chunk_off;         // [nchunks + 1] first record of every chunk
  int32_t* rec_n;             // records written
  float* carry;               // (k_fin_apply) the worker's carry
  const SelScratch* div_sc;   // (k_fin_apply) its dividing selection of block b
  PeerSync ps;                // waits on remote blocks of the global gradient
};
int launch_fin_records(const FinRecTask* tasks_dev, int ntask, int64_t max_blk,
                       int32_t* apply_flag, cudaStream_t s);
// apply pending records to the carry in place (a reader between iterations)
int launch_fin_apply(const FinRecTask* tasks_dev, int ntask, int64_t max_blk,
                     int32_t* apply_flag, cudaStream_t s);
// abort (nullable): the peer-timeout flag; when set the persistent-state
// writers (finalize, ledger, controller) leave their state untouched
int launch_finalize(const FinalizeTask* tasks_dev, int ntask, int64_t max_blk, int m,
                    int max_div, const int32_t* abort, cudaStream_t s);

// ledger: scalars += 2 * count for each (worker slot, count pointer)
struct LedgerAdd {
  int64_t* dst;
  const int32_t* cnt;
};
int launch_ledger(const LedgerAdd* adds_dev, int nadd, const int32_t* abort, cudaStream_t s);

// B-SAG controller (Algorithm 2, inc/sag.hpp:37-90) on the device
struct HCtl {
  double lower, upper;
  int64_t target;
  double h, step;
  int32_t flag;
  int32_t pad_;
};
struct CtlTask {
  HCtl* ctl;                  // this worker's controller
  const int64_t* n_t;         // its group's union size
  int64_t* budget;            // pre-selection budget for the next run
};
int launch_controller(const CtlTask* tasks_dev, int ntask, int observe, const int32_t* abort,
                      cudaStream_t s);

// fp64 components of the C++ drop-in surface (components64.cu)
int launch_topk64(const int64_t* idx, const double* val, int n, long long budget, uint8_t* flag,
                  cudaStream_t s);
int launch_merge64(const int64_t* ai, const double* av, int na, const int64_t* bi,
                   const double* bv, int nb, int64_t* ti, double* tv, int64_t* oi, double* ov,
                   int64_t* no, cudaStream_t s);

// peer-memory transport (transport.cu): iteration epoch, readiness flags
int launch_begin(long long* epoch, const long long* const* done, int n, int32_t* err,
                 unsigned long long timeout_ns, cudaStream_t s);
int launch_publish(long long* const* targets, int n, const long long* epoch, cudaStream_t s);

}  // namespace sdl
