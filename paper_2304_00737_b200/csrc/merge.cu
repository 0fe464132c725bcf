// r-way index merge with a left fold of the values in list order.
//
// Semantics: acc = l0; for t in 1..r-1: acc = merge_add(acc, l_t)
// (inc/sparse.hpp:182-208, applied as the reference applies it: SRS merges
// received blocks into the held block in arrival order,
// inc/reduce_scatter.hpp:190-202; B-SAG folds the gathered blocks in source
// rank order, inc/sag.hpp:231-236).  For an index present in several lists
// the value is ((v_a + v_b) + v_c) ... in list order -- every add is one
// IEEE round-to-nearest fp32 add (__fadd_rn, never contracted).
//
// Partitioning: every T-th entry of every list is a splitter.  Between two
// consecutive splitters each list contributes at most T entries, all inside
// one "window" of T consecutive entries of that list, so a CTA merges its
// partition from <= r windows staged in shared memory.  The partition output
// is written at the partition's position in concatenation space, so the
// result is a segmented list (one segment per partition, gaps where indices
// coincided) that the select kernels consume directly.
#include <algorithm>
#include <climits>
#include <cstdlib>

#include <mutex>

#include "common.cuh"
#include "kernels.cuh"
#include "wsel_common.cuh"

namespace sdl {

namespace {

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const size_t ga = __cvta_generic_to_global(gmem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(ga) : "memory");
}

// Rank all samples of a task; write the sorted splitters and, for each
// splitter, the window of every list that can hold its partition.
__global__ void __launch_bounds__(kThreads) k_merge_rank(const MergeTask* __restrict__ tasks) {
  pdl_enter();
  const MergeTask& t = tasks[blockIdx.y];
  peer_wait(t.ps);   // remote input lists published (k_merge_part follows in order)
  const int r = t.r, T = t.T;
  __shared__ int32_t samp[kMaxSamples];
  __shared__ int base[kMaxR + 1];
  if (threadIdx.x == 0) {
    int b = 0;
    for (int l = 0; l < r; ++l) {
      const int n = *t.in_cnt[l];
      base[l] = b;
      b += (n + T - 1) / T;
    }
    base[r] = b;
  }
  __syncthreads();
  const int S = base[r];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    t.splitters[S] = INT_MAX;
    *t.nparts = S;
  }
  if ((int)(blockIdx.x * blockDim.x) >= S) return;
  for (int q = threadIdx.x; q < S; q += blockDim.x) {
    int l = 0;
    while (q >= base[l + 1]) ++l;
    samp[q] = t.in_idx[l][(q - base[l]) * T];
  }
  __syncthreads();
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < S; q += gridDim.x * blockDim.x) {
    int l = 0;
    while (q >= base[l + 1]) ++l;
    const int j = q - base[l];
    const int32_t v = samp[q];
    int rank = j;
    int win[kMaxR];
    for (int u = 0; u < r; ++u) {
      if (u == l) {
        win[u] = j;
        continue;
      }
      const int32_t* a = samp + base[u];
      const int n = base[u + 1] - base[u];
      const int ub = upper_bound_i32(a, n, v);
      win[u] = ub - 1;
      rank += (u < l) ? ub : lower_bound_i32(a, n, v);
    }
    t.splitters[rank] = v;
    for (int u = 0; u < r; ++u) t.windows[(size_t)rank * r + u] = win[u];
  }
}

#ifndef SPARDL_MERGE_THREADS
#define SPARDL_MERGE_THREADS 256
#endif
constexpr int kMergeThreads = SPARDL_MERGE_THREADS;   // threads per partition CTA
#ifndef SPARDL_MERGE_MINB
#define SPARDL_MERGE_MINB 6   // 6 CTAs per SM (<= 42 registers): fewer waves for r >= 4
#endif
#ifndef SPARDL_MERGE_PATH_MAXR   // widest merge folded by merge-path passes (else rank scatter)
#define SPARDL_MERGE_PATH_MAXR 3
#endif
#ifndef SPARDL_MERGE_PATH_MINB   // merge-path variant (6: <= 42 registers, no spills; C4 SRS 0.773 -> 0.759 ms; 8 spills)
#define SPARDL_MERGE_PATH_MINB 6
#endif

__device__ __forceinline__ void mstamp(const MergeTask& t, int q, int k) {
  if (SPARDL_STAMPS && t.dbg && q < 8 && threadIdx.x == 0) {
    long long ts;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts));
    t.dbg[q * 8 + k] = ts;
  }
}

// Entries of one 2-way merge pass: A (the fold so far) and B (the next
// list), both ascending in index; equal indices are folded acc + next.
struct Run {
  const int32_t* idx;
  const float* val;
  int n;
};

// One merge-path pass over the CTA: thread t owns the merged positions
// [t*E, (t+1)*E) (ties: A first), finds its start with one binary search and
// merges sequentially.  An index present in both A and B is one output,
// folded by whichever thread owns its A entry (the next thread skips the B
// entry).  Returns the output count; writes idx/val at out + rank.
__device__ __forceinline__ int merge_pass(Run A, Run B, int32_t* out_idx, float* out_val,
                                          int* scratch) {
  const int n = A.n + B.n;
  const int E = (n + kMergeThreads - 1) / kMergeThreads;
  const int d0 = min(n, (int)threadIdx.x * E), d1 = min(n, d0 + E);
  // co-rank: i = #A among the first d0 merged entries
  int lo = max(0, d0 - B.n), hi = min(d0, A.n);
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (A.idx[mid] <= B.idx[d0 - 1 - mid]) lo = mid + 1;
    else hi = mid;
  }
  const int i0 = lo, j0 = d0 - lo;
  // the first entry is B's half of a fold the previous thread owns
  const bool skip_first = d0 < d1 && j0 < B.n && i0 > 0 && (i0 == A.n || B.idx[j0] < A.idx[i0]) &&
                          A.idx[i0 - 1] == B.idx[j0];
  // sweep 1: count outputs (a fold consumes two merged positions)
  int cnt = 0;
  {
    int i = i0, j = j0;
    bool first = true;
    while (i + j < d1) {
      const bool take_a = j >= B.n || (i < A.n && A.idx[i] <= B.idx[j]);
      if (take_a) {
        if (j < B.n && B.idx[j] == A.idx[i]) ++j;   // folded partner, maybe past d1
        ++i;
        ++cnt;
      } else {
        if (!(first && skip_first)) ++cnt;
        ++j;
      }
      first = false;
    }
  }
  int total;
  const int base = block_exscan(cnt, scratch, &total);
  // sweep 2: write
  {
    int i = i0, j = j0, o = base;
    bool first = true;
    while (i + j < d1) {
      const bool take_a = j >= B.n || (i < A.n && A.idx[i] <= B.idx[j]);
      if (take_a) {
        const int32_t x = A.idx[i];
        float v = A.val[i];
        if (j < B.n && B.idx[j] == x) v = __fadd_rn(v, B.val[j++]);
        ++i;
        out_idx[o] = x;
        out_val[o] = v;
        ++o;
      } else {
        if (!(first && skip_first)) {
          out_idx[o] = B.idx[j];
          out_val[o] = B.val[j];
          ++o;
        }
        ++j;
      }
      first = false;
    }
  }
  __syncthreads();   // outputs visible before they are read as the next A
  return total;
}

// Merge of partition q: entries with v_lo <= index < v_hi, from list l's
// window win[l] (-1: none).
template <bool PATH>
__device__ __forceinline__ void merge_body(const MergeTask& t, int q, int32_t v_lo, int32_t v_hi,
                                           const int* win) {
  const int r = t.r, T = t.T;
  extern __shared__ __align__(16) unsigned char smem[];
  int32_t* w_idx = reinterpret_cast<int32_t*>(smem);          // [r*T]
  float* w_val = reinterpret_cast<float*>(w_idx + r * T);      // [r*T]
  int32_t* m_idx = reinterpret_cast<int32_t*>(w_val + r * T);  // [r*T]
  float* m_val = reinterpret_cast<float*>(m_idx + r * T);      // [r*T]
  __shared__ int wlen[kMaxR], wstart[kMaxR], a_[kMaxR], b_[kMaxR], sz_pref[kMaxR + 1];
  __shared__ int seg_base;
  __shared__ int scratch[40];
  if (threadIdx.x < r) {
    const int l = threadIdx.x;
    const int w = win[l];
    const int n = *t.in_cnt[l];
    if (w < 0) {
      wstart[l] = 0;
      wlen[l] = 0;
    } else {
      wstart[l] = w * T;
      const int rem = n - w * T;
      wlen[l] = rem < T ? rem : T;
    }
  }
  __syncthreads();
  // stage the windows with asynchronous 16-byte copies: every thread issues
  // all of its copies before waiting once (16-byte aligned windows: block
  // buffers are, and T % 4 == 0); the < 4-entry tail and unaligned lists
  // (component API inputs) are copied with plain loads
  for (int l = 0; l < r; ++l) {
    const int32_t* gi = t.in_idx[l] + wstart[l];
    const float* gv = t.in_val[l] + wstart[l];
    const bool al = ((reinterpret_cast<uintptr_t>(gi) | reinterpret_cast<uintptr_t>(gv)) & 15) == 0;
    const int n4 = al ? (wlen[l] >> 2) : 0;
    for (int j = threadIdx.x; j < n4; j += blockDim.x) {
      cp_async16(w_idx + l * T + 4 * j, gi + 4 * j);
      cp_async16(w_val + l * T + 4 * j, gv + 4 * j);
    }
    for (int j = 4 * n4 + threadIdx.x; j < wlen[l]; j += blockDim.x) {
      w_idx[l * T + j] = gi[j];
      w_val[l * T + j] = gv[j];
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  mstamp(t, q, 4);
  if (threadIdx.x < r) {
    const int l = threadIdx.x;
    a_[l] = lower_bound_i32(w_idx + l * T, wlen[l], v_lo);
    b_[l] = lower_bound_i32(w_idx + l * T, wlen[l], v_hi);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0, base = 0;
    for (int l = 0; l < r; ++l) {
      sz_pref[l] = s;
      s += b_[l] - a_[l];
      base += wstart[l] + a_[l];
    }
    sz_pref[r] = s;
    seg_base = base;
  }
  __syncthreads();
  mstamp(t, q, 5);
  if constexpr (PATH) {
    // left fold ((l0 + l1) + l2) + ... as r-1 merge-path passes; the last
    // pass writes the segment, the others ping-pong between two buffers
    int32_t* const q_idx = reinterpret_cast<int32_t*>(m_val + r * T);   // second buffer
    float* const q_val = reinterpret_cast<float*>(q_idx + r * T);
    SPARDL_BOUND(seg_base + sz_pref[r] - 1, t.out_cap + (sz_pref[r] == 0));
    Run acc{w_idx + a_[0], w_val + a_[0], b_[0] - a_[0]};
    int out = acc.n;
    if (r == 1) {
      for (int e = threadIdx.x; e < acc.n; e += blockDim.x) {
        SPARDL_BOUND(seg_base + e, t.out_cap);
        t.out_idx[seg_base + e] = acc.idx[e];
        t.out_val[seg_base + e] = acc.val[e];
      }
    }
    for (int u = 1; u < r; ++u) {
      const Run B{w_idx + u * T + a_[u], w_val + u * T + a_[u], b_[u] - a_[u]};
      const bool last = u == r - 1;
      int32_t* oi = last ? t.out_idx + seg_base : ((u & 1) ? m_idx : q_idx);
      float* ov = last ? t.out_val + seg_base : ((u & 1) ? m_val : q_val);
      out = merge_pass(acc, B, oi, ov, scratch);
      acc = Run{oi, ov, out};
    }
    if (threadIdx.x == 0) {
      t.seg_off[q] = seg_base;
      t.seg_cnt[q] = out;
    }
    mstamp(t, q, 6);
    return;
  }
  const int M = sz_pref[r];
  // stable r-way merge by (index, list): scatter every entry to its rank
  for (int e = threadIdx.x; e < M; e += blockDim.x) {
    int l = 0;
    while (e >= sz_pref[l + 1]) ++l;
    const int i = a_[l] + (e - sz_pref[l]);
    const int32_t x = w_idx[l * T + i];
    int pos = i - a_[l];
    for (int u = 0; u < r; ++u) {
      if (u == l) continue;
      const int32_t* a = w_idx + u * T + a_[u];
      const int n = b_[u] - a_[u];
      pos += (u < l) ? upper_bound_i32(a, n, x) : lower_bound_i32(a, n, x);
    }
    m_idx[pos] = x;
    m_val[pos] = w_val[l * T + i];
  }
  __syncthreads();
  // fold runs of equal index (at most r long, in list order) and compact
  int out = 0;
  for (int e0 = 0; e0 < M; e0 += blockDim.x) {
    const int e = e0 + threadIdx.x;
    const bool head = e < M && (e == 0 || m_idx[e] != m_idx[e - 1]);
    int tot;
    const int rk = out + block_rank(head, scratch, &tot);
    if (head) {
      const int32_t x = m_idx[e];
      float acc = m_val[e];
      for (int f = e + 1; f < M && m_idx[f] == x; ++f) acc = __fadd_rn(acc, m_val[f]);
      SPARDL_BOUND(seg_base + rk, t.out_cap);
      t.out_idx[seg_base + rk] = x;
      t.out_val[seg_base + rk] = acc;
    }
    out += tot;
  }
  if (threadIdx.x == 0) {
    t.seg_off[q] = seg_base;
    t.seg_cnt[q] = out;
  }
}

template <bool PATH>
__device__ __forceinline__ void merge_part_body(const MergeTask& t, int q) {
  const int S = *t.nparts;
  if (q >= t.max_parts) return;
  if (q >= S) {
    if (threadIdx.x == 0) {
      t.seg_off[q] = 0;
      t.seg_cnt[q] = 0;
    }
    return;
  }
  const int32_t v_lo = t.splitters[q];
  const int32_t v_hi = t.splitters[q + 1];
  if (v_lo == v_hi) {
    if (threadIdx.x == 0) {
      t.seg_off[q] = 0;
      t.seg_cnt[q] = 0;
    }
    return;
  }
  __shared__ int win[kMaxR];
  if (threadIdx.x < t.r) win[threadIdx.x] = t.windows[(size_t)q * t.r + threadIdx.x];
  __syncthreads();
  merge_body<PATH>(t, q, v_lo, v_hi, win);
}

// One kernel per merge batch when the splitter samples are few (<= 4 per
// thread): every partition CTA loads all samples of its task, ranks them in
// shared memory and takes its own splitters and windows -- the ranking that
// k_merge_rank does once, repeated per CTA, instead of a kernel boundary and
// two more dependent global round trips.
constexpr int kOneShotSamples = 4 * kMergeThreads;

template <bool PATH>
__device__ __forceinline__ void merge_one_body(const MergeTask& t, int q) {
  if (q >= t.max_parts) return;
  mstamp(t, q, 0);
  peer_wait(t.ps);   // remote input lists published
  const int r = t.r, T = t.T;
  __shared__ int base[kMaxR + 1];
  __shared__ int32_t samp[kOneShotSamples];
  __shared__ int win[kMaxR];
  __shared__ int32_t s_lo, s_hi;
  if (threadIdx.x < r) base[threadIdx.x + 1] = *t.in_cnt[threadIdx.x];
  __syncthreads();
  if (threadIdx.x == 0) {
    int b = 0;
    base[0] = 0;
    for (int l = 0; l < r; ++l) {
      const int n = base[l + 1];
      b += (n + T - 1) / T;
      base[l + 1] = b;
    }
    s_lo = INT_MIN;
    s_hi = INT_MAX;   // the last partition is open above
  }
  __syncthreads();
  mstamp(t, q, 1);
  const int S = base[r];
  if (q >= S) {
    if (threadIdx.x == 0) {
      t.seg_off[q] = 0;
      t.seg_cnt[q] = 0;
    }
    return;
  }
  for (int i = threadIdx.x; i < S; i += kMergeThreads) {
    int l = 0;
    while (i >= base[l + 1]) ++l;
    samp[i] = t.in_idx[l][(i - base[l]) * T];
  }
  __syncthreads();
  mstamp(t, q, 2);
  // rank every sample (ties: list order); keep the splitters of ranks q, q+1
  for (int i = threadIdx.x; i < S; i += kMergeThreads) {
    int l = 0;
    while (i >= base[l + 1]) ++l;
    const int j = i - base[l];
    const int32_t v = samp[i];
    int rank = j;
    for (int u = 0; u < r; ++u) {
      if (u == l) continue;
      const int32_t* a = samp + base[u];
      const int n = base[u + 1] - base[u];
      rank += (u < l) ? upper_bound_i32(a, n, v) : lower_bound_i32(a, n, v);
    }
    if (rank == q) {
      s_lo = v;
      for (int u = 0; u < r; ++u)
        win[u] = u == l ? j : upper_bound_i32(samp + base[u], base[u + 1] - base[u], v) - 1;
    } else if (rank == q + 1) {
      s_hi = v;
    }
  }
  __syncthreads();
  mstamp(t, q, 3);
  const int32_t v_lo = s_lo, v_hi = s_hi;
  if (v_lo == v_hi) {
    if (threadIdx.x == 0) {
      t.seg_off[q] = 0;
      t.seg_cnt[q] = 0;
    }
    return;
  }
  merge_body<PATH>(t, q, v_lo, v_hi, win);
}

static_assert(kMergeThreads == kWDecideThreads, "the merge CTA runs the wide-select decider");

// The consuming wide select's level-1 histogram (MergeTask::ws): every
// partition CTA histograms the segment it just wrote (shared bins, one
// flush); the CTA completing the task decides the select's run.  Every CTA
// of the grid arrives, with or without a partition.
__device__ void merge_wsel_epilogue(const MergeTask& t, int q) {
  WScratch* ws = t.ws;
  const SelTask& ts = *t.sel;
  int mode;
  uint32_t base, shift;
  w_geometry(ts, *ws, mode, base, shift);
  __shared__ uint32_t h[kWBins];
  __shared__ uint32_t s_ab[2];
  __shared__ int s_last;
  __shared__ int scratch[40];
  __shared__ long long lsh[3 * 32];
  for (int b = threadIdx.x; b < kWBins; b += kMergeThreads) h[b] = 0;
  if (threadIdx.x < 2) s_ab[threadIdx.x] = 0;
  __syncthreads();   // (and the segment written by this CTA is visible to it)
  uint32_t nb = 0, na = 0;
  if (q < t.max_parts) {
    const int off = t.seg_off[q], cnt = t.seg_cnt[q];
    for (int j = threadIdx.x; j < cnt; j += kMergeThreads) {
      const int b = w_bin(mode, base, shift, mag_key(t.out_val[off + j]));
      if (b < 0) ++nb;
      else if (b >= kWBins) ++na;
      else atomicAdd(&h[b], 1u);
    }
  }
  nb = __reduce_add_sync(0xffffffffu, nb);
  na = __reduce_add_sync(0xffffffffu, na);
  if ((threadIdx.x & 31) == 0 && (nb | na)) {
    atomicAdd(&s_ab[0], nb);
    atomicAdd(&s_ab[1], na);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < kWBins; b += kMergeThreads)
    if (h[b]) atomicAdd(&ws->hist[b], h[b]);
  if (threadIdx.x == 0) {
    if (s_ab[0]) atomicAdd(&ws->below, s_ab[0]);
    if (s_ab[1]) atomicAdd(&ws->above, s_ab[1]);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = (int)(atomicAdd(&ws->harrive, 1u) == gridDim.y - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int64_t budget = ts.budget_dev ? *ts.budget_dev : ts.budget;
  const long long total = w_hist_total(ws, lsh) + __ldcg(&ws->above) + __ldcg(&ws->below);
  w_decide(ws, total, false, budget, mode, base, shift, scratch, lsh);
}

// grid (task, partition): partitions of every task come first in launch
// order, so the live ones (q < nparts, usually far fewer than max_parts)
// all start in the first wave
template <bool PATH>
__global__ void __launch_bounds__(kMergeThreads, PATH ? SPARDL_MERGE_PATH_MINB : SPARDL_MERGE_MINB) k_merge_part(const MergeTask* __restrict__ tasks) {
  pdl_enter();
  const MergeTask& t = tasks[blockIdx.x];
  merge_part_body<PATH>(t, blockIdx.y);
  if (t.ws) merge_wsel_epilogue(t, blockIdx.y);
}

template <bool PATH>
__global__ void __launch_bounds__(kMergeThreads, PATH ? SPARDL_MERGE_PATH_MINB : SPARDL_MERGE_MINB) k_merge_one(const MergeTask* __restrict__ tasks) {
  pdl_enter();
  const MergeTask& t = tasks[blockIdx.x];
  merge_one_body<PATH>(t, blockIdx.y);
  if (t.ws) merge_wsel_epilogue(t, blockIdx.y);
}

bool merge_path_on() {
  static const bool on = [] {
    const char* e = getenv("SPARDL_MERGE_PATH");   // tuning experiments only
    return !(e && e[0] == '0');
  }();
  return on;
}

bool merge_one_shot() {
  static const bool on = [] {
    const char* e = getenv("SPARDL_MERGE_ONESHOT");   // tuning experiments only
    return !(e && e[0] == '0');
  }();
  return on;
}

}  // namespace

int launch_merge(const MergeTask* tasks_dev, int ntask, int max_parts, int max_r_T, int max_r,
                 cudaStream_t s) {
  if (ntask <= 0 || max_parts <= 0) return 0;
  // merge-path folds: the windows plus one intermediate buffer for r = 3 and
  // two for r >= 4 (8 B per window entry each; r = 2 writes straight to the
  // output, so a CTA needs 16 KB and the whole batch fits one wave); the
  // rank-scatter fallback 16 B per entry
  const size_t path_bytes = (size_t)max_r_T * 8 * (1 + std::min(std::max(max_r - 2, 0), 2));
  // (r >= 4: two intermediates cost more occupancy than the rank scatter)
  const bool path = merge_path_on() && max_r <= SPARDL_MERGE_PATH_MAXR && path_bytes <= 200 * 1024;
  const size_t smem = path ? path_bytes : (size_t)max_r_T * 16;
  const bool one = max_parts <= kOneShotSamples && merge_one_shot();
  auto part = path ? k_merge_part<true> : k_merge_part<false>;
  auto single = path ? k_merge_one<true> : k_merge_one<false>;
  // (dynamic + static shared memory above 48 KB needs the opt-in)
  static std::mutex mu;
  static size_t configured[kMaxDevices][2][2] = {};   // per device
  {
    const int dev = cur_device();
    std::lock_guard<std::mutex> lock(mu);
    if (smem > configured[dev][path][one]) {
      cudaFuncSetAttribute(one ? single : part, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem);
      configured[dev][path][one] = smem;
    }
  }
  if (one) {
    launch_pdl(single, dim3(ntask, max_parts), dim3(kMergeThreads), smem, s, tasks_dev);
    return 1;
  }
  const int rx = (max_parts + kThreads - 1) / kThreads;
  launch_pdl(k_merge_rank, dim3(rx, ntask), dim3(kThreads), 0, s, tasks_dev);
  launch_pdl(part, dim3(ntask, max_parts), dim3(kMergeThreads), smem, s, tasks_dev);
  return 2;
}

}  // namespace sdl
