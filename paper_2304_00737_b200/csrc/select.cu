// Deterministic top-L selection over segmented sparse lists -- one kernel.
//
// Semantics: inc/sparse.hpp:136-162 (top_k_select) -- keep the min(budget,
// nnz) entries that come first in the order (|v| desc, index asc); return
// the kept and the discarded entries, each in index order.
//
// Method: one thread-block cluster of kCl CTAs per task (Blackwell clusters,
// distributed shared memory).  Every CTA owns a contiguous range of the
// task's segments (segments are in index order, so CTA order == index order).
//   1. counts: CTA totals exchanged through DSMEM -> total, identity case.
//   2. radix select on the 31-bit magnitude key, digits 11/11/9 bits: each
//      CTA histograms its entries matching the current prefix in shared
//      memory and sums them into 32-bin super-bins; after ONE cluster barrier
//      every CTA reads the CL super-bin histograms through DSMEM, finds the
//      super-bin holding the rank-th largest key, reads the CL copies of its
//      32 bins and finds the digit itself (identical data, no leader, no
//      global atomics, no kernel boundaries; histograms double-buffered
//      across passes).  The previous run's top digit is tried first.  After
//      the passes the threshold key T is exact, and need_eq = L - #{key > T}
//      entries of key T are kept: the lowest-index ones (the reference's tie
//      rule).
//   3. per segment (one warp each) #{key > T}, #{key == T}; CTA totals go
//      through DSMEM so every CTA knows the tie quota and the output offsets
//      of the CTAs before it; a CTA-wide scan places each segment.
//   4. ordered compaction with warp ballots of the selected entries and of
//      the discarded ones, the latter scaled by the residual share with an
//      explicitly rounded multiply (no FMA contraction, inc/residual.hpp:119).
#include <cooperative_groups.h>

#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>

#include <mutex>

#include "common.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace sdl {

namespace {

constexpr int kSelThreads = 512;   // 16 warps per CTA
#ifndef SPARDL_SEL_MINB
#define SPARDL_SEL_MINB 1
#endif
constexpr int kWarps = kSelThreads / 32;
#ifndef SPARDL_SEL_ILP
#define SPARDL_SEL_ILP 4
#endif
constexpr int kIlp = SPARDL_SEL_ILP;   // 32-entry groups loaded per warp step (memory-level parallelism)
constexpr int kChunkE = 32 * kIlp;   // flat entries per work chunk (one warp step)
// wide clusters (>= 6 CTAs: the Spar-Reduce-Scatter / SAG batches of 8-16
// selections of 2-4 L merged entries, mostly past the on-chip copy) keep
// twice as many loads in flight per warp; measured on B200 at C4 (one GPU):
// SRS 0.808 -> 0.773 ms, while the 2-wide dividing selects lose with 8
#ifndef SPARDL_SEL_ILP_WIDE
#define SPARDL_SEL_ILP_WIDE 8
#endif

__device__ __forceinline__ int resolve_mode(const SelTask& t) {
  if (!t.mode_from_cand) return t.mode;
  const int64_t need = t.budget_dev ? *t.budget_dev : t.budget;
  return (*t.cand_bad != 0 || *t.cand_total < need) ? 1 : 0;
}

// segments actually in use (the planner sizes nseg for the worst case)
__device__ __forceinline__ int nseg_of(const SelTask& t, int mode) {
  if (mode == 1) return t.dnseg;
  if (t.nseg_dev) return min(*t.nseg_dev, t.nseg);
  if (!t.seg_cnt) return min(t.nseg, (*t.count + t.stride - 1) / t.stride);
  return t.nseg;
}

// segment s: entries [off, off + cnt) of the task's input
__device__ __forceinline__ void seg_bounds(const SelTask& t, int mode, int s, int& off,
                                           int& cnt) {
  int c;
  if (mode == 1) {
    off = s * t.dstride;
    c = t.dn - off;
    c = c > t.dstride ? t.dstride : c;
  } else {
    off = t.seg_off ? t.seg_off[s] : s * t.stride;
    c = t.seg_cnt ? t.seg_cnt[s] : *t.count - off;
    c = c > t.stride ? t.stride : c;
  }
  cnt = c < 0 ? 0 : c;
}

// shared-memory histogram increment (the keys of a warp spread over many bins,
// so plain shared atomics beat warp aggregation with match.any)
__device__ __forceinline__ void hist_add(uint32_t* h, uint32_t bin, bool active) {
  if (active) atomicAdd(&h[bin], 1u);
}

struct RadixState {     // lives in CTA 0, read by the cluster through DSMEM
  uint32_t prefix;
  uint32_t pmask;
  int64_t rank;         // rank still to find inside the prefix
  int64_t total;
  int64_t budget;
  int32_t all;          // 1: everything kept, 2: nothing kept, 0: threshold
  int32_t hit;          // the guessed top digit held the rank
};

struct CtaTotals {      // per-CTA counters exchanged through DSMEM
  long long cnt, gt, eq;
};

__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const size_t ga = __cvta_generic_to_global(gmem);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(ga) : "memory");
}

__device__ __forceinline__ int32_t lds_i32(unsigned addr) {
  int32_t v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(addr));
  return v;
}

// list holding position p of a concatenation with list starts base[0..r]
__device__ __forceinline__ int list_of(const int* base, int r, int p) {
  int l = 0;
  while (l + 1 < r && p >= base[l + 1]) ++l;
  return l;
}

// Fused merge (inc/sparse.hpp:182-208 folded left over the lists, as in
// merge.cu) of one cluster CTA's index range.  The task's lists are cut at
// union splitter samples (every Ts-th entry of every list): CTA cr takes the
// index range between the samples of union rank S*cr/CL and S*(cr+1)/CL, so
// equal indices never straddle two CTAs and each CTA holds at most
// sum/CL + (2r + 2) Ts entries.  Its windows are staged in shared memory and
// every entry is written at its stable merged rank inside the CTA's output
// range [sum of window starts, + window size): the first entry of an index
// (lowest list) carries the fold in list order, later copies become holes.
// Builds the CTA's work items and returns the task's merged total.
template <int CL>
__device__ long long merge_prologue(const MergeTask& mt, int cr, int32_t* w_idx, float* w_val,
                                    int32_t* samp, int win_cap, int32_t* iof, int32_t* ilen,
                                    int tab_cap, int& s_F, int& s_before, int& s_nit,
                                    long long* lscr, CtaTotals* tot,
                                    cg::cluster_group& cluster, SelScratch* sc) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  auto pstamp = [&](int i) {
    if (SPARDL_STAMPS && cr == 0 && tid == 0) {
      long long ts;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts));
      sc->pro_ts[i] = ts;
    }
  };
  const int r = mt.r, Ts = mt.T;
  __shared__ int ncnt[kMaxR], sb[kMaxR + 1], lo_q[kMaxR], hi_q[kMaxR], wb[kMaxR + 1];
  __shared__ int32_t vb[2];
  __shared__ int s_base, s_nin;
  if (tid < r) ncnt[tid] = *mt.in_cnt[tid];
  if (tid == 0) {
    vb[0] = INT_MIN;
    vb[1] = INT_MAX;
  }
  __syncthreads();
  if (tid == 0) {
    int S = 0;
    for (int q = 0; q < r; ++q) {
      sb[q] = S;
      S += (ncnt[q] + Ts - 1) / Ts;
    }
    sb[r] = S;
  }
  __syncthreads();
  const int S = sb[r];
  pstamp(0);
  // samples: every Ts-th index of every list
  for (int i = tid; i < S; i += kSelThreads) {
    const int q = list_of(sb, r, i);
    samp[i] = mt.in_idx[q][(size_t)(i - sb[q]) * Ts];
  }
  __syncthreads();
  pstamp(1);
  // the two splitters of this CTA: samples of union rank S*cr/CL, S*(cr+1)/CL
  // (ties ordered by list, as the merge orders equal indices)
  const int rlo = (int)((long long)S * cr / CL), rhi = (int)((long long)S * (cr + 1) / CL);
  for (int i = tid; i < S; i += kSelThreads) {
    const int q = list_of(sb, r, i);
    const int32_t v = samp[i];
    int rank = i - sb[q];
    for (int u = 0; u < r; ++u) {
      if (u == q) continue;
      const int n = sb[u + 1] - sb[u];
      rank += u < q ? upper_bound_i32(samp + sb[u], n, v) : lower_bound_i32(samp + sb[u], n, v);
    }
    if (cr > 0 && rank == rlo) vb[0] = v;
    if (rank == rhi) vb[1] = v;   // rhi == S (last CTA) matches no sample: stays +inf
  }
  __syncthreads();
  pstamp(2);
  // window bounds: lower_bound of each splitter in each list, bracketed by
  // the list's own samples to < Ts entries (one warp per bound)
  for (int p = warp; p < 2 * r; p += kWarps) {
    const int q = p >> 1;
    const int32_t v = vb[p & 1];
    const int n = ncnt[q];
    int pos;
    if (v == INT_MIN) {
      pos = 0;
    } else if (v == INT_MAX) {
      pos = n;
    } else {
      const int c = lower_bound_i32(samp + sb[q], sb[q + 1] - sb[q], v);   // samples < v
      const int lo = c == 0 ? 0 : (c - 1) * Ts + 1;
      const int hi = min(c * Ts, n);
      int cnt = 0;
      for (int j = lo + lane; j < hi; j += 32) cnt += mt.in_idx[q][j] < v;
      pos = lo + __reduce_add_sync(0xffffffffu, cnt);
    }
    if (lane == 0) (p & 1 ? hi_q : lo_q)[q] = pos;
  }
  __syncthreads();
  if (tid == 0) {
    int w = 0, base = 0;
    for (int q = 0; q < r; ++q) {
      wb[q] = w;
      w += max(0, hi_q[q] - lo_q[q]);
      base += lo_q[q];
    }
    wb[r] = w;
    s_base = base;
    s_nin = min(w, win_cap);   // the planner sizes win_cap so this never clips
  }
  __syncthreads();
  const int nin = s_nin, base = s_base;
  pstamp(3);
  // stage the windows (asynchronous copies, one wait)
  for (int e = tid; e < nin; e += kSelThreads) {
    const int q = list_of(wb, r, e);
    const int j = lo_q[q] + (e - wb[q]);
    cp_async4(w_idx + e, mt.in_idx[q] + j);
    cp_async4(w_val + e, mt.in_val[q] + j);
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  pstamp(4);
  // stable merged rank of every entry; the head of an index (its copy in the
  // lowest list) folds the later copies in list order.  Batches of kMB
  // entries per thread share every binary-search step (independent loads).
  constexpr int kMB = 8;
  int heads = 0;
  for (int e0 = 0; e0 < nin; e0 += kSelThreads * kMB) {
    int32_t x[kMB];
    int q[kMB], rank[kMB];
    float acc[kMB];
    bool head[kMB];
#pragma unroll
    for (int b = 0; b < kMB; ++b) {
      const int e = e0 + b * kSelThreads + tid;
      q[b] = -1;
      x[b] = 0;
      rank[b] = 0;
      acc[b] = 0.f;
      head[b] = false;
      if (e < nin) {
        q[b] = list_of(wb, r, e);
        x[b] = w_idx[e];
        acc[b] = w_val[e];
        rank[b] = e - wb[q[b]];
        head[b] = true;
      }
    }
    for (int u = 0; u < r; ++u) {   // ascending: the fold follows list order
      const int32_t* a = w_idx + wb[u];
      const unsigned a_s = static_cast<unsigned>(__cvta_generic_to_shared(a));
      const int n = wb[u + 1] - wb[u];
      int step = 1;
      while (step * 2 <= n) step *= 2;
      int32_t tgt[kMB];
      int pos[kMB];
#pragma unroll
      for (int b = 0; b < kMB; ++b) {
        tgt[b] = q[b] >= 0 && u < q[b] ? x[b] + 1 : x[b];   // upper_bound == lower_bound(x + 1)
        pos[b] = 0;
      }
      // branch-free steps: the kMB probes of a step are independent loads
      for (; n > 0 && step > 0; step >>= 1) {
        int32_t av[kMB];
#pragma unroll
        for (int b = 0; b < kMB; ++b) av[b] = lds_i32(a_s + 4u * (min(pos[b] + step, n) - 1));
#pragma unroll
        for (int b = 0; b < kMB; ++b) {
          const int p = pos[b] + step;
          pos[b] = (p <= n && av[b] < tgt[b]) ? p : pos[b];
        }
      }
#pragma unroll
      for (int b = 0; b < kMB; ++b) {
        if (q[b] < 0 || u == q[b]) continue;
        if (u < q[b]) {
          rank[b] += pos[b];
          if (pos[b] > 0 && a[pos[b] - 1] == x[b]) head[b] = false;
        } else {
          rank[b] += pos[b];
          if (pos[b] < n && a[pos[b]] == x[b]) acc[b] = __fadd_rn(acc[b], w_val[wb[u] + pos[b]]);
        }
      }
    }
#pragma unroll
    for (int b = 0; b < kMB; ++b) {
      if (q[b] < 0) continue;
      heads += head[b];
      SPARDL_BOUND(base + rank[b], mt.out_cap);
      mt.out_idx[base + rank[b]] = x[b];
      mt.out_val[base + rank[b]] = head[b] ? acc[b] : __uint_as_float(kHoleBits);
    }
  }
  const long long my_heads = block_sum_ll(heads, lscr);   // (syncs: outputs visible in-CTA)
  pstamp(5);
  // the CTA's work items: pieces of its output range
  const int nit = min((nin + kChunkE - 1) / kChunkE, tab_cap);
  const int plen = nit > 0 ? ((nin + nit - 1) / nit + 31) & ~31 : kChunkE;
  for (int k = tid; k < nit; k += kSelThreads) {
    iof[k] = base + k * plen;
    ilen[k] = max(0, min(plen, nin - k * plen));
  }
  if (tid == 0) {
    s_F = nin;
    s_before = base / kChunkE + cr;
    s_nit = nit;
    cluster.map_shared_rank(tot, 0)[cr].cnt = my_heads;
  }
  cluster.sync();
  pstamp(6);
  long long total = 0;
  for (int q = 0; q < CL; ++q) total += cluster.map_shared_rank(tot, 0)[q].cnt;
  return total;
}

template <int CL, bool FUSED>
__global__ void __launch_bounds__(kSelThreads, SPARDL_SEL_MINB)
    k_select(const SelTask* __restrict__ tasks, int tab_cap, int win_cap, int vcap) {
  constexpr int kIlp = CL >= 6 ? SPARDL_SEL_ILP_WIDE : SPARDL_SEL_ILP;   // (shadows the default)
  constexpr int kChunkE = 32 * kIlp;
  pdl_enter();
  cg::cluster_group cluster = cg::this_cluster();
  const int cr = (int)cluster.block_rank();
  const SelTask t = tasks[blockIdx.y];   // by value: fields live in registers, not re-read
  // the wide path (wselect.cu) selected this task already unless it handed
  // it back (uniform per cluster: every CTA returns, no barrier is pending)
  if (!FUSED && t.ws && t.ws->state != kWFallback) return;
  SelScratch* sc = t.scr;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  // this CTA's histograms, double-buffered across exchanges (peers read
  // exchange e's buffer until they reach the barrier of exchange e + 1), and
  // their 32-bin super-bin sums
  __shared__ uint32_t histb[2][kBins];
  __shared__ uint32_t coarse[2][kBins / 32];
  uint32_t* hist = histb[0];
  __shared__ CtaTotals tot[CL];                     // every CTA's totals (every CTA a copy)
  __shared__ int scratch[40];
  __shared__ long long lscr[3 * 32];
  __shared__ RadixState my;                         // radix state (identical in every CTA)
  // this CTA's work items: contiguous pieces of its segments, <= plen long
  // (item i = input elements [iof[i], iof[i] + ilen[i])), so the warps share
  // long merge partitions evenly and never re-read segment bounds
  extern __shared__ int32_t dyn[];
  int32_t* iof = dyn;
  int32_t* ilen = dyn + tab_cap;
  // per-item counters (#above, #equal, #entries -> output offsets and tie
  // quota), kept on chip: the scan and the compaction read them without a
  // round trip to L2
  int32_t* c_a = dyn + 2 * tab_cap;
  int32_t* c_b = dyn + 3 * tab_cap;
  int32_t* c_c = dyn + 4 * tab_cap;
  // on-chip copy of the CTA's entries: item k's values at vc[coff[k]...] and
  // indices at ic[coff[k]...], staged once (1c) so that every pass reads
  // shared memory instead of L2 (items past vcap stay in memory)
  int32_t* coff = dyn + 5 * tab_cap;
  float* vc = reinterpret_cast<float*>(dyn + 6 * tab_cap);
  int32_t* ic = dyn + 6 * tab_cap + vcap;   // the indices beside them
  // fused merge: the CTA's input windows and the task's splitter samples
  int32_t* w_idx = dyn + 6 * tab_cap;
  float* w_val = reinterpret_cast<float*>(w_idx + win_cap);
  int32_t* samp = reinterpret_cast<int32_t*>(w_val + win_cap);


  if (!FUSED) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  peer_wait(t.ps);   // remote inputs (a slot, or the fused merge's lists)
  const int mode = resolve_mode(t);
  const int nseg = nseg_of(t, mode);
  // the previous run's threshold: its top digit is this run's first guess
  const uint32_t prev_T = sc->prefix;
  const bool have_prev = sc->all == 0 && prev_T != 0;

  auto stamp = [&](int i) {
    if (SPARDL_STAMPS && cr == 0 && threadIdx.x == 0) {
      long long ts;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts));
      sc->tstamp[i] = ts;
    }
  };
  stamp(0);
  auto cta_stamp = [&](int k) {
    if (SPARDL_STAMPS && threadIdx.x == 0 && cr < 16) {
      long long ts;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts));
      sc->cta_ts[k][cr] = ts;
    }
  };
  cta_stamp(0);
  __shared__ int s_lo, s_hi, s_F, s_before;
  __shared__ int s_nit, s_plen;
  long long total = 0;
  if (FUSED && t.merge) {
    total = merge_prologue<CL>(*t.merge, cr, w_idx, w_val, samp, win_cap, iof, ilen, tab_cap,
                               s_F, s_before, s_nit, lscr, tot, cluster, sc);
  } else {
  // ---- 1. totals and an entry-balanced split of the segments over the
  // cluster: every CTA scans all segment lengths (cheap: <= 8192 counts) and
  // owns the segments whose first entry falls in its 1/CL of the entries.
  // The segment bounds are read once (all loads in flight) into the counter
  // arrays, which are free until the counting phase.
  for (int s = threadIdx.x; s < nseg; s += kSelThreads) {
    int off, c;
    seg_bounds(t, mode, s, off, c);
    c_a[s] = off;
    c_b[s] = c;
  }
  __syncthreads();
  {
    // pass A: the total
    long long part = 0;
    for (int s = threadIdx.x; s < nseg; s += kSelThreads) part += c_b[s];
    {
      long long u0 = 0, u1 = 0;
      block_sum3_ll(part, u0, u1, lscr);
      total = part;
    }
    const long long lo_t = total * cr / CL, hi_t = total * (cr + 1) / CL;
    // pass B: s0 = #{s : start(s) < lo_t}, s1 = #{s : start(s) < hi_t}
    int carry = 0, n_lo = 0, n_hi = 0;
    for (int b0 = 0; b0 < nseg; b0 += kSelThreads) {
      const int s = b0 + threadIdx.x;
      const int c = s < nseg ? c_b[s] : 0;
      int tt;
      const long long start = carry + block_exscan(c, scratch, &tt);
      n_lo += __syncthreads_count(s < nseg && start < lo_t);
      n_hi += __syncthreads_count(s < nseg && start < hi_t);
      carry += tt;
    }
    if (threadIdx.x == 0) {
      s_lo = cr == 0 ? 0 : n_lo;
      s_hi = cr == CL - 1 ? nseg : n_hi;
    }
    __syncthreads();
  }
  const int s0 = s_lo, s1 = s_hi;
  const int nloc = s1 - s0;
  // ---- 1b. the work items of this CTA
  {
    long long here = 0;
    for (int s = s0 + threadIdx.x; s < s1; s += kSelThreads) here += c_b[s];
    {
      long long u0 = 0, u1 = 0;
      block_sum3_ll(here, u0, u1, lscr);
    }
    // smallest piece length (kChunkE * 2^j) whose items fit the table
    long long plen = kChunkE;
    while (nloc + (here + plen - 1) / plen > tab_cap && plen < (1ll << 30)) plen <<= 1;
    int carry = 0;
    for (int b0 = 0; b0 < nloc; b0 += kSelThreads) {
      const int ls = b0 + threadIdx.x;
      const int off = ls < nloc ? c_a[s0 + ls] : 0;
      const int c = ls < nloc ? c_b[s0 + ls] : 0;
      const int np = (int)((c + plen - 1) / plen);
      int tt;
      int it = carry + block_exscan(np, scratch, &tt);
      for (int j = 0; j < np && it < tab_cap; ++j, ++it) {
        iof[it] = off + j * (int)plen;
        ilen[it] = min((int)plen, c - j * (int)plen);
      }
      carry += tt;
    }
    if (threadIdx.x == 0) {
      s_nit = min(carry, tab_cap);
      s_plen = (int)plen;
      s_F = (int)here;
    }
    if (vcap > 0) {
      __syncthreads();
      const int n = s_nit;
      int ccar = 0;
      for (int b0 = 0; b0 < n; b0 += kSelThreads) {
        const int k = b0 + threadIdx.x;
        int tt;
        const int o = ccar + block_exscan(k < n ? ilen[k] : 0, scratch, &tt);
        if (k < n) coff[k] = o;
        ccar += tt;
      }
    }
  }
  }
  const int64_t budget = t.budget_dev ? *t.budget_dev : t.budget;
  if (cr == 0 && threadIdx.x == 0) sc->cut_idx = -1;
  if (threadIdx.x == 0) {
    my.total = total;
    my.budget = budget;
    my.prefix = 0;
    my.pmask = 0;
    my.rank = budget;
    my.all = total <= budget ? 1 : (budget <= 0 ? 2 : 0);   // identity case, sparse.hpp:143-146
    my.hit = 0;
  }
  // the fused prologue's totals live in CTA 0's `tot`, which the exchanges
  // below overwrite: every CTA must have read them first
  if (FUSED) {
    cluster.sync();
  } else {
    // every CTA of the cluster has started (arrived at kernel entry): its
    // shared memory may be accessed from here on
    asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
    __syncthreads();
  }
  stamp(1);
  const int nit = s_nit;
  const float* __restrict__ vbase = mode == 1 ? t.dval : t.val;
  const int32_t* __restrict__ ibase = mode == 1 ? nullptr : t.idx;
  // merged inputs were written by this kernel: read them through L2 (the
  // read-only path is only for data that is constant during the kernel)
  const bool merged = FUSED && t.merge != nullptr;
  auto ldv = [&](const float* p) { return FUSED ? __ldcg(p) : __ldg(p); };
  auto ldi = [&](const int32_t* p) { return FUSED ? __ldcg(p) : __ldg(p); };
  // ---- 1c. stage the CTA's entries on chip: every item that fits is copied
  // with 4-byte asynchronous copies, all in flight at once (one memory
  // round trip instead of one per chunk and pass); the passes below read
  // shared memory, items past vcap read memory
  if (vcap > 0) {
    for (int k = warp; k < nit; k += kWarps) {
      const int c = ilen[k], cb = coff[k];
      if (cb + c > vcap) continue;
      const float* vp = vbase + iof[k];
      for (int j = lane; j < c; j += 32) cp_async4(vc + cb + j, vp + j);
      if (ibase) {
        const int32_t* ip = ibase + iof[k];
        for (int j = lane; j < c; j += 32) cp_async4(ic + cb + j, ip + j);
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
    __syncthreads();
  }
  // the staged items are a prefix (coff is their running sum): items < kst,
  // entries vc[0, nst) -- the histogram passes sweep them flat, whatever
  // the item boundaries (short candidate segments would leave lanes idle)
  __shared__ int s_kst;
  if (threadIdx.x == 0) s_kst = nit;
  __syncthreads();
  if (vcap > 0)
    for (int k = threadIdx.x; k < nit; k += kSelThreads)
      if (coff[k] + ilen[k] > vcap) atomicMin(&s_kst, k);
  __syncthreads();
  const int kst = vcap > 0 ? s_kst : 0;
  const int nst = kst > 0 ? coff[kst - 1] + ilen[kst - 1] : 0;
  auto staged = [&](int cb, int c) { return vcap > 0 && cb + c <= vcap; };
  auto fetch = [&](int cb, const float* __restrict__ vp, int c, int j0, float* v) {
    if (staged(cb, c)) {
#pragma unroll
      for (int u = 0; u < kIlp; ++u) {
        const int j = j0 + u * 32 + lane;
        v[u] = j < c ? vc[cb + j] : __uint_as_float(kHoleBits);
      }
    } else {
#pragma unroll
      for (int u = 0; u < kIlp; ++u) {   // all loads in flight first
        const int j = j0 + u * 32 + lane;
        v[u] = j < c ? ldv(vp + j) : __uint_as_float(kHoleBits);
      }
    }
  };

  // Cluster exchange of a pass (one barrier): every CTA histograms its own
  // entries into histb[x] and sums them into 32-bin super-bins; after the
  // cluster barrier every CTA reads the CL super-bin histograms (DSMEM),
  // finds the super-bin holding the rank, reads the CL copies of its 32 bins
  // and finds the digit -- all CTAs on identical data, no leader, no
  // broadcast, no second barrier.
  int xb = 0;   // exchange buffer
  auto make_coarse = [&](int nb) {   // after the histogram is complete
    __syncthreads();
    for (int c = warp; c < nb / 32; c += kWarps) {
      const uint32_t v = __reduce_add_sync(0xffffffffu, hist[c * 32 + lane]);
      if (lane == 0) coarse[xb][c] = v;
    }
  };
  __shared__ int s_sb;
  __shared__ long long s_above;
  auto find_digit_x = [&](int nb, int shift) {   // after the cluster barrier
    const int nc = nb / 32;            // 64 or 16 super-bins
    const int spl = nc >= 32 ? nc / 32 : 1;
    if (warp == 0) {
      long long part[2] = {0, 0};
      for (int q = 0; q < CL; ++q) {
        const uint32_t* cq = cluster.map_shared_rank(coarse[xb], q);
#pragma unroll
        for (int i = 0; i < 2; ++i)
          if (i < spl && lane * spl + i < nc) part[i] += cq[lane * spl + i];
      }
      const long long mine = part[0] + part[1];
      long long x = mine;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_down_sync(0xffffffffu, x, o);
        if (lane + o < 32) x += y;
      }
      const long long above = x - mine;
      const int64_t rank = my.rank;
      if (above < rank && rank <= above + mine) {
        long long cum = above;
        for (int i = spl - 1; i >= 0; --i) {
          if (cum + part[i] >= rank) {
            s_sb = lane * spl + i;
            s_above = cum;
            break;
          }
          cum += part[i];
        }
      }
      __syncwarp();
      const int sb = s_sb;
      const int bin = sb * 32 + lane;
      long long f = 0;
      for (int q = 0; q < CL; ++q) f += cluster.map_shared_rank(histb[xb], q)[bin];
      long long y = f;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long z = __shfl_down_sync(0xffffffffu, y, o);
        if (lane + o < 32) y += z;
      }
      const long long ab = s_above + (y - f);
      if (ab < rank && rank <= ab + f) {
        my.prefix |= (uint32_t)bin << shift;
        my.pmask |= (uint32_t)(nb - 1) << shift;
        my.rank = rank - ab;
      }
    }
    __syncthreads();
  };
  // CTA totals go to every CTA's `tot` (thread q stores into CTA q)
  auto bcast_tot = [&](CtaTotals v) {
    if (threadIdx.x < CL) cluster.map_shared_rank(tot, (int)threadIdx.x)[cr] = v;
  };

  // ---- 2. radix passes: warp w histograms chunks w, w + kWarps, ...
  int first_pass = 0;
  if (my.all == 0 && have_prev) {
    // One pass with the previous threshold's top digit d0 as a guess: the
    // histogram of the next 11 bits of the entries in d0, and the counts
    // above and inside d0.  If d0 holds the rank, pass 0 is skipped.
    const uint32_t d0 = prev_T >> 20;
    hist = histb[xb];
    for (int b = threadIdx.x; b < kBins; b += kSelThreads) hist[b] = 0;
    __syncthreads();
    long long above = 0, inside = 0;
    for (int e0 = threadIdx.x; e0 < nst; e0 += kSelThreads * kIlp) {
      uint32_t key[kIlp];
#pragma unroll
      for (int u = 0; u < kIlp; ++u) {
        const int e = e0 + u * kSelThreads;
        key[u] = e < nst ? mag_key(vc[e]) : kHoleKey;
      }
#pragma unroll
      for (int u = 0; u < kIlp; ++u) {
        const bool valid = key[u] != kHoleKey;
        const uint32_t top = key[u] >> 20;
        above += valid && top > d0;
        inside += valid && top == d0;
        hist_add(hist, (key[u] >> 9) & (kBins - 1), valid && top == d0);
      }
    }
    for (int k = kst + warp; k < nit; k += kWarps) {
      const int c = ilen[k];
      const int cb = vcap > 0 ? coff[k] : 0;
      const float* __restrict__ vp = vbase + iof[k];
      for (int j0 = 0; j0 < c; j0 += kChunkE) {
        float v[kIlp];
        fetch(cb, vp, c, j0, v);
        uint32_t key[kIlp];
#pragma unroll
        for (int u = 0; u < kIlp; ++u) key[u] = mag_key(v[u]);
#pragma unroll
        for (int u = 0; u < kIlp; ++u) {
          const bool valid = key[u] != kHoleKey;
          const uint32_t top = key[u] >> 20;
          above += valid && top > d0;
          inside += valid && top == d0;
          hist_add(hist, (key[u] >> 9) & (kBins - 1), valid && top == d0);
        }
      }
    }
    {
      long long unused = 0;
      block_sum3_ll(above, inside, unused, lscr);
    }
    stamp(2);
    bcast_tot({0, above, inside});
    make_coarse(kBins);
    cluster.sync();   // histograms, super-bins and totals of every CTA final
    stamp(3);
    __shared__ int s_hit;
    if (threadIdx.x == 0) {
      long long a = 0, in = 0;
      for (int q = 0; q < CL; ++q) {
        a += tot[q].gt;
        in += tot[q].eq;
      }
      const int hit = a < my.rank && my.rank <= a + in;
      if (cr == 0) {   // diagnostics: guess inputs
        sc->pro_ts[3] = d0;
        sc->pro_ts[4] = a;
        sc->pro_ts[5] = in;
        sc->pro_ts[6] = my.rank;
      }
      s_hit = hit;
      my.hit = hit;
      if (hit) {
        my.prefix = d0 << 20;
        my.pmask = (uint32_t)(kBins - 1) << 20;
        my.rank -= a;
      }
    }
    __syncthreads();
    if (s_hit) {
      find_digit_x(kBins, 9);
      first_pass = 2;
    }
    xb ^= 1;
    stamp(4);
    if (cr == 0 && threadIdx.x == 0) sc->pro_ts[7] = 100 + s_hit;   // diagnostics: guess outcome
  }
  if (my.all == 0) {
#pragma unroll 1
    for (int pass = first_pass; pass < 3; ++pass) {
      const int shift = pass == 0 ? 20 : (pass == 1 ? 9 : 0);
      const int nb = pass == 2 ? 512 : kBins;
      hist = histb[xb];
      for (int b = threadIdx.x; b < nb; b += kSelThreads) hist[b] = 0;
      __syncthreads();
      const uint32_t prefix = my.prefix, pmask = my.pmask;
      for (int e0 = threadIdx.x; e0 < nst; e0 += kSelThreads * kIlp) {
        uint32_t key[kIlp];
#pragma unroll
        for (int u = 0; u < kIlp; ++u) {
          const int e = e0 + u * kSelThreads;
          key[u] = e < nst ? mag_key(vc[e]) : kHoleKey;
        }
#pragma unroll
        for (int u = 0; u < kIlp; ++u)
          hist_add(hist, (key[u] >> shift) & (nb - 1),
                   key[u] != kHoleKey && (key[u] & pmask) == prefix);
      }
      for (int k = kst + warp; k < nit; k += kWarps) {
        const int c = ilen[k];
        const int cb = vcap > 0 ? coff[k] : 0;
        const float* __restrict__ vp = vbase + iof[k];
        for (int j0 = 0; j0 < c; j0 += kChunkE) {
          float v[kIlp];
          fetch(cb, vp, c, j0, v);
#pragma unroll
          for (int u = 0; u < kIlp; ++u) {
            const uint32_t key = mag_key(v[u]);
            hist_add(hist, (key >> shift) & (nb - 1),
                     key != kHoleKey && (key & pmask) == prefix);
          }
        }
      }
      __syncthreads();
      stamp(2 + 3 * pass);
      if (pass == 0) cta_stamp(1);
      make_coarse(nb);
      cluster.sync();   // every CTA's histogram and super-bins final
      stamp(3 + 3 * pass);
      find_digit_x(nb, shift);
      xb ^= 1;
      stamp(4 + 3 * pass);
    }
  }
  const int all = my.all;
  const uint32_t T = my.prefix;
  const int64_t need_eq = all == 0 ? my.rank : 0;

  // ---- 3. per-item counts (entries above T, equal to T, not holes), offsets
  long long g_loc = 0, e_loc = 0, v_loc = 0;
  for (int k = warp; k < nit; k += kWarps) {
    const int c = ilen[k];
    int gt = 0, eq = 0, nv = c;
    if (all == 0 || merged) {
      const float* __restrict__ vp = vbase + iof[k];
      const int cb = vcap > 0 ? coff[k] : 0;
      nv = 0;
      for (int j0 = 0; j0 < c; j0 += kChunkE) {
        float v[kIlp];
        fetch(cb, vp, c, j0, v);
        uint32_t key[kIlp];
#pragma unroll
        for (int u = 0; u < kIlp; ++u) key[u] = mag_key(v[u]);
#pragma unroll
        for (int u = 0; u < kIlp; ++u) {
          const bool in = key[u] != kHoleKey;
          nv += in;
          gt += in && key[u] > T;
          eq += in && key[u] == T;
        }
      }
      nv = __reduce_add_sync(0xffffffffu, nv);
      gt = __reduce_add_sync(0xffffffffu, gt);
      eq = __reduce_add_sync(0xffffffffu, eq);
    }
    if (all == 1) {
      gt = nv;
      eq = 0;
    } else if (all == 2) {
      gt = 0;
      eq = 0;
    }
    if (lane == 0) {
      c_a[k] = gt;
      c_b[k] = eq;
      c_c[k] = nv;
      g_loc += gt;
      e_loc += eq;
      v_loc += nv;
    }
  }
  block_sum3_ll(g_loc, e_loc, v_loc, lscr);
  bcast_tot({v_loc, g_loc, e_loc});
  cluster.sync();
  // Offsets in cluster order.  The tie quota is filled by the equal-key
  // entries in index order, so the entries selected before a position are
  // #{key > T before it} + min(#{key == T before it}, need_eq).
  __shared__ long long base_eq, base_gt, base_cnt, all_sel, all_cnt;
  if (threadIdx.x == 0) {
    long long be = 0, bg = 0, bc = 0;
    for (int q = 0; q < CL; ++q) {
      const CtaTotals x = tot[q];
      if (q == cr) {
        base_eq = be;
        base_gt = bg;
        base_cnt = bc;
      }
      be += x.eq;
      bg += x.gt;
      bc += x.cnt;
    }
    all_sel = bg + (be < need_eq ? be : need_eq);
    all_cnt = bc;
  }
  __syncthreads();
  {
    __shared__ int scr3[3 * 33];
    int g_carry = (int)base_gt, e_carry = (int)base_eq, c_carry = (int)base_cnt;
    for (int l0 = 0; l0 < nit; l0 += kSelThreads) {
      const int k = l0 + threadIdx.x;
      int gt = 0, eq = 0, c = 0;
      if (k < nit) {
        gt = c_a[k];
        eq = c_b[k];
        c = c_c[k];
      }
      int gb, eb, cb, tg, te, tc;
      block_exscan3(gt, eq, c, scr3, gb, eb, cb, tg, te, tc);
      gb += g_carry;
      eb += e_carry;
      cb += c_carry;
      const long long q = need_eq - eb;
      const int take = q <= 0 ? 0 : (q >= eq ? eq : (int)q);
      const int sel_off = gb + (int)(eb < need_eq ? (long long)eb : need_eq);
      if (k < nit) {
        c_a[k] = sel_off;   // in place: item k is this thread's alone
        c_b[k] = take == eq ? -1 : take;   // -1: every tie of the item is kept
        c_c[k] = cb - sel_off;
      }
      g_carry += tg;
      e_carry += te;
      c_carry += tc;
    }
  }
  __syncthreads();

  stamp(10);
  // ---- 4. ordered compaction, chunk by chunk
  const float w = t.weight;
  const bool want_dis = t.dis_idx != nullptr;
  // consumer ranks' copies (peer transport): bases held in registers
  const int npush = t.npush;
  int32_t* pidx[kMaxPush];
  float* pval[kMaxPush];
  if (npush > 0) {
#pragma unroll
    for (int p = 0; p < kMaxPush; ++p) {
      unsigned char* b = p < npush ? t.push_base[p] : nullptr;
      pidx[p] = reinterpret_cast<int32_t*>(b + 16);
      pval[p] = reinterpret_cast<float*>(b + 16 + 4 * (size_t)t.push_cap);
    }
  }
  const uint32_t lt = lanemask_lt();
  int cut = -1;
  for (int k = warp; k < nit; k += kWarps) {
    const int c = ilen[k], e0 = iof[k];
    const int sel_base = c_a[k], dis_base = c_c[k], take = c_b[k];
    int eq_seen = 0, sel_seen = 0, val_seen = 0;
    const float* __restrict__ vp = vbase + e0;
    const int32_t* __restrict__ ip = ibase ? ibase + e0 : nullptr;
    const int32_t ib = t.dbase + e0;
    const int cb = vcap > 0 ? coff[k] : 0;
    for (int j00 = 0; j00 < c; j00 += kChunkE) {
      float vv[kIlp];
      int32_t iv[kIlp];
      if (staged(cb, c)) {
#pragma unroll
        for (int u = 0; u < kIlp; ++u) {
          const int j = j00 + u * 32 + lane;
          iv[u] = j < c ? (ip ? ic[cb + j] : ib + j) : 0;
        }
      } else {
#pragma unroll
        for (int u = 0; u < kIlp; ++u) {   // index loads first, then the values
          const int j = j00 + u * 32 + lane;
          iv[u] = j < c ? (ip ? ldi(ip + j) : ib + j) : 0;
        }
      }
      fetch(cb, vp, c, j00, vv);
#pragma unroll
      for (int u = 0; u < kIlp; ++u) {
        const float v = vv[u];
        const int32_t ix = iv[u];
        const uint32_t key = mag_key(v);
        // holes exist only in fused-merge inputs; otherwise validity is the
        // position (lanes past the item hold hole bits)
        const int j = j00 + u * 32 + lane;
        const bool valid = FUSED ? key != kHoleKey : j < c;
        bool is_sel;
        if (all == 1) {
          is_sel = valid;
        } else if (all == 2) {
          is_sel = false;
        } else if (take < 0) {   // all ties of this item kept: no tie ranking
          is_sel = valid && key >= T;
          if (is_sel && key == T) cut = max(cut, ix);
        } else {
          const bool is_eq = valid && key == T;
          const uint32_t be = __ballot_sync(0xffffffffu, is_eq);
          const int eq_rank = eq_seen + __popc(be & lt);
          eq_seen += __popc(be);
          is_sel = valid && (key > T || (is_eq && eq_rank < take));
          if (is_sel && is_eq) cut = max(cut, ix);
        }
        const uint32_t bs = __ballot_sync(0xffffffffu, is_sel);
        const int sel_rank = sel_seen + __popc(bs & lt);
        sel_seen += __popc(bs);
        int val_rank = j;   // entries of the item before this one
        if (FUSED) {
          const uint32_t bv = __ballot_sync(0xffffffffu, valid);
          val_rank = val_seen + __popc(bv & lt);
          val_seen += __popc(bv);
        }
        if (is_sel) {
          SPARDL_BOUND_CAP(sel_base + sel_rank, t.sel_cap);
          t.sel_idx[sel_base + sel_rank] = ix;
          t.sel_val[sel_base + sel_rank] = v;
          if (npush > 0) {
#pragma unroll
            for (int p = 0; p < kMaxPush; ++p)
              if (p < npush) {
                SPARDL_BOUND_CAP(sel_base + sel_rank, t.push_cap);
                pidx[p][sel_base + sel_rank] = ix;
                pval[p][sel_base + sel_rank] = v;
              }
          }
        } else if (valid && want_dis) {
          const int p = dis_base + (val_rank - sel_rank);
          SPARDL_BOUND_CAP(p, t.dis_cap);
          t.dis_idx[p] = ix;
          t.dis_val[p] = __fmul_rn(v, w);
        }
      }
    }
  }
  if (all == 0) {
    cut = __reduce_max_sync(0xffffffffu, cut);
    if (lane == 0 && cut >= 0) atomicMax(&sc->cut_idx, cut);
  }
  if (cr == 0 && threadIdx.x == 0) {
    *t.sel_cnt = (int32_t)all_sel;
    for (int p = 0; p < npush; ++p) *reinterpret_cast<int32_t*>(t.push_base[p]) = (int32_t)all_sel;
    if (t.dis_cnt) *t.dis_cnt = (int32_t)(all_cnt - all_sel);
    if (t.total_out) *t.total_out = my.total;
    // the finished selection, for membership tests (sel_member)
    sc->prefix = T;
    sc->all = all;
    sc->mode = mode;
    sc->total = my.total;
    if (all == 1 && mode == 0 && t.mode_from_cand) {
      // exactly L candidates, all kept: the selection is {key >= pre-threshold},
      // not the whole block
      sc->all = 0;
      sc->prefix = *t.pre_key_dev;
      sc->cut_idx = INT_MAX;
    }
    if (t.div_hist) update_history(t.div_hist, mode, all, T, *t.pre_key_dev, total, budget);
    if (t.fallbacks && t.mode_from_cand && mode == 1) atomicAdd(t.fallbacks, 1ull);
  }
  stamp(11);
  // (no shared-memory access crosses CTAs after the totals exchange)
  if (t.ps.npub > 0) {
    // every CTA's output writes are ordered before this cluster barrier: the
    // block can go to its consumers now, not at the end of the batch (the
    // copy pushed into a peer's memory is fenced at system scope first)
    if (npush > 0) __threadfence_system();
    cluster.sync();
    if (cr == 0 && threadIdx.x == 0) peer_publish(t.ps);
  }
}

}  // namespace

int sel_prepare(SelTask& t, int max_seg_len) {
  (void)max_seg_len;
  if (t.dn > 0) {
    // dense slices: tiles of >= 256 entries, at most kMaxSegPerTask of them
    int stride = kTile;
    while ((int64_t)(t.dn + stride - 1) / stride > kMaxSegPerTask) stride += kTile;
    t.dstride = stride;
    t.dnseg = (t.dn + stride - 1) / stride;
  }
  return t.nseg;
}

int sel_scratch_segments(const SelTask& t) { return t.nseg > t.dnseg ? t.nseg : t.dnseg; }

int sel_grid_segments(const SelTask& t) {
  if (t.mode == 1 && !t.mode_from_cand) return t.dnseg;
  return t.nseg;
}

namespace {
template <int CL>
cudaLaunchConfig_t cl_config(int ntask, size_t smem, cudaStream_t s, cudaLaunchAttribute* attr) {
  cudaLaunchConfig_t lc{};
  lc.gridDim = dim3(CL, ntask);
  lc.blockDim = dim3(kSelThreads);
  lc.dynamicSmemBytes = smem;
  lc.stream = s;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CL;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = attr;
  lc.numAttrs = pdl_enabled() && s ? 2 : 1;
  return lc;
}

// item table: iof, ilen, three counters, cache offset
size_t table_bytes(int tab_cap) { return sizeof(int32_t) * 6 * static_cast<size_t>(tab_cap); }

int max_dyn_smem();

// entries of the on-chip value copy: whatever shared memory the table
// leaves (one CTA per SM either way: 512 threads at > 64 registers)
int value_cache_cap(int tab_cap) {
  static const bool off = [] {
    const char* e = getenv("SPARDL_SEL_VCACHE");   // tuning experiments only
    return e && e[0] == '0';
  }();
  if (off) return 0;
  // (SPARDL_SEL_MINB CTAs share an SM's 228 KB; ~24 KB of static shared
  // memory and reserve per CTA)
  const long long budget = SPARDL_SEL_MINB > 1 ? 233472ll / SPARDL_SEL_MINB - 24 * 1024
                                               : (long long)max_dyn_smem();
  const long long avail = budget - (long long)table_bytes(tab_cap);
  return avail >= 8 * 1024 ? (int)((avail / 8) & ~31ll) : 0;
}

size_t dyn_bytes(int tab_cap, int win_cap) {
  size_t b = table_bytes(tab_cap);
  if (win_cap > 0) b += 8 * static_cast<size_t>(win_cap) + sizeof(int32_t) * (kMergeSamples + kMaxR);
  else b += 8 * static_cast<size_t>(value_cache_cap(tab_cap));   // value + index
  return b;
}

int optin_smem() {
  int dev = 0, optin = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  return optin;
}

template <int CL, bool F>
int configure() {   // returns the dynamic shared memory this instantiation may use
  static std::mutex mu;
  static int maxdyn[kMaxDevices] = {};   // 0: not configured on that device
  const int dev = cur_device();
  std::lock_guard<std::mutex> lock(mu);
  if (maxdyn[dev] <= 0) {   // 16 is a non-portable cluster size on sm_100
    cudaFuncSetAttribute(k_select<CL, F>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(k_select<CL, F>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, k_select<CL, F>);
    int md = optin_smem() - (int)fa.sharedSizeBytes;
    if (cudaFuncSetAttribute(k_select<CL, F>, cudaFuncAttributeMaxDynamicSharedMemorySize, md) !=
        cudaSuccess) {
      cudaGetLastError();
      md = 48 * 1024 - (int)fa.sharedSizeBytes;
    }
    maxdyn[dev] = md;
  }
  return maxdyn[dev];
}

// dynamic shared memory every instantiation may use
int max_dyn_smem() {
  const int a = std::min(configure<16, true>(), configure<8, true>());
  const int b = std::min(configure<4, true>(), configure<2, true>());
  const int c = std::min(std::min(configure<16, false>(), configure<10, false>()),
                         configure<8, false>());
  const int d = std::min(std::min(configure<6, false>(), configure<4, false>()),
                         configure<2, false>());
  return std::min(std::min(a, b), std::min(c, d));
}

// clusters of width CL that can be resident at once on this device (a
// cluster must fit in one GPC, so wide clusters leave SMs unused)
template <int CL, bool F>
int max_clusters(size_t smem) {
  configure<CL, F>();
  static std::mutex mu;
  static size_t last_smem[kMaxDevices];
  static int n[kMaxDevices] = {};
  static bool init = [] {
    for (auto& x : last_smem) x = ~size_t(0);
    return true;
  }();
  (void)init;
  const int dev = cur_device();
  std::lock_guard<std::mutex> lock(mu);
  if (smem != last_smem[dev]) {
    cudaLaunchAttribute attr[2];
    cudaLaunchConfig_t lc = cl_config<CL>(1, smem, nullptr, attr);
    int c = 0;
    if (cudaOccupancyMaxActiveClusters(&c, k_select<CL, F>, &lc) != cudaSuccess) {
      cudaGetLastError();
      c = 0;
    }
    n[dev] = c;
    last_smem[dev] = smem;
    if (getenv("SPARDL_DEBUG"))
      fprintf(stderr, "k_select<%d,%d>: %d resident clusters (%zu B dynamic smem)\n", CL, (int)F,
              c, smem);
  }
  return n[dev];
}

template <bool F>
int clusters_for(int cl, size_t smem) {
  if (cl >= 16) return max_clusters<16, F>(smem);
  if constexpr (!F) {
    if (cl >= 10) return max_clusters<10, F>(smem);
  }
  if (cl >= 8) return max_clusters<8, F>(smem);
  if constexpr (!F) {
    if (cl >= 6) return max_clusters<6, F>(smem);
  }
  if (cl >= 4) return max_clusters<4, F>(smem);
  return max_clusters<2, F>(smem);
}

template <int CL, bool F>
void launch_cl(const SelTask* tasks_dev, int ntask, int tab_cap, int win_cap, cudaStream_t s) {
  const size_t smem = dyn_bytes(tab_cap, win_cap);
  const int vcap = win_cap > 0 ? 0 : value_cache_cap(tab_cap);
  configure<CL, F>();
  cudaLaunchAttribute attr[3];
  cudaLaunchConfig_t lc = cl_config<CL>(ntask, smem, s, attr);
  // a select on a high-priority stream (overlapping a streaming pass) keeps
  // its priority inside a captured graph as a node attribute
  int prio = 0;
  if (s && cudaStreamGetPriority(s, &prio) == cudaSuccess && prio != 0) {
    attr[lc.numAttrs].id = cudaLaunchAttributePriority;
    attr[lc.numAttrs].val.priority = prio;
    ++lc.numAttrs;
  }
  note_launch(cudaLaunchKernelEx(&lc, k_select<CL, F>, tasks_dev, tab_cap, win_cap, vcap));
}

template <bool F>
void launch_w(int cl, const SelTask* tasks_dev, int ntask, int tab_cap, int win_cap, cudaStream_t s) {
  if constexpr (!F) {   // widths that are not powers of two: plain selects only
    if (cl >= 10 && cl < 16) return launch_cl<10, F>(tasks_dev, ntask, tab_cap, win_cap, s);
    if (cl >= 6 && cl < 8) return launch_cl<6, F>(tasks_dev, ntask, tab_cap, win_cap, s);
  }
  if (cl >= 16) launch_cl<16, F>(tasks_dev, ntask, tab_cap, win_cap, s);
  else if (cl >= 8) launch_cl<8, F>(tasks_dev, ntask, tab_cap, win_cap, s);
  else if (cl >= 4) launch_cl<4, F>(tasks_dev, ntask, tab_cap, win_cap, s);
  else launch_cl<2, F>(tasks_dev, ntask, tab_cap, win_cap, s);
}

int forced_cl() {
  static int f = -1;
  if (f < 0) {
    const char* e = getenv("SPARDL_SELECT_CLUSTER");   // tuning experiments only
    f = e ? atoi(e) : 0;
  }
  return f;
}

int table_cap(int max_nseg) { return max_nseg < 2048 ? 2048 : max_nseg; }
}  // namespace

int sel_chunk_capacity(const SelTask& t) {
  const int64_t ex = (int64_t)t.nseg * t.stride;
  const int64_t mx = ex > t.dn ? ex : t.dn;
  const int ns = t.nseg > t.dnseg ? t.nseg : t.dnseg;
  return ns + (int)((mx + kChunkE - 1) / kChunkE) + kCl + 2;
}

int select_max_window() {
  const int avail = max_dyn_smem() - (int)table_bytes(table_cap(1)) -
                    (int)(sizeof(int32_t) * (kMergeSamples + kMaxR)) - 1024;
  return avail > 0 ? avail / 8 : 0;
}

int select_resident_clusters(int cl, int tab_cap, int win_cap) {
  return clusters_for<true>(cl, dyn_bytes(table_cap(tab_cap), win_cap));
}

int launch_select(const SelTask* tasks_dev, int ntask, int max_nseg, cudaStream_t s, int cluster,
                  int win_cap) {
  if (ntask <= 0) return 0;
  // item table: at least 2048 entries so long inputs split into short pieces
  const int tab_cap = table_cap(max_nseg);
  const size_t smem = dyn_bytes(tab_cap, win_cap);
  // the widest cluster for which every task's cluster is resident in one
  // wave (a second wave would double the latency of the whole batch)
  int cl = cluster > 0 ? cluster : forced_cl();
  if (cl == 0) {
    // widths 10 and 6 fill the GPCs better than 8 and 4 (B200: 11 and 22
    // resident clusters against 15 and 33, i.e. 80/96 CTAs for 8/16 tasks)
    cl = 2;
    for (int w : {16, 10, 8, 6, 4})
      if (clusters_for<false>(w, smem) >= ntask) {
        cl = w;
        break;
      }
  }
  static int dbg = 0;
  if (dbg < 8 && getenv("SPARDL_DEBUG")) {
    ++dbg;
    fprintf(stderr, "select batch: %d tasks -> cluster %d (window %d)\n", ntask, cl, win_cap);
  }
  if (win_cap > 0) launch_w<true>(cl, tasks_dev, ntask, tab_cap, win_cap, s);
  else launch_w<false>(cl, tasks_dev, ntask, tab_cap, win_cap, s);
  return 1;
}

}  // namespace sdl
