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
//      memory, adds the non-zero bins into CTA 0's histogram through DSMEM,
//      CTA 0 locates the digit holding the rank-th largest key and the other
//      CTAs read the new prefix from CTA 0 -- two cluster barriers per pass,
//      no global atomics, no kernel boundaries.  After the three passes the
//      threshold key T is exact, and need_eq = L - #{key > T} entries of key
//      T are kept: the lowest-index ones (the reference's tie rule).
//   3. per segment (one warp each) #{key > T}, #{key == T}; CTA totals go
//      through DSMEM so every CTA knows the tie quota and the output offsets
//      of the CTAs before it; a CTA-wide scan places each segment.
//   4. ordered compaction with warp ballots of the selected entries and of
//      the discarded ones, the latter scaled by the residual share with an
//      explicitly rounded multiply (no FMA contraction, inc/residual.hpp:119).
#include <cooperative_groups.h>

#include <climits>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace sdl {

namespace {

constexpr int kSelThreads = 512;   // 16 warps per CTA
constexpr int kWarps = kSelThreads / 32;
#ifndef SPARDL_SEL_ILP
#define SPARDL_SEL_ILP 8
#endif
constexpr int kIlp = SPARDL_SEL_ILP;   // 32-entry groups loaded per warp step (memory-level parallelism)
constexpr int kChunkE = 32 * kIlp;   // flat entries per work chunk (one warp step)

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
  int32_t pad_;
};

struct CtaTotals {      // per-CTA counters exchanged through DSMEM
  long long cnt, gt, eq;
};

// Dividing select epilogue: the pre-threshold of the next iteration.
__device__ void update_history(DivHistory* h, int mode, int all, uint32_t T, uint32_t pre,
                               long long cand, long long budget) {
  constexpr uint32_t kMinDelta = 1u << 12, kMaxDelta = 1u << 26;
  constexpr double kTarget = 1.5;    // wanted candidates / L
  if (mode != 0 || all != 0 || budget <= 0) {   // dense fallback (or trivial): sample again
    if (h->valid) h->delta = h->delta < kMaxDelta / 2 ? h->delta * 2 : kMaxDelta;
    h->valid = 0;
    h->has_T = all == 0 && budget > 0;
    h->last_T = T;
    return;
  }
  // secant in (key, log count): count(pre) = cand, count(T) = budget
  const double span = (double)(T - pre);
  const double ratio = (double)cand / (double)budget;
  double d;
  if (ratio > 1.02 && span > 0) d = span * log(kTarget) / log(ratio);
  else d = 2.0 * (span > 0 ? span : (double)kMinDelta);
  if (h->valid) {   // at most x2 / x0.5 per run
    const double old = (double)h->delta;
    d = d > 2 * old ? 2 * old : (d < old / 2 ? old / 2 : d);
  }
  d = d < kMinDelta ? kMinDelta : (d > kMaxDelta ? kMaxDelta : d);
  // a threshold that grows from run to run (residual accumulation) is
  // extrapolated linearly in magnitude
  const float tv = __uint_as_float(T), tp = __uint_as_float(h->last_T);
  const float grown = h->has_T && tv > tp ? tv + (tv - tp) : tv;
  const uint32_t Tn = grown < 3.0e38f ? __float_as_uint(grown) : T;
  long long next = (long long)Tn - (long long)d;
  h->delta = (uint32_t)d;
  h->next_pre = next < 0 ? 0u : (uint32_t)next;
  // the first threshold after a (re)start only seeds the trend: trust the
  // carried pre-threshold from the second sampled run on
  h->valid = h->has_T;
  h->last_T = T;
  h->has_T = 1;
}

// CTA 0: locate the digit holding the rank-th largest key in agg[0..nb).
__device__ void find_digit(uint32_t* agg, int nb, int shift, RadixState* st, long long* suf) {
  const int bpt = nb / kSelThreads;
  long long mine = 0;
  for (int q = 0; q < bpt; ++q) mine += agg[threadIdx.x * bpt + q];
  const int r = kSelThreads - 1 - threadIdx.x;     // bins ascend with tid; scan from the top
  suf[r] = mine;
  __syncthreads();
  for (int o = 1; o < kSelThreads; o <<= 1) {
    const long long add = threadIdx.x >= (unsigned)o ? suf[threadIdx.x - o] : 0;
    __syncthreads();
    suf[threadIdx.x] += add;
    __syncthreads();
  }
  const long long above = r > 0 ? suf[r - 1] : 0;
  const int64_t rank = st->rank;
  __syncthreads();
  if (above < rank && rank <= above + mine) {
    long long cum = above;
    for (int q = bpt - 1; q >= 0; --q) {
      const uint32_t c = agg[threadIdx.x * bpt + q];
      if (cum + (long long)c >= rank) {
        const uint32_t digit = threadIdx.x * bpt + q;
        st->prefix |= digit << shift;
        st->pmask |= (uint32_t)(nb - 1) << shift;
        st->rank = rank - cum;
        break;
      }
      cum += c;
    }
  }
  __syncthreads();
  for (int q = 0; q < bpt; ++q) agg[threadIdx.x * bpt + q] = 0;   // ready for the next pass
}

#ifndef SPARDL_SEL_MINB
#define SPARDL_SEL_MINB 1
#endif
template <int CL>
__global__ void __launch_bounds__(kSelThreads, SPARDL_SEL_MINB)
    k_select(const SelTask* __restrict__ tasks, int tab_cap) {
  cg::cluster_group cluster = cg::this_cluster();
  const int cr = (int)cluster.block_rank();
  const SelTask t = tasks[blockIdx.y];   // by value: fields live in registers, not re-read
  SelScratch* sc = t.scr;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  __shared__ uint32_t hist[kBins];
  __shared__ uint32_t agg[kBins];                   // meaningful in CTA 0
  __shared__ RadixState st;                         // meaningful in CTA 0
  __shared__ CtaTotals tot[CL];                     // meaningful in CTA 0
  __shared__ long long suf[kSelThreads];
  __shared__ int scratch[40];
  __shared__ long long lscr[32];
  __shared__ RadixState my;                         // this CTA's copy of CTA 0's state
  // this CTA's work items: contiguous pieces of its segments, <= plen long
  // (item i = input elements [iof[i], iof[i] + ilen[i])), so the warps share
  // long merge partitions evenly and never re-read segment bounds
  extern __shared__ int32_t dyn[];
  int32_t* iof = dyn;
  int32_t* ilen = dyn + tab_cap;

  RadixState* st0 = cluster.map_shared_rank(&st, 0);
  uint32_t* agg0 = cluster.map_shared_rank(agg, 0);
  CtaTotals* tot0 = cluster.map_shared_rank(tot, 0);

  const int mode = resolve_mode(t);
  const int nseg = nseg_of(t, mode);

  auto stamp = [&](int i) {
    if (cr == 0 && threadIdx.x == 0) {
      long long ts;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts));
      sc->tstamp[i] = ts;
    }
  };
  stamp(0);
  auto cta_stamp = [&](int k) {
    if (threadIdx.x == 0 && cr < 16) {
      long long ts;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts));
      sc->cta_ts[k][cr] = ts;
    }
  };
  cta_stamp(0);
  // ---- 1. totals and an entry-balanced split of the segments over the
  // cluster: every CTA scans all segment lengths (cheap: <= 8192 counts) and
  // owns the segments whose first entry falls in its 1/CL of the entries.
  __shared__ int s_lo, s_hi, s_F, s_before;
  long long total = 0;
  {
    // pass A: the total
    long long part = 0;
    for (int s = threadIdx.x; s < nseg; s += kSelThreads) {
      int off, c;
      seg_bounds(t, mode, s, off, c);
      part += c;
    }
    total = block_sum_ll(part, lscr);
    const long long lo_t = total * cr / CL, hi_t = total * (cr + 1) / CL;
    // pass B: s0 = #{s : start(s) < lo_t}, s1 = #{s : start(s) < hi_t}
    int carry = 0, n_lo = 0, n_hi = 0;
    for (int b0 = 0; b0 < nseg; b0 += kSelThreads) {
      const int s = b0 + threadIdx.x;
      int c = 0;
      if (s < nseg) {
        int off;
        seg_bounds(t, mode, s, off, c);
      }
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
  // ---- 1b. the work items of this CTA; its per-item scratch starts at
  // s0 + (entries before it) / kChunkE + cr (disjoint across the cluster)
  __shared__ int s_nit, s_plen;
  {
    long long before = 0, here = 0;
    for (int s = threadIdx.x; s < s1; s += kSelThreads) {
      int off, c;
      seg_bounds(t, mode, s, off, c);
      if (s < s0) before += c;
      else here += c;
    }
    before = block_sum_ll(before, lscr);
    here = block_sum_ll(here, lscr);
    // smallest piece length (kChunkE * 2^j) whose items fit the table
    long long plen = kChunkE;
    while (nloc + (here + plen - 1) / plen > tab_cap && plen < (1ll << 30)) plen <<= 1;
    int carry = 0;
    for (int b0 = 0; b0 < nloc; b0 += kSelThreads) {
      const int ls = b0 + threadIdx.x;
      int off = 0, c = 0;
      if (ls < nloc) seg_bounds(t, mode, s0 + ls, off, c);
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
      s_before = s0 + (int)(before / kChunkE) + cr;
    }
  }
  for (int b = threadIdx.x; b < kBins; b += kSelThreads) agg[b] = 0;
  const int64_t budget = t.budget_dev ? *t.budget_dev : t.budget;
  if (cr == 0 && threadIdx.x == 0) {
    st.total = total;
    st.budget = budget;
    st.prefix = 0;
    st.pmask = 0;
    st.rank = budget;
    st.all = total <= budget ? 1 : (budget <= 0 ? 2 : 0);   // identity case, sparse.hpp:143-146
    sc->cut_idx = -1;
  }
  if (threadIdx.x == 0) {
    my.total = total;
    my.budget = budget;
    my.prefix = 0;
    my.pmask = 0;
    my.rank = budget;
    my.all = total <= budget ? 1 : (budget <= 0 ? 2 : 0);
  }
  cluster.sync();   // CTA 0's aggregation histogram is zeroed; tables are visible
  stamp(1);
  const int nit = s_nit;
  // per-item counters of this CTA (task scratch, L2 resident)
  int* c_gt = t.seg_gt + s_before;
  int* c_eq = t.seg_eq + s_before;
  int* c_take = t.seg_take + s_before;
  int* c_sel = t.seg_sel_off + s_before;
  int* c_dis = t.seg_dis_off + s_before;
  const float* __restrict__ vbase = mode == 1 ? t.dval : t.val;
  const int32_t* __restrict__ ibase = mode == 1 ? nullptr : t.idx;

  // ---- 2. radix passes: warp w histograms chunks w, w + kWarps, ...
  if (my.all == 0) {
#pragma unroll 1
    for (int pass = 0; pass < 3; ++pass) {
      const int shift = pass == 0 ? 20 : (pass == 1 ? 9 : 0);
      const int nb = pass == 2 ? 512 : kBins;
      for (int b = threadIdx.x; b < nb; b += kSelThreads) hist[b] = 0;
      __syncthreads();
      const uint32_t prefix = my.prefix, pmask = my.pmask;
      for (int k = warp; k < nit; k += kWarps) {
        const int c = ilen[k];
        const float* __restrict__ vp = vbase + iof[k];
        for (int j0 = 0; j0 < c; j0 += kChunkE) {
          uint32_t key[kIlp];
#pragma unroll
          for (int u = 0; u < kIlp; ++u) {   // all loads in flight first
            const int j = j0 + u * 32 + lane;
            key[u] = j < c ? mag_key(__ldg(vp + j)) : 0u;
          }
#pragma unroll
          for (int u = 0; u < kIlp; ++u) {
            const int j = j0 + u * 32 + lane;
            hist_add(hist, (key[u] >> shift) & (nb - 1), j < c && (key[u] & pmask) == prefix);
          }
        }
      }
      __syncthreads();
      stamp(2 + 3 * pass);
      if (pass == 0) cta_stamp(1);
      // distributed reduction: CTA r sums its 1/CL slice of the bins over
      // all CTAs' histograms (DSMEM loads) and stores it into CTA 0's copy
      cluster.sync();
      {
        const int per = nb / CL;
        for (int b = cr * per + threadIdx.x; b < (cr + 1) * per; b += kSelThreads) {
          uint32_t sum = 0;
#pragma unroll
          for (int q = 0; q < CL; ++q) sum += cluster.map_shared_rank(hist, q)[b];
          agg0[b] = sum;
        }
      }
      cluster.sync();
      stamp(3 + 3 * pass);
      if (cr == 0) find_digit(agg, nb, shift, &st, suf);
      cluster.sync();
      if (threadIdx.x == 0) my = *st0;
      __syncthreads();
      stamp(4 + 3 * pass);
    }
  }
  const int all = my.all;
  const uint32_t T = my.prefix;
  const int64_t need_eq = all == 0 ? my.rank : 0;

  // ---- 3. per-chunk counts, offsets
  long long g_loc = 0, e_loc = 0;
  for (int k = warp; k < nit; k += kWarps) {
    const int c = ilen[k];
    int gt = 0, eq = 0;
    if (all == 1) {
      gt = c;
    } else if (all == 0) {
      const float* __restrict__ vp = vbase + iof[k];
      for (int j0 = 0; j0 < c; j0 += kChunkE) {
        uint32_t key[kIlp];
#pragma unroll
        for (int u = 0; u < kIlp; ++u) {
          const int j = j0 + u * 32 + lane;
          key[u] = j < c ? mag_key(__ldg(vp + j)) : 0u;
        }
#pragma unroll
        for (int u = 0; u < kIlp; ++u) {
          const bool in = j0 + u * 32 + lane < c;
          gt += in && key[u] > T;
          eq += in && key[u] == T;
        }
      }
      gt = __reduce_add_sync(0xffffffffu, gt);
      eq = __reduce_add_sync(0xffffffffu, eq);
    }
    if (lane == 0) {
      c_gt[k] = gt;
      c_eq[k] = eq;
      g_loc += gt;
      e_loc += eq;
    }
  }
  g_loc = block_sum_ll(g_loc, lscr);
  e_loc = block_sum_ll(e_loc, lscr);
  if (threadIdx.x == 0) tot0[cr] = {(long long)s_F, g_loc, e_loc};
  cluster.sync();
  __shared__ long long base_eq, base_sel, base_cnt, all_sel, all_cnt;
  if (threadIdx.x == 0) {
    long long be = 0, bs = 0, bc = 0, ts = 0, tc = 0;
    for (int q = 0; q < CL; ++q) {
      const CtaTotals x = tot0[q];
      long long take = need_eq - be;
      take = take < 0 ? 0 : (take > x.eq ? x.eq : take);
      if (q == cr) {
        base_eq = be;
        base_sel = bs;
        base_cnt = bc;
      }
      be += x.eq;
      bs += x.gt + take;
      bc += x.cnt;
      ts += x.gt + take;
      tc += x.cnt;
    }
    all_sel = ts;
    all_cnt = tc;
  }
  cluster.sync();   // every CTA has read CTA 0's totals
  __syncthreads();
  {
    int eq_carry = (int)base_eq, sel_carry = (int)base_sel, cnt_carry = (int)base_cnt;
    for (int l0 = 0; l0 < nit; l0 += kSelThreads) {
      const int k = l0 + threadIdx.x;
      int gt = 0, eq = 0, c = 0;
      if (k < nit) {
        gt = c_gt[k];
        eq = c_eq[k];
        c = ilen[k];
      }
      int teq, tsel, tcnt;
      const int eq_before = eq_carry + block_exscan(eq, scratch, &teq);
      const long long q = need_eq - eq_before;
      const int take = q <= 0 ? 0 : (q >= eq ? eq : (int)q);
      const int sel = gt + take;
      const int sel_off = sel_carry + block_exscan(sel, scratch, &tsel);
      const int cnt_off = cnt_carry + block_exscan(c, scratch, &tcnt);
      if (k < nit) {
        c_take[k] = take;
        c_sel[k] = sel_off;
        c_dis[k] = cnt_off - sel_off;
      }
      eq_carry += teq;
      sel_carry += tsel;
      cnt_carry += tcnt;
    }
  }
  __syncthreads();

  stamp(10);
  // ---- 4. ordered compaction, chunk by chunk
  const float w = t.weight;
  const bool want_dis = t.dis_idx != nullptr;
  const uint32_t lt = lanemask_lt();
  int cut = -1;
  for (int k = warp; k < nit; k += kWarps) {
    const int c = ilen[k], e0 = iof[k];
    const int sel_base = c_sel[k], dis_base = c_dis[k], take = c_take[k];
    int eq_seen = 0, sel_seen = 0;
    const float* __restrict__ vp = vbase + e0;
    const int32_t* __restrict__ ip = ibase ? ibase + e0 : nullptr;
    const int32_t ib = t.dbase + e0;
    for (int j00 = 0; j00 < c; j00 += kChunkE) {
      float vv[kIlp];
      int32_t iv[kIlp];
#pragma unroll
      for (int u = 0; u < kIlp; ++u) {   // all loads in flight first
        const int j = j00 + u * 32 + lane;
        vv[u] = j < c ? __ldg(vp + j) : 0.f;
        iv[u] = j < c ? (ip ? __ldg(ip + j) : ib + j) : 0;
      }
#pragma unroll
      for (int u = 0; u < kIlp; ++u) {
        const int j = j00 + u * 32 + lane;
        const bool valid = j < c;
        const float v = vv[u];
        const int32_t ix = iv[u];
        const uint32_t key = mag_key(v);
        bool is_sel;
        if (all == 1) {
          is_sel = valid;
        } else if (all == 2) {
          is_sel = false;
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
        if (is_sel) {
          t.sel_idx[sel_base + sel_rank] = ix;
          t.sel_val[sel_base + sel_rank] = v;
        } else if (valid && want_dis) {
          const int p = dis_base + (j - sel_rank);
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
  }
  stamp(11);
  cluster.sync();   // keep CTA 0's shared memory alive until every reader is done
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
  lc.attrs = attr;
  lc.numAttrs = 1;
  return lc;
}

size_t table_bytes(int tab_cap) { return sizeof(int32_t) * 2 * static_cast<size_t>(tab_cap); }

// clusters of width CL that can be resident at once on this device (a
// cluster must fit in one GPC, so wide clusters leave SMs unused)
template <int CL>
int max_clusters(size_t smem) {
  static bool configured = false;
  static size_t last_smem = ~size_t(0);
  static int n = 0;
  if (!configured) {   // 16 is a non-portable cluster size on sm_100
    cudaFuncSetAttribute(k_select<CL>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaFuncSetAttribute(k_select<CL>, cudaFuncAttributePreferredSharedMemoryCarveout, 100);
    cudaFuncSetAttribute(k_select<CL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)table_bytes(kMaxSegPerTask));
    configured = true;
  }
  if (smem != last_smem) {
    cudaLaunchAttribute attr[1];
    cudaLaunchConfig_t lc = cl_config<CL>(1, smem, nullptr, attr);
    int c = 0;
    if (cudaOccupancyMaxActiveClusters(&c, k_select<CL>, &lc) != cudaSuccess) {
      cudaGetLastError();
      c = 0;
    }
    n = c;
    last_smem = smem;
    if (getenv("SPARDL_DEBUG"))
      fprintf(stderr, "k_select<%d>: %d resident clusters (%zu B tables)\n", CL, n, smem);
  }
  return n;
}

template <int CL>
void launch_cl(const SelTask* tasks_dev, int ntask, int tab_cap, cudaStream_t s) {
  const size_t smem = table_bytes(tab_cap);
  max_clusters<CL>(smem);
  cudaLaunchAttribute attr[1];
  cudaLaunchConfig_t lc = cl_config<CL>(ntask, smem, s, attr);
  cudaLaunchKernelEx(&lc, k_select<CL>, tasks_dev, tab_cap);
}

int forced_cl() {
  static int f = -1;
  if (f < 0) {
    const char* e = getenv("SPARDL_SELECT_CLUSTER");   // tuning experiments only
    f = e ? atoi(e) : 0;
  }
  return f;
}
}  // namespace

int sel_chunk_capacity(const SelTask& t) {
  const int64_t ex = (int64_t)t.nseg * t.stride;
  const int64_t mx = ex > t.dn ? ex : t.dn;
  const int ns = t.nseg > t.dnseg ? t.nseg : t.dnseg;
  return ns + (int)((mx + kChunkE - 1) / kChunkE) + kCl + 2;
}

int launch_select(const SelTask* tasks_dev, int ntask, int max_nseg, cudaStream_t s) {
  if (ntask <= 0) return 0;
  // item table: at least 2048 entries so long inputs split into short pieces
  const int tab_cap = max_nseg < 2048 ? 2048 : max_nseg;
  const size_t smem = table_bytes(tab_cap);
  // the widest cluster for which every task's cluster is resident in one
  // wave (a second wave would double the latency of the whole batch)
  int cl = forced_cl();
  if (cl == 0) {
    if (max_clusters<16>(smem) >= ntask) cl = 16;
    else if (max_clusters<8>(smem) >= ntask) cl = 8;
    else if (max_clusters<4>(smem) >= ntask) cl = 4;
    else cl = 2;
  }
  static int dbg = 0;
  if (dbg < 8 && getenv("SPARDL_DEBUG")) {
    ++dbg;
    fprintf(stderr, "select batch: %d tasks -> cluster %d\n", ntask, cl);
  }
  if (cl >= 16) launch_cl<16>(tasks_dev, ntask, tab_cap, s);
  else if (cl >= 8) launch_cl<8>(tasks_dev, ntask, tab_cap, s);
  else if (cl >= 4) launch_cl<4>(tasks_dev, ntask, tab_cap, s);
  else launch_cl<2>(tasks_dev, ntask, tab_cap, s);
  return 1;
}

}  // namespace sdl
