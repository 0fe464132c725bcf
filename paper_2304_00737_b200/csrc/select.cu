// Deterministic top-L selection over segmented sparse lists.
//
// Semantics: inc/sparse.hpp:136-162 (top_k_select) -- keep the min(budget,
// nnz) entries that come first in the order (|v| desc, index asc); return
// the kept and the discarded entries, each in index order.
//
// Method (per task, all tasks of a batch in one launch per kernel):
//   hist<0..2> + find<0..2>: radix select on the 31-bit magnitude key
//       (digits 11 / 11 / 9 bits).  After the three passes the threshold key
//       T is exact, cnt_gt = #{key > T} and need_eq = L - cnt_gt entries of
//       key == T are taken -- the lowest-index ones, which is exactly the
//       reference's tie rule.  For the dividing select the first histogram is
//       built by the candidate pass itself (divide.cu), so hist<0> skips it.
//   count: per segment (one warp each) #{key > T} and #{key == T}
//   scan:  per segment tie quota and output offsets (segments are in index
//          order, so offsets preserve index order)
//   write: ordered compaction (one warp per segment, ballots) of selected and
//          discarded entries; discards are scaled by the residual share with
//          an explicitly rounded multiply (no FMA contraction), matching
//          inc/residual.hpp:119.
#include "common.cuh"
#include "kernels.cuh"

namespace sdl {

namespace {

constexpr int kWarps = kThreads / 32;

__device__ __forceinline__ int resolve_mode(const SelTask& t) {
  if (!t.mode_from_cand) return t.mode;
  const int64_t need = t.budget_dev ? *t.budget_dev : t.budget;
  return (*t.cand_bad != 0 || *t.cand_total < need) ? 1 : 0;
}

// Is the pass-0 histogram already built by the dividing candidate pass?  In
// candidate mode yes; after a candidate-list overflow (flags == 2) too: every
// chunk histogrammed its candidates before the overflow was detected, and
// the L-th largest key lies above the pre-threshold because more than the
// capacity (> L) of entries passed it.
__device__ __forceinline__ bool hist0_ready(const SelTask& t, int mode) {
  if (!t.cand_hist) return false;
  return mode == 0 || *t.cand_bad == 2;
}

__device__ __forceinline__ int nseg_of(const SelTask& t, int mode) {
  return mode == 1 ? t.dnseg : t.nseg * t.tiles;
}

// Segment s of a task.  Explicit inputs are cut further into `tiles` tiles
// of <= kTile entries per input segment (tile order == index order), so every
// warp-level work item is small regardless of how the input was segmented.
__device__ __forceinline__ void seg_bounds(const SelTask& t, int mode, int s, int& off,
                                           int& cnt) {
  if (mode == 1) {
    off = s * t.dstride;
    const int c = t.dn - off;
    cnt = c < 0 ? 0 : (c > t.dstride ? t.dstride : c);
  } else {
    const int tiles = t.tiles;
    const int si = s / tiles, ti = s - si * tiles;
    int o, c;
    o = t.seg_off ? t.seg_off[si] : si * t.stride;
    if (t.seg_cnt) {
      c = t.seg_cnt[si];
    } else {
      c = *t.count - o;
      c = c < 0 ? 0 : (c > t.stride ? t.stride : c);
    }
    off = o + ti * kTile;
    c -= ti * kTile;
    cnt = c < 0 ? 0 : (c > kTile ? kTile : c);
  }
}

__device__ __forceinline__ float seg_val(const SelTask& t, int mode, int p) {
  return mode == 1 ? t.dval[p] : t.val[p];
}
__device__ __forceinline__ int32_t seg_idx(const SelTask& t, int mode, int p) {
  return mode == 1 ? t.dbase + p : t.idx[p];
}

template <int PASS>
struct Digit {
  static constexpr int shift = PASS == 0 ? 20 : (PASS == 1 ? 9 : 0);
  static constexpr int nbins = PASS == 2 ? 512 : 2048;
};

// warp-aggregated shared-memory histogram increment
__device__ __forceinline__ void hist_add(uint32_t* h, uint32_t bin, bool active) {
  const uint32_t am = __ballot_sync(0xffffffffu, active);
  if (!active) return;
  const uint32_t peers = __match_any_sync(am, bin);
  const int leader = __ffs(peers) - 1;
  if ((int)(threadIdx.x & 31) == leader) atomicAdd(&h[bin], (uint32_t)__popc(peers));
}

// ---------------------------------------------------------------------------
template <int PASS>
__global__ void __launch_bounds__(kThreads) k_sel_hist(const SelTask* __restrict__ tasks) {
  const SelTask& t = tasks[blockIdx.y];
  SelScratch* sc = t.scr;
  int mode;
  uint32_t prefix = 0, pmask = 0;
  if (PASS == 0) {
    mode = resolve_mode(t);
    if (hist0_ready(t, mode)) return;   // built by the candidate pass
  } else {
    if (sc->all) return;
    mode = sc->mode;
    prefix = sc->prefix;
    pmask = sc->pmask;
  }
  const int nseg = nseg_of(t, mode);
  const int per = (nseg + gridDim.x - 1) / gridDim.x;
  const int s0 = blockIdx.x * per;
  if (s0 >= nseg) return;
  const int s1 = min(nseg, s0 + per);
  constexpr int NB = Digit<PASS>::nbins;
  constexpr int SH = Digit<PASS>::shift;
  __shared__ uint32_t h[NB];
  for (int b = threadIdx.x; b < NB; b += blockDim.x) h[b] = 0;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int s = s0 + warp; s < s1; s += kWarps) {
    int off, cnt;
    seg_bounds(t, mode, s, off, cnt);
    for (int j0 = 0; j0 < cnt; j0 += 32) {
      const int j = j0 + lane;
      uint32_t key = 0;
      if (j < cnt) key = mag_key(seg_val(t, mode, off + j));
      const bool in = j < cnt && (key & pmask) == prefix;
      hist_add(h, (key >> SH) & (NB - 1), in);
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < NB; b += blockDim.x)
    if (h[b]) atomicAdd(&sc->hist[b], h[b]);
}

// One CTA per task: locate the digit holding the rank-th largest key.
template <int PASS>
__global__ void __launch_bounds__(kThreads) k_sel_find(const SelTask* __restrict__ tasks) {
  const SelTask& t = tasks[blockIdx.x];
  SelScratch* sc = t.scr;
  constexpr int NB = Digit<PASS>::nbins;
  constexpr int SH = Digit<PASS>::shift;
  constexpr int BPT = NB / kThreads;
  __shared__ long long lscr[32];
  __shared__ long long suf[kThreads];
  if (PASS > 0 && sc->all) return;
  int mode = 0;
  const uint32_t* src = sc->hist;
  if (PASS == 0) {
    mode = resolve_mode(t);
    if (hist0_ready(t, mode)) src = t.cand_hist;
  }
  uint32_t c[BPT];
  long long mine = 0;
#pragma unroll
  for (int q = 0; q < BPT; ++q) {
    c[q] = src[threadIdx.x * BPT + q];
    mine += c[q];
  }
#pragma unroll
  for (int q = 0; q < BPT; ++q) {
    sc->hist[threadIdx.x * BPT + q] = 0;
    if (PASS == 0 && t.cand_hist) t.cand_hist[threadIdx.x * BPT + q] = 0;
  }
  int64_t rank, cnt_gt;
  uint32_t prefix, pmask;
  if (PASS == 0) {
    const long long total = block_sum_ll(mine, lscr);
    const int64_t budget = t.budget_dev ? *t.budget_dev : t.budget;
    if (threadIdx.x == 0) {
      sc->total = total;
      sc->budget = budget;
      sc->mode = mode;
      sc->cut_idx = -1;
      if (total <= budget) sc->all = 1;          // identity case, inc/sparse.hpp:143-146
      else if (budget <= 0) sc->all = 2;         // nothing kept
      else sc->all = 0;
      sc->prefix = 0;
      sc->pmask = 0;
      sc->rank = budget;
      sc->cnt_gt = 0;
    }
    __syncthreads();
    if (total <= budget || budget <= 0) return;
    rank = budget;
    cnt_gt = 0;
    prefix = 0;
    pmask = 0;
  } else {
    rank = sc->rank;
    cnt_gt = sc->cnt_gt;
    prefix = sc->prefix;
    pmask = sc->pmask;
  }
  __syncthreads();
  // above(tid) = count in the bins of all threads > tid (bins ascend with tid)
  const int r = blockDim.x - 1 - threadIdx.x;
  suf[r] = mine;
  __syncthreads();
  for (int o = 1; o < (int)blockDim.x; o <<= 1) {
    const long long add = threadIdx.x >= (unsigned)o ? suf[threadIdx.x - o] : 0;
    __syncthreads();
    suf[threadIdx.x] += add;
    __syncthreads();
  }
  const long long above = r > 0 ? suf[r - 1] : 0;
  if (above < rank && rank <= above + mine) {
    long long cum = above;
    for (int q = BPT - 1; q >= 0; --q) {
      if (cum + (long long)c[q] >= rank) {
        const uint32_t digit = threadIdx.x * BPT + q;
        sc->prefix = prefix | (digit << SH);
        sc->pmask = pmask | ((uint32_t)(NB - 1) << SH);
        sc->rank = rank - cum;
        sc->cnt_gt = cnt_gt + cum;
        break;
      }
      cum += c[q];
    }
  }
}

// Per segment (one warp): #{key > T}, #{key == T}
__global__ void __launch_bounds__(kThreads) k_sel_count(const SelTask* __restrict__ tasks) {
  const SelTask& t = tasks[blockIdx.y];
  const SelScratch* sc = t.scr;
  const int mode = sc->mode;
  const int nseg = nseg_of(t, mode);
  const int all = sc->all;
  const uint32_t T = sc->prefix;
  const int lane = threadIdx.x & 31;
  for (int s = blockIdx.x * kWarps + (threadIdx.x >> 5); s < nseg; s += gridDim.x * kWarps) {
    int off, cnt;
    seg_bounds(t, mode, s, off, cnt);
    int gt = 0, eq = 0;
    if (all == 1) {
      gt = cnt;
    } else if (all == 0) {
      for (int j = lane; j < cnt; j += 32) {
        const uint32_t key = mag_key(seg_val(t, mode, off + j));
        gt += key > T;
        eq += key == T;
      }
      gt = __reduce_add_sync(0xffffffffu, gt);
      eq = __reduce_add_sync(0xffffffffu, eq);
    }
    if (lane == 0) {
      t.seg_gt[s] = gt;
      t.seg_eq[s] = eq;
    }
  }
}

// One CTA per task: tie quotas and output offsets per segment.
__global__ void __launch_bounds__(1024) k_sel_scan(const SelTask* __restrict__ tasks) {
  const SelTask& t = tasks[blockIdx.x];
  SelScratch* sc = t.scr;
  const int mode = sc->mode;
  const int nseg = nseg_of(t, mode);
  const int all = sc->all;
  const int64_t need_eq = all == 0 ? sc->rank : 0;
  __shared__ int scratch[40];
  int eq_carry = 0, sel_carry = 0, cnt_carry = 0;
  for (int s0 = 0; s0 < nseg; s0 += blockDim.x) {
    const int s = s0 + threadIdx.x;
    int gt = 0, eq = 0, cnt = 0;
    if (s < nseg) {
      int off;
      seg_bounds(t, mode, s, off, cnt);
      gt = t.seg_gt[s];
      eq = t.seg_eq[s];
    }
    int teq, tsel, tcnt;
    const int eq_before = eq_carry + block_exscan(eq, scratch, &teq);
    long long q = need_eq - eq_before;
    const int take = q <= 0 ? 0 : (q >= eq ? eq : (int)q);
    const int sel = gt + take;
    const int sel_off = sel_carry + block_exscan(sel, scratch, &tsel);
    const int cnt_off = cnt_carry + block_exscan(cnt, scratch, &tcnt);
    if (s < nseg) {
      t.seg_take[s] = take;
      t.seg_sel_off[s] = sel_off;
      t.seg_dis_off[s] = cnt_off - sel_off;
    }
    eq_carry += teq;
    sel_carry += tsel;
    cnt_carry += tcnt;
  }
  if (threadIdx.x == 0) {
    *t.sel_cnt = sel_carry;
    if (t.dis_cnt) *t.dis_cnt = cnt_carry - sel_carry;
    if (t.total_out) *t.total_out = sc->total;
  }
}

// Ordered compaction, one warp per segment.
__global__ void __launch_bounds__(kThreads) k_sel_write(const SelTask* __restrict__ tasks) {
  const SelTask& t = tasks[blockIdx.y];
  SelScratch* sc = t.scr;
  const int mode = sc->mode;
  const int nseg = nseg_of(t, mode);
  const int all = sc->all;
  const uint32_t T = sc->prefix;
  const float w = t.weight;
  const bool want_dis = t.dis_idx != nullptr;
  const int lane = threadIdx.x & 31;
  const uint32_t lt = lanemask_lt();
  int cut = -1;
  for (int s = blockIdx.x * kWarps + (threadIdx.x >> 5); s < nseg; s += gridDim.x * kWarps) {
    int off, cnt;
    seg_bounds(t, mode, s, off, cnt);
    if (cnt == 0) continue;
    const int sel_base = t.seg_sel_off[s];
    const int dis_base = t.seg_dis_off[s];
    const int take = t.seg_take[s];
    int eq_seen = 0, sel_seen = 0;
    for (int j0 = 0; j0 < cnt; j0 += 32) {
      const int j = j0 + lane;
      const bool valid = j < cnt;
      float v = 0.f;
      int32_t ix = 0;
      uint32_t key = 0;
      if (valid) {
        v = seg_val(t, mode, off + j);
        ix = seg_idx(t, mode, off + j);
        key = mag_key(v);
      }
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
  if (all == 0) {
    cut = __reduce_max_sync(0xffffffffu, cut);
    if (lane == 0 && cut >= 0) atomicMax(&sc->cut_idx, cut);
  }
}

inline int clampi(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }

}  // namespace

int sel_prepare(SelTask& t, int max_seg_len) {
  t.tiles = max_seg_len <= kTile ? 1 : (max_seg_len + kTile - 1) / kTile;
  if (t.dn > 0) {
    t.dstride = kTile;
    t.dnseg = (t.dn + kTile - 1) / kTile;
  }
  return t.nseg * t.tiles;
}

int sel_scratch_segments(const SelTask& t) {
  const int ne = t.nseg * t.tiles;
  return ne > t.dnseg ? ne : t.dnseg;
}

int sel_grid_segments(const SelTask& t) {
  // grids are sized for the expected (explicit / candidate) input; the dense
  // fallback of the dividing select grid-strides over its larger range
  if (t.mode == 1 && !t.mode_from_cand) return t.dnseg;
  return t.nseg * t.tiles;
}

int launch_select(const SelTask* tasks_dev, int ntask, int max_nseg, cudaStream_t s) {
  if (ntask <= 0) return 0;
  // histogram CTAs cover ~16 segments each; count/write use a warp per segment
  const int hx = clampi((max_nseg + 15) / 16, 1, 1184);
  const int wx = clampi((max_nseg + kWarps - 1) / kWarps, 1, 4096);
  dim3 gh(hx, ntask), gw(wx, ntask);
  k_sel_hist<0><<<gh, kThreads, 0, s>>>(tasks_dev);
  k_sel_find<0><<<ntask, kThreads, 0, s>>>(tasks_dev);
  k_sel_hist<1><<<gh, kThreads, 0, s>>>(tasks_dev);
  k_sel_find<1><<<ntask, kThreads, 0, s>>>(tasks_dev);
  k_sel_hist<2><<<gh, kThreads, 0, s>>>(tasks_dev);
  k_sel_find<2><<<ntask, kThreads, 0, s>>>(tasks_dev);
  k_sel_count<<<gw, kThreads, 0, s>>>(tasks_dev);
  k_sel_scan<<<ntask, 1024, 0, s>>>(tasks_dev);
  k_sel_write<<<gw, kThreads, 0, s>>>(tasks_dev);
  return 9;
}

}  // namespace sdl
