// Wide select: one deterministic top-L selection spread over the whole GPU.
//
// Semantics: inc/sparse.hpp:136-162 (top_k_select) -- keep the min(budget,
// nnz) entries first in the order (|v| desc, index asc), return the kept and
// the discarded ones, each in index order; discards scaled by the residual
// share with an explicitly rounded multiply (inc/residual.hpp:104-124).
//
// The cluster select (select.cu) gives one task at most 16 CTAs; a stage of
// the Spar-Reduce-Scatter with one worker per GPU has one or two tasks, so
// most SMs would idle.  Here a task is cut into tiles (groups of its input
// segments, in index order) and every kernel runs one CTA per tile:
//   k_wsel_hist    level-1 histogram of the magnitude keys, 2048 bins over a
//                  window: above the dividing pre-threshold, or around the
//                  task's previous threshold (full key range, key >> 20,
//                  when there is none); a per-CTA shared histogram over 16
//                  tiles, flushed once (fusing it into the candidate pass
//                  as global reductions was measured 1.5x slower: the hot
//                  bins serialise)
//   k_wsel_gather  every CTA locates the bin holding the L-th key (suffix
//                  scan of the histogram, identical in every CTA), counts its
//                  tile's entries above that bin and appends the bin's
//                  entries (key, index, tile) to the bin buffer; the last CTA
//                  of the task (arrival counter) selects the exact boundary
//                  entry inside the bin -- a radix select on the composite
//                  (key << 32 | ~index), i.e. key desc, index asc -- adds the
//                  in-bin winners to their tiles, scans the per-tile output
//                  offsets and records the selection (threshold T, largest
//                  kept index among key == T) for sel_member and the
//                  dividing history
//   k_wsel_write   ordered compaction of every tile: warp ballots place the
//                  kept and the discarded entries; the last CTA of the task
//                  writes the counts and publishes the block to its peers
// A task the wide path cannot finish -- dividing candidates incomplete,
// threshold outside the dividing window, bin buffer overflow (massive key
// ties) -- is marked kWFallback and k_select (launched right after) selects
// it; every other task makes k_select return at once.
#include <algorithm>
#include <climits>
#include <cstdio>
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"
#include "wsel_common.cuh"

namespace sdl {

namespace {

constexpr int kWThreads = 256;
constexpr int kWWarps = kWThreads / 32;
constexpr int kWMaxGroup = 64;     // segments per tile (bound of the write pass tables)
constexpr int kWSmemSel = 2048;    // bin entries the finisher selects in shared memory

__device__ __forceinline__ int w_nseg(const WScratch& w) {
  int n = w.nseg;
  if (w.nseg_dev) n = min(n, *w.nseg_dev);
  else if (!w.seg_cnt && w.count) n = min(n, (*w.count + w.stride - 1) / w.stride);
  return n < 0 ? 0 : n;
}

__device__ __forceinline__ void w_seg(const WScratch& w, int s, int& off, int& cnt) {
  off = w.seg_off ? w.seg_off[s] : s * w.stride;
  int c = w.seg_cnt ? w.seg_cnt[s] : *w.count - off;
  c = c > w.stride ? w.stride : c;
  cnt = c < 0 ? 0 : c;
}

__device__ __forceinline__ unsigned long long w_comp(uint32_t key, int32_t idx) {
  return ((unsigned long long)key << 32) | (unsigned long long)(0x7fffffffu - (uint32_t)idx);
}

// A tile of a task: its segments' input offsets and the exclusive prefix of
// their lengths, in shared memory.  Entries are addressed flat (tile order ==
// index order): the CTA sweeps them in rounds of kWRound, warp w owning
// flat [w * kWPer * 32, (w + 1) * kWPer * 32) of a round, lane l element
// i * 32 + l of that -- kWPer coalesced loads in flight per thread.
constexpr int kWPer = 16;
constexpr int kWRound = kWThreads * kWPer;
struct TileMap {
  int n;
  int nseg;
  int off[kWMaxGroup];
  int pre[kWMaxGroup + 1];
};

__device__ void tile_map_load(const WScratch& w, int q, int nseg_total, TileMap& tm) {
  const int G = w.group;
  const int s0 = q * G;
  const int ns = max(0, min(nseg_total, s0 + G) - s0);
  __shared__ int cnts[kWMaxGroup];
  if ((int)threadIdx.x < ns) {
    int off, cnt;
    w_seg(w, s0 + threadIdx.x, off, cnt);
    tm.off[threadIdx.x] = off;
    cnts[threadIdx.x] = cnt;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int a = 0;
    for (int i = 0; i < ns; ++i) {
      tm.pre[i] = a;
      a += cnts[i];
    }
    tm.pre[ns] = a;
    tm.n = a;
    tm.nseg = ns;
  }
  __syncthreads();
}

// input position of flat entry p (0 <= p < tm.n): the last segment starting
// at or before p (empty segments share their successor's start)
// Branch-free (a fixed, unrolled search) so that a thread's kWPer loads are
// all issued before the first one is used.
__device__ __forceinline__ int tile_src(const TileMap& tm, int p) {
  int lo = 0;
#pragma unroll
  for (int step = kWMaxGroup / 2; step >= 1; step >>= 1) {
    const int mid = lo + step;
    lo = (mid < tm.nseg && tm.pre[mid] <= p) ? mid : lo;
  }
  return tm.off[lo] + (p - tm.pre[lo]);
}

// The need-th largest composite value among c[0, n) (1 <= need <= n), by a
// radix select over 8-bit digits; whole CTA.  Entries are read from global
// memory until the candidates fit the shared buffer.
__device__ unsigned long long w_select_kth(const unsigned long long* __restrict__ c, int n,
                                           long long need, int* scratch) {
  __shared__ unsigned long long buf[kWSmemSel];
  __shared__ uint32_t h[256];
  __shared__ int s_m, s_d;
  __shared__ long long s_need;
  __shared__ unsigned long long s_or, s_and;
  const int tid = threadIdx.x;
  // constant leading bits: skip the digits every entry shares
  unsigned long long o = 0, a = ~0ull;
  for (int i = tid; i < n; i += kWThreads) {
    const unsigned long long x = __ldcg(c + i);
    o |= x;
    a &= x;
  }
  if (tid == 0) {
    s_or = 0;
    s_and = ~0ull;
  }
  __syncthreads();
  atomicOr(&s_or, o);
  atomicAnd(&s_and, a);
  __syncthreads();
  const unsigned long long diff = s_or ^ s_and;
  if (diff == 0) return s_or;   // all equal
  int shift = ((63 - __clzll(diff)) / 8) * 8;
  unsigned long long prefix = s_and & ~((2ull << (shift + 7)) - 1) ;
  // (bits above the first varying digit are common: prefix holds them)
  if (shift + 8 >= 64) prefix = 0;
  bool in_smem = n <= kWSmemSel;
  int m = n;
  if (in_smem) {
    for (int i = tid; i < n; i += kWThreads) buf[i] = __ldcg(c + i);
    __syncthreads();
  }
  for (; shift >= 0; shift -= 8) {
    const unsigned long long hi_mask = shift + 8 >= 64 ? 0ull : ~((1ull << (shift + 8)) - 1);
    h[tid] = 0;
    __syncthreads();
    for (int i = tid; i < m; i += kWThreads) {
      const unsigned long long x = in_smem ? buf[i] : __ldcg(c + i);
      if ((x & hi_mask) == prefix) atomicAdd(&h[(x >> shift) & 255u], 1u);
    }
    __syncthreads();
    // digit holding rank `need`, counting from the top digit down
    const int dgt = 255 - tid;
    const int cnt = (int)h[dgt];
    int tot = 0;
    const int ex = block_exscan(cnt, scratch, &tot);
    if (ex < need && need <= ex + cnt) {
      s_d = dgt;
      s_need = need - ex;
      s_m = cnt;
    }
    __syncthreads();
    const int d = s_d;
    need = s_need;
    const int nm = s_m;
    __syncthreads();   // every thread has read the digit before s_m is reused
    prefix |= (unsigned long long)d << shift;
    if (shift == 0) break;
    if (!in_smem && nm <= kWSmemSel) {   // gather the survivors on chip
      const unsigned long long mask2 = ~((1ull << shift) - 1);
      if (tid == 0) s_m = 0;
      __syncthreads();
      for (int i = tid; i < m; i += kWThreads) {
        const unsigned long long x = __ldcg(c + i);
        if ((x & mask2) == prefix) buf[atomicAdd(&s_m, 1)] = x;
      }
      __syncthreads();
      m = s_m;
      in_smem = true;
    }
    __syncthreads();
  }
  return prefix;
}

// ---------------------------------------------------------------------------
// Histogram pass.  Every CTA adds its tile's key counts; the last CTA of the
// task (the decider) fixes the run state, the boundary bin and this run's
// geometry in the scratch, then zeroes the histogram for the next run.
__global__ void __launch_bounds__(kWThreads) k_wsel_hist(const SelTask* __restrict__ tasks) {
  pdl_enter();
  const SelTask& t = tasks[blockIdx.y];
  WScratch* __restrict__ ws = t.ws;
  if (ws->by_merge) return;   // histogrammed and decided by the merge feeding it
  const int nseg = w_nseg(*ws);
  const int q = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  int mode;
  uint32_t base, shift;
  w_geometry(t, *ws, mode, base, shift);
  __shared__ TileMap tm;
  __shared__ uint32_t h[kWBins];
  __shared__ uint32_t s_ab[2];
  __shared__ int s_last;
  __shared__ int scratch[40];
  __shared__ long long lsh[3 * 32];
  if (q * ws->group < nseg) {
    peer_wait(t.ps);
    for (int b = tid; b < kWBins; b += kWThreads) h[b] = 0;
    if (tid < 2) s_ab[tid] = 0;
    tile_map_load(*ws, q, nseg, tm);
    const float* __restrict__ val = ws->val;
    uint32_t nbelow = 0, nabove = 0;
    for (int r0 = 0; r0 < tm.n; r0 += kWRound) {
      const int p0 = r0 + warp * (kWPer * 32) + lane;
      int src[kWPer];
#pragma unroll
      for (int i = 0; i < kWPer; ++i) src[i] = tile_src(tm, min(p0 + i * 32, tm.n - 1));
      float v[kWPer];
#pragma unroll
      for (int i = 0; i < kWPer; ++i) v[i] = __ldcg(val + src[i]);   // (clamped: in bounds)
#pragma unroll
      for (int i = 0; i < kWPer; ++i)
        if (p0 + i * 32 < tm.n) {
          const int b = w_bin(mode, base, shift, mag_key(v[i]));
          if (b < 0) ++nbelow;
          else if (b >= kWBins) ++nabove;
          else atomicAdd(&h[b], 1u);
        }
    }
    nbelow = __reduce_add_sync(0xffffffffu, nbelow);
    nabove = __reduce_add_sync(0xffffffffu, nabove);
    if (lane == 0 && (nbelow | nabove)) {
      atomicAdd(&s_ab[0], nbelow);
      atomicAdd(&s_ab[1], nabove);
    }
    __syncthreads();
    for (int b = tid; b < kWBins; b += kWThreads)
      if (h[b]) atomicAdd(&ws->hist[b], h[b]);
    if (tid == 0) {
      if (s_ab[0]) atomicAdd(&ws->below, s_ab[0]);
      if (s_ab[1]) atomicAdd(&ws->above, s_ab[1]);
    }
  }
  // ---- arrival; the decider
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    s_last = (int)(atomicAdd(&ws->harrive, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const int64_t budget = t.budget_dev ? *t.budget_dev : t.budget;
  long long total = w_hist_total(ws, lsh) + __ldcg(&ws->above) + __ldcg(&ws->below);
  bool bad = false;
  if (ws->is_div) {
    total = *t.cand_total;
    // incomplete candidates: dense fallback in k_select (bit 2, the cluster
    // select's work list, does not concern the wide select)
    bad = (*t.cand_bad & 3) != 0 || total < budget;
  }
  w_decide(ws, total, bad, budget, mode, base, shift, scratch, lsh);
}

// ---------------------------------------------------------------------------
// Gather pass: entries above the boundary bin are counted per tile, the
// bin's entries collected.  The last CTA of the task (the finisher) selects
// the boundary entry, fixes the per-tile output offsets and records the
// selection.
__global__ void __launch_bounds__(kWThreads, 2) k_wsel_gather(const SelTask* __restrict__ tasks) {
  pdl_enter();
  const SelTask& t = tasks[blockIdx.y];
  WScratch* __restrict__ ws = t.ws;
  __shared__ int scratch[40];
  __shared__ int s_last;
  __shared__ unsigned int s_na;
  __shared__ TileMap tm;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  int state = ws->state;
  const int mode = ws->run_mode;
  const uint32_t base = ws->run_base, shift = ws->run_shift;
  const int bstar = ws->bstar;
  const int nseg = w_nseg(*ws);
  const int G = ws->group;
  const int ntiles = (nseg + G - 1) / G;
  const int q = blockIdx.x;
  if (tid == 0) s_na = 0;
  if (q < ntiles && state != kWFallback) {
    peer_wait(t.ps);
    tile_map_load(*ws, q, nseg, tm);
    unsigned int na = 0;
    if (state == kWOk) {
      const float* __restrict__ val = ws->val;
      const int32_t* __restrict__ idx = ws->idx;
      unsigned long long* __restrict__ bin_c = ws->bin_c;
      int32_t* __restrict__ bin_tile = ws->bin_tile;
      const int bin_cap = ws->bin_cap;
      const uint32_t lt = lanemask_lt();
      for (int r0 = 0; r0 < tm.n; r0 += kWRound) {
        const int p0 = r0 + warp * (kWPer * 32) + lane;
        int src[kWPer];
#pragma unroll
        for (int i = 0; i < kWPer; ++i) src[i] = tile_src(tm, min(p0 + i * 32, tm.n - 1));
        float v[kWPer];
#pragma unroll
        for (int i = 0; i < kWPer; ++i) v[i] = __ldcg(val + src[i]);   // (clamped: in bounds)
#pragma unroll
        for (int i = 0; i < kWPer; ++i) {
          const uint32_t key = mag_key(v[i]);
          const int b = p0 + i * 32 < tm.n ? w_bin(mode, base, shift, key) : -1;
          na += b > bstar;
          const bool in = b == bstar;
          const uint32_t bal = __ballot_sync(0xffffffffu, in);
          if (bal) {
            int pb = 0;
            if (lane == 0) pb = (int)atomicAdd(&ws->bin_n, (unsigned)__popc(bal));
            pb = __shfl_sync(0xffffffffu, pb, 0);
            if (in) {
              const int pp = pb + __popc(bal & lt);
              if (pp < bin_cap) {
                bin_c[pp] = w_comp(key, __ldcg(idx + src[i]));
                bin_tile[pp] = q;
              }
            }
          }
        }
      }
    }
    na = __reduce_add_sync(0xffffffffu, na);
    if (lane == 0 && na) atomicAdd(&s_na, na);
    __syncthreads();
    if (tid == 0) {
      ws->tile_n[q] = tm.n;
      ws->tile_sel[q] = state == kWOk ? (int)s_na : (state == kWAll ? tm.n : 0);
    }
  }
  // ---- arrival; the finisher
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    s_last = (int)(atomicAdd(&ws->arrive, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  SelScratch* sc = t.scr;
  const int64_t budget = t.budget_dev ? *t.budget_dev : t.budget;
  if (state == kWOk) {
    const long long nb = (long long)__ldcg(&ws->bin_n);
    if (nb > ws->bin_cap || nb != (long long)ws->bin_expect)
      state = kWFallback;   // bin buffer overflow (massive key ties): k_select
  }
#ifdef SPARDL_WSEL_DEBUG
  if (tid == 0)
    printf("wsel task %d div %d mode %d state %d total %lld budget %lld bstar %d before %lld "
           "bin_n %u expect %u cap %d base %u shift %u ntiles %d\n",
           (int)blockIdx.y, ws->is_div, mode, state, ws->total_in, (long long)budget, bstar,
           ws->before, __ldcg(&ws->bin_n), ws->bin_expect, ws->bin_cap, base, shift, ntiles);
#endif
  unsigned long long cstar = 0;
  if (state == kWOk) {
    const int nb = (int)__ldcg(&ws->bin_n);
    cstar = w_select_kth(ws->bin_c, nb, budget - ws->before, scratch);
    for (int i = tid; i < nb; i += kWThreads)
      if (__ldcg(ws->bin_c + i) >= cstar) atomicAdd(ws->tile_sel + __ldcg(ws->bin_tile + i), 1);
    __threadfence();
    __syncthreads();
  }
  long long tot_sel = 0, tot_all = 0;
  if (state != kWFallback) {
    int carry_s = 0, carry_d = 0;
    for (int q0 = 0; q0 < ntiles; q0 += kWThreads) {
      const int qq = q0 + tid;
      const int nn = qq < ntiles ? __ldcg(ws->tile_n + qq) : 0;
      const int ns = qq < ntiles ? __ldcg(ws->tile_sel + qq) : 0;
      int ts = 0, td = 0;
      const int es = block_exscan(ns, scratch, &ts);
      const int ed = block_exscan(nn - ns, scratch, &td);
      if (qq < ntiles) {
        ws->tile_sel_off[qq] = carry_s + es;
        ws->tile_dis_off[qq] = carry_d + ed;
      }
      carry_s += ts;
      carry_d += td;
    }
    tot_sel = carry_s;
    tot_all = (long long)carry_s + carry_d;
  }
  // ---- the selection record and the dividing history
  if (tid == 0) {
    const uint32_t T = (uint32_t)(cstar >> 32);
    const int32_t cut = (int32_t)(0x7fffffffu - (uint32_t)(cstar & 0xffffffffull));
    ws->state = state;
    if (state == kWFallback && ws->handed_back) atomicAdd(ws->handed_back, 1ull);
    ws->T = T;
    ws->cut = cut;
    ws->ntiles = ntiles;
    ws->total = tot_all;
    ws->total_sel = tot_sel;
    ws->bin_n = 0;
    ws->arrive = 0;
    if (state != kWFallback) {
      const int all = state == kWAll ? 1 : (state == kWNone ? 2 : 0);
      sc->mode = 0;
      sc->total = tot_all;
      sc->prefix = state == kWOk ? T : 0;
      sc->cut_idx = state == kWOk ? cut : -1;
      sc->all = all;
      if (ws->is_div) {
        if (all == 1) {
          // exactly L candidates, all kept: the selection is {key >= pre-threshold}
          sc->all = 0;
          sc->prefix = *t.pre_key_dev;
          sc->cut_idx = INT_MAX;
        }
        if (t.div_hist)
          update_history(t.div_hist, 0, all, state == kWOk ? T : 0u, *t.pre_key_dev,
                         ws->total_in, budget);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Write pass: ordered compaction of every tile (round by round: warp ballots,
// then the warps' totals), kept entries to the output block (and the peers'
// copies), discarded ones scaled to the discard list.
constexpr int kWPerW = 8;   // entries per thread and round here (register budget)
constexpr int kWRoundW = kWThreads * kWPerW;

__global__ void __launch_bounds__(kWThreads, 3) k_wsel_write(const SelTask* __restrict__ tasks) {
  pdl_enter();
  const SelTask& t = tasks[blockIdx.y];
  const WScratch* __restrict__ ws = t.ws;
  const int state = ws->state;
  if (state == kWFallback) return;   // k_select selects this task
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q = blockIdx.x;
  const int ntiles = ws->ntiles;
  const int npush = t.npush;
  __shared__ TileMap tm;
  __shared__ int wsum[2][kWWarps];
  __shared__ int s_last;
  if (q < ntiles) {
    peer_wait(t.ps);
    tile_map_load(*ws, q, w_nseg(*ws), tm);
    const uint32_t T = ws->T;
    const int32_t cut = ws->cut;
    int ks = ws->tile_sel_off[q];   // output positions of the round (CTA-uniform)
    int kd = ws->tile_dis_off[q];
    int32_t* __restrict__ sel_idx = t.sel_idx;
    float* __restrict__ sel_val = t.sel_val;
    int32_t* __restrict__ dis_idx = t.dis_idx;
    float* __restrict__ dis_val = t.dis_val;
    unsigned char* const* push_base = t.push_base;
    const size_t push_voff = 16 + 4 * (size_t)t.push_cap;
    const float w = t.weight;
    const uint32_t lt = lanemask_lt();
    const float* __restrict__ val = ws->val;
    const int32_t* __restrict__ idx = ws->idx;
    for (int r0 = 0; r0 < tm.n; r0 += kWRoundW) {
      const int p0 = r0 + warp * (kWPerW * 32) + lane;
      int src[kWPerW];
#pragma unroll
      for (int i = 0; i < kWPerW; ++i) src[i] = tile_src(tm, min(p0 + i * 32, tm.n - 1));
      float v[kWPerW];
      int32_t ix[kWPerW];
#pragma unroll
      for (int i = 0; i < kWPerW; ++i) {   // (clamped: in bounds; past the tile: ix = -1)
        v[i] = __ldcg(val + src[i]);
        ix[i] = __ldcg(idx + src[i]);
      }
#pragma unroll
      for (int i = 0; i < kWPerW; ++i)
        if (p0 + i * 32 >= tm.n) ix[i] = -1;
      auto keep = [&](int i) {
        const uint32_t key = mag_key(v[i]);
        return ix[i] >= 0 && (state == kWAll ||
                              (state == kWOk && (key > T || (key == T && ix[i] <= cut))));
      };
      int cs = 0, cd = 0;
#pragma unroll
      for (int i = 0; i < kWPerW; ++i) {
        const bool kp = keep(i);
        cs += __popc(__ballot_sync(0xffffffffu, kp));
        cd += __popc(__ballot_sync(0xffffffffu, ix[i] >= 0 && !kp));
      }
      if (lane == 0) {
        wsum[0][warp] = cs;
        wsum[1][warp] = cd;
      }
      __syncthreads();
      int bs = ks, bdd = kd, ts = 0, td = 0;
#pragma unroll
      for (int u = 0; u < kWWarps; ++u) {
        const int a0 = wsum[0][u], a1 = wsum[1][u];
        if (u < warp) {
          bs += a0;
          bdd += a1;
        }
        ts += a0;
        td += a1;
      }
#pragma unroll
      for (int i = 0; i < kWPerW; ++i) {
        const bool kp = keep(i);
        const uint32_t bk = __ballot_sync(0xffffffffu, kp);
        const uint32_t bd = __ballot_sync(0xffffffffu, ix[i] >= 0 && !kp);
        if (kp) {
          const int p = bs + __popc(bk & lt);
          SPARDL_BOUND_CAP(p, t.sel_cap);
          sel_idx[p] = ix[i];
          sel_val[p] = v[i];
          if (npush > 0) SPARDL_BOUND_CAP(p, t.push_cap);
          for (int pp = 0; pp < npush; ++pp) {   // peers' copies (slot layout)
            unsigned char* b = push_base[pp];
            reinterpret_cast<int32_t*>(b + 16)[p] = ix[i];
            reinterpret_cast<float*>(b + push_voff)[p] = v[i];
          }
        } else if (dis_idx && ix[i] >= 0) {
          const int p = bdd + __popc(bd & lt);
          SPARDL_BOUND_CAP(p, t.dis_cap);
          dis_idx[p] = ix[i];
          dis_val[p] = __fmul_rn(v[i], w);
        }
        bs += __popc(bk);
        bdd += __popc(bd);
      }
      ks += ts;
      kd += td;
      __syncthreads();   // wsum is reused by the next round
    }
  }
  // ---- completion: the last CTA of the task writes the counts and publishes
  __syncthreads();
  if (tid == 0) {
    if (npush > 0) __threadfence_system();
    else __threadfence();
    s_last = (int)(atomicAdd(const_cast<uint32_t*>(&ws->wdone), 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last || tid != 0) return;
  const long long ns = ws->total_sel, nt = ws->total;
  *t.sel_cnt = (int32_t)ns;
  for (int p = 0; p < npush; ++p) *reinterpret_cast<int32_t*>(t.push_base[p]) = (int32_t)ns;
  if (t.dis_cnt) *t.dis_cnt = (int32_t)(nt - ns);
  if (t.total_out) *t.total_out = nt;
  const_cast<WScratch*>(ws)->wdone = 0;
  peer_publish(t.ps);   // (fences at system scope first)
}

// ---------------------------------------------------------------------------
// Cooperative form: the whole select of a task in ONE kernel, G CTAs per task
// (all co-resident: the grid never exceeds one wave), every CTA holding a
// contiguous 1/G of the task's entries (index order) in shared memory.
//   stage     the CTA's entries (4-byte cp.async, all in flight) into shared
//             memory -- the only global read of the input
//   3 levels  exact radix select of the magnitude key (11 / 11 / 9 bits):
//             shared histogram of the entries inside the prefix, flushed to a
//             per-task global histogram; task barrier; every CTA reads the
//             global histogram and finds the digit holding the rank itself
//   counts    #(key > T), #(key == T) per CTA; task barrier; every CTA takes
//             the exclusive prefix over the lower CTAs: its output offsets
//             and its share of the tie quota (ties go to the smaller index,
//             i.e. the earlier CTA)
//   write     ordered compaction from shared memory (warp ballots)
// The last CTA (arrival counter) records the selection, writes the counts,
// leaves the scratch zeroed and publishes.  Three kernel boundaries, the
// serial finisher and two re-reads of the input of the tiled form go away.
// A task whose entries do not fit (or a dividing select with incomplete
// candidates) is handed to k_select (kWFallback), as in the tiled form.
constexpr int kCoopThreads = 512;
constexpr int kCoopWarps = kCoopThreads / 32;
constexpr int kCoopMaxSeg = 8192;    // input segments per task (shared prefix table)
constexpr int kCoopMaxG = 512;       // CTAs per task
// coop scratch in the bin buffer (uint32 view): level-2 / level-3 histograms,
// the task barrier, per-CTA counts
constexpr int kCoopH2 = 0, kCoopH3 = 2048, kCoopBar = 2560, kCoopGt = 2564,
              kCoopEq = kCoopGt + kCoopMaxG, kCoopH2g = kCoopEq + kCoopMaxG,
              kCoopWords = kCoopH2g + 2048;

__device__ __forceinline__ uint32_t ld_acq_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// every CTA of the task: arrive, wait for all G (counter never reset mid-run)
__device__ __forceinline__ void coop_barrier(uint32_t* ctr, uint32_t target) {
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    atomicAdd(ctr, 1u);
    const unsigned long long t0 = gtime();
    unsigned ns = 32;
    while (ld_acq_u32(ctr) < target) {
      __nanosleep(ns);
      if (ns < 256) ns <<= 1;
      if (gtime() - t0 > 5000000000ull) __trap();   // a CTA never became resident
    }
  }
  __syncthreads();
}

// the digit of `nb` bins (descending) holding rank `rank` in the global
// histogram gh; returns it, *above = entries in higher bins (same in every CTA)
__device__ int coop_digit(const uint32_t* gh, int nb, long long rank, long long* above,
                          int* scratch) {
  __shared__ int s_d;
  __shared__ long long s_ab;
  const int per = nb / kCoopThreads;   // 4 (2048 bins) or 1 (512)
  // thread i: bins nb-1-i*per .. nb-per-i*per (descending order = thread order)
  uint32_t c[4];
  int mine = 0;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    c[u] = u < per ? __ldcg(gh + nb - 1 - ((int)threadIdx.x * per + u)) : 0u;
    mine += (int)c[u];
  }
  int tot;
  const int ex = block_exscan(mine, scratch, &tot);
  if (ex < rank && rank <= (long long)ex + mine) {
    long long cum = ex;
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (u < per) {
        if (cum + c[u] >= rank) {
          s_d = nb - 1 - ((int)threadIdx.x * per + u);
          s_ab = cum;
          break;
        }
        cum += c[u];
      }
  }
  __syncthreads();
  *above = s_ab;
  const int d = s_d;
  __syncthreads();
  return d;
}

__global__ void __launch_bounds__(kCoopThreads, 1)
    k_wsel_coop(const SelTask* __restrict__ tasks, int cap, int tabn) {
  pdl_enter();
  const SelTask& t = tasks[blockIdx.y];
  WScratch* __restrict__ ws = t.ws;
  const int G = gridDim.x, c = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  extern __shared__ __align__(16) unsigned char dsm[];
  // segment table sized for this launch's tasks (tabn >= every task's segments)
  int32_t* pre = reinterpret_cast<int32_t*>(dsm);               // [tabn + 1]
  int32_t* soff = pre + tabn + 1;                               // [tabn]
  float* sv = reinterpret_cast<float*>(soff + tabn + ((tabn + 1) & 1) + 2);   // [cap], 16 B aligned
  int32_t* si = reinterpret_cast<int32_t*>(sv + cap);           // [cap]
  __shared__ uint32_t h[kWBins];
  __shared__ int scratch[40];
  __shared__ int wcnt[3][kCoopWarps];
  __shared__ int s_flag;
  uint32_t* cs = reinterpret_cast<uint32_t*>(ws->bin_c);        // coop scratch
  uint32_t* bar = cs + kCoopBar;
  auto stamp = [&](int i) {   // phase timestamps of CTA 0 (-DSPARDL_STAMPS=1 builds)
    if (SPARDL_STAMPS && c == 0 && tid == 0) {
      long long ts;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts));
      t.scr->tstamp[i] = ts;
    }
  };
  stamp(0);
  peer_wait(t.ps);
  const int64_t budget = t.budget_dev ? *t.budget_dev : t.budget;
  // ---- the task's segments: offsets and the exclusive prefix of the counts
  const int nseg = min(w_nseg(*ws), tabn);   // (the planner sized tabn for every task)
  int carry = 0;
  for (int s0 = 0; s0 < nseg; s0 += kCoopThreads) {
    const int s = s0 + tid;
    int off = 0, cnt = 0;
    if (s < nseg) w_seg(*ws, s, off, cnt);
    int tt;
    const int e = carry + block_exscan(cnt, scratch, &tt);
    if (s < nseg) {
      pre[s] = e;
      soff[s] = off;
    }
    carry += tt;
  }
  if (tid == 0) pre[nseg] = carry;
  __syncthreads();
  const long long total = carry;
  // run state (identical in every CTA)
  int state;
  bool bad = false;
  if (ws->is_div) bad = (*t.cand_bad & 3) != 0 || total < budget;
  if (bad) state = kWFallback;
  else if (total <= budget) state = kWAll;
  else if (budget <= 0) state = kWNone;
  else state = ((total + G - 1) / G > cap && (!ws->ov_val || total > ws->ov_cap)) ? kWFallback
                                                                                 : kWOk;
  if (state == kWFallback) {   // k_select selects this task (no barrier was entered)
    if (c == 0 && tid == 0) {
      ws->state = kWFallback;
      if (ws->handed_back) atomicAdd(ws->handed_back, 1ull);
    }
    return;
  }
  const int e0 = (int)(total * c / G), e1 = (int)(total * (c + 1) / G);
  const int n = state == kWOk ? e1 - e0 : 0;
  // entry q of this CTA: shared memory below `cap`, the overflow scratch past it
  float* __restrict__ ovv = ws->ov_val;
  int32_t* __restrict__ ovi = ws->ov_idx;
  auto getv = [&](int q) { return q < cap ? sv[q] : __ldcg(ovv + e0 + q); };
  auto geti = [&](int q) { return q < cap ? si[q] : __ldcg(ovi + e0 + q); };
  // ---- stage this CTA's entries (flat positions e0..e1, index order): warp w
  // walks its 1/16 of the range segment by segment (one search for the first)
  if (n > 0) {
    const int a = (int)((long long)n * warp / kCoopWarps);
    const int b = (int)((long long)n * (warp + 1) / kCoopWarps);
    if (a < b) {
      int p = e0 + a;
      int lo = 0, hi = nseg - 1;   // last segment with pre[s] <= p
      while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (pre[mid] <= p) lo = mid;
        else hi = mid - 1;
      }
      const float* __restrict__ gv = ws->val;
      const int32_t* __restrict__ gi = ws->idx;
      for (int sg = lo; p < e0 + b; ++sg) {
        const int upto = min(pre[sg + 1], e0 + b);
        const int base = soff[sg] - pre[sg];
        for (int x = p + lane; x < upto; x += 32) {
          const int q = x - e0;
          if (q < cap) {
            const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(sv + q));
            const unsigned sb = static_cast<unsigned>(__cvta_generic_to_shared(si + q));
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sa), "l"(gv + base + x)
                         : "memory");
            asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(sb), "l"(gi + base + x)
                         : "memory");
          } else {   // past the shared copy: the contiguous overflow scratch
            ovv[x] = __ldcg(gv + base + x);
            ovi[x] = __ldcg(gi + base + x);
          }
        }
        p = max(p, upto);
      }
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  }
  __syncthreads();
  stamp(1);
  // ---- exact threshold: three radix levels over the global histograms
  uint32_t T = 0;
  long long need_eq = 0;
  uint32_t nbar = 0;
  if (state == kWOk) {
    uint32_t prefix = 0, pmask = 0;
    long long rank = budget;
    // Level 1 together with a guessed level 2: the previous run's top digit
    // d0 (the threshold moves little between iterations).  If level 1 finds
    // d0 again, the level-2 histogram of the d0 entries is already complete
    // and one level (a sweep and a task barrier) is skipped.
    const uint32_t prevT = t.scr->prefix;
    const bool guess = t.scr->all == 0 && prevT != 0;
    const uint32_t d0 = prevT >> 20;
    __shared__ uint32_t hg[kWBins];
    for (int b = tid; b < kWBins; b += kCoopThreads) {
      h[b] = 0;
      hg[b] = 0;
    }
    __syncthreads();
    for (int q0 = tid; q0 < n; q0 += 4 * kCoopThreads) {
      float v4[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int q = q0 + u * kCoopThreads;
        v4[u] = q < n ? getv(q) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (q0 + u * kCoopThreads < n) {
          const uint32_t key = mag_key(v4[u]);
          atomicAdd(&h[key >> 20], 1u);
          if (guess && (key >> 20) == d0) atomicAdd(&hg[(key >> 9) & (kWBins - 1)], 1u);
        }
    }
    __syncthreads();
    for (int b = tid; b < kWBins; b += kCoopThreads) {
      if (h[b]) atomicAdd(ws->hist + b, h[b]);
      if (hg[b]) atomicAdd(cs + kCoopH2g + b, hg[b]);
    }
    coop_barrier(bar, (uint32_t)G * ++nbar);
    stamp(2);
    int lvl0 = 1;
    {
      long long above = 0;
      const int d = coop_digit(ws->hist, kWBins, rank, &above, scratch);
      prefix = (uint32_t)d << 20;
      pmask = (uint32_t)(kWBins - 1) << 20;
      rank -= above;
      if (guess && (uint32_t)d == d0) {   // the guessed level-2 histogram holds the rank
        const int d2 = coop_digit(cs + kCoopH2g, kWBins, rank, &above, scratch);
        prefix |= (uint32_t)d2 << 9;
        pmask |= (uint32_t)(kWBins - 1) << 9;
        rank -= above;
        lvl0 = 2;
      }
    }
    for (int lvl = lvl0; lvl < 3; ++lvl) {
      const int shift = lvl == 0 ? 20 : (lvl == 1 ? 9 : 0);
      const int nb = lvl == 2 ? 512 : kWBins;
      uint32_t* gh = lvl == 0 ? ws->hist : cs + (lvl == 1 ? kCoopH2 : kCoopH3);
      for (int b = tid; b < nb; b += kCoopThreads) h[b] = 0;
      __syncthreads();
      for (int q0 = tid; q0 < n; q0 += 4 * kCoopThreads) {   // (4 loads in flight)
        float v4[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int q = q0 + u * kCoopThreads;
          v4[u] = q < n ? getv(q) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t key = mag_key(v4[u]);
          if (q0 + u * kCoopThreads < n && (key & pmask) == prefix)
            atomicAdd(&h[(key >> shift) & (nb - 1)], 1u);
        }
      }
      __syncthreads();
      for (int b = tid; b < nb; b += kCoopThreads)
        if (h[b]) atomicAdd(gh + b, h[b]);
      coop_barrier(bar, (uint32_t)G * ++nbar);
      stamp(2 + lvl);
      long long above = 0;
      const int d = coop_digit(gh, nb, rank, &above, scratch);
      prefix |= (uint32_t)d << shift;
      pmask |= (uint32_t)(nb - 1) << shift;
      rank -= above;
    }
    T = prefix;
    need_eq = rank;   // entries with key == T still to take (>= 1)
  }
  // ---- per-CTA counts -> offsets and tie quota
  int gt = 0, eq = 0;
  if (state == kWOk)
    for (int q0 = tid; q0 < n; q0 += 4 * kCoopThreads) {
      float v4[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int q = q0 + u * kCoopThreads;
        v4[u] = q < n ? getv(q) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t key = mag_key(v4[u]);
        const bool in = q0 + u * kCoopThreads < n;
        gt += in && key > T;
        eq += in && key == T;
      }
    }
  {
    int tt;
    block_exscan(gt, scratch, &tt);
    gt = tt;
    block_exscan(eq, scratch, &tt);
    eq = tt;
  }
  long long base_gt = 0, base_eq = 0;
  if (state == kWOk) {
    if (tid == 0) {
      cs[kCoopGt + c] = (uint32_t)gt;
      cs[kCoopEq + c] = (uint32_t)eq;
    }
    coop_barrier(bar, (uint32_t)G * ++nbar);
    stamp(5);
    long long a = 0, b = 0;
    for (int q = tid; q < c; q += kCoopThreads) {
      a += __ldcg(cs + kCoopGt + q);
      b += __ldcg(cs + kCoopEq + q);
    }
    __shared__ long long lsh3[3 * 32];
    long long z = 0;
    block_sum3_ll(a, b, z, lsh3);
    base_gt = a;
    base_eq = b;
  }
  // ---- write: selected (and pushed) / discarded, in index order
  const long long q_take = need_eq - base_eq;
  const int take = state != kWOk ? 0 : (int)(q_take <= 0 ? 0 : (q_take >= eq ? eq : q_take));
  const long long sel_before =
      state == kWAll ? e0 : (state == kWOk ? base_gt + (base_eq < need_eq ? base_eq : need_eq) : 0);
  // (kWAll / kWNone: every CTA sweeps its flat range straight from memory)
  const int nn = state == kWOk ? n : e1 - e0;
  int ks = (int)sel_before;
  int kd = e0 - (int)sel_before;
  int eqs = 0;   // ties of this CTA seen
  int cutv = -1;
  const uint32_t lt = lanemask_lt();
  const int npush = t.npush;
  const size_t push_voff = 16 + 4 * (size_t)t.push_cap;
  const float w = t.weight;
  for (int r0 = 0; r0 < nn; r0 += kCoopThreads * 4) {
    float v[4];
    int32_t ix[4];
    bool val[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int q = r0 + warp * 128 + u * 32 + lane;   // warp-major: index order
      val[u] = q < nn;
      v[u] = 0.f;
      ix[u] = 0;
      if (val[u]) {
        if (state == kWOk) {
          v[u] = getv(q);
          ix[u] = geti(q);
        } else {
          const int p = e0 + q;
          int lo = 0, hi = nseg - 1;
          while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (pre[mid] <= p) lo = mid;
            else hi = mid - 1;
          }
          const int src = soff[lo] + (p - pre[lo]);
          v[u] = __ldcg(ws->val + src);
          ix[u] = __ldcg(ws->idx + src);
        }
      }
    }
    // ties in order: warp tie counts -> CTA prefix
    int we = 0;
    uint32_t beq[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      beq[u] = __ballot_sync(0xffffffffu, state == kWOk && val[u] && mag_key(v[u]) == T);
      we += __popc(beq[u]);
    }
    if (lane == 0) wcnt[0][warp] = we;
    __syncthreads();
    int eb = eqs, etot = 0;
    for (int u = 0; u < kCoopWarps; ++u) {
      const int x = wcnt[0][u];
      if (u < warp) eb += x;
      etot += x;
    }
    bool sel[4];
    int ws_ = 0, wd = 0;
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t key = mag_key(v[u]);
      const bool is_eq = (beq[u] >> lane) & 1u;
      const int er = eb + __popc(beq[u] & lt);
      eb += __popc(beq[u]);
      sel[u] = val[u] && (state == kWAll || (state == kWOk && (key > T || (is_eq && er < take))));
      if (sel[u] && is_eq) cutv = max(cutv, ix[u]);
      ws_ += __popc(__ballot_sync(0xffffffffu, sel[u]));
      wd += __popc(__ballot_sync(0xffffffffu, val[u] && !sel[u]));
    }
    if (lane == 0) {
      wcnt[1][warp] = ws_;
      wcnt[2][warp] = wd;
    }
    __syncthreads();
    int bs = ks, bd = kd, ts = 0, td = 0;
    for (int u = 0; u < kCoopWarps; ++u) {
      const int a0 = wcnt[1][u], a1 = wcnt[2][u];
      if (u < warp) {
        bs += a0;
        bd += a1;
      }
      ts += a0;
      td += a1;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t bk = __ballot_sync(0xffffffffu, sel[u]);
      const uint32_t bdd = __ballot_sync(0xffffffffu, val[u] && !sel[u]);
      if (sel[u]) {
        const int p = bs + __popc(bk & lt);
        SPARDL_BOUND_CAP(p, t.sel_cap);
        if (state == kWOk) {   // compacted in place (positions <= this round's), copied out below
          const int lp = p - (int)sel_before;
          if (lp < cap) {
            si[lp] = ix[u];
            sv[lp] = v[u];
          } else {
            ovi[e0 + lp] = ix[u];
            ovv[e0 + lp] = v[u];
          }
        } else {
          t.sel_idx[p] = ix[u];
          t.sel_val[p] = v[u];
          if (npush > 0) SPARDL_BOUND_CAP(p, t.push_cap);
          for (int pp = 0; pp < npush; ++pp) {
            unsigned char* b = t.push_base[pp];
            reinterpret_cast<int32_t*>(b + 16)[p] = ix[u];
            reinterpret_cast<float*>(b + push_voff)[p] = v[u];
          }
        }
      } else if (val[u] && t.dis_idx) {
        const int p = bd + __popc(bdd & lt);
        SPARDL_BOUND_CAP(p, t.dis_cap);
        t.dis_idx[p] = ix[u];
        t.dis_val[p] = __fmul_rn(v[u], w);
      }
      bs += __popc(bk);
      bd += __popc(bdd);
    }
    ks += ts;
    kd += td;
    eqs += etot;
    __syncthreads();   // wcnt reused
  }
  // the CTA's selected entries (contiguous in the output from sel_before) to the
  // block and every peer's copy: 16-byte stores from the compacted shared copy
  // (a remote store per 4-byte entry and lane wasted most of the NVLink packet)
  if (state == kWOk) {
    __syncthreads();
    const int ns = ks - (int)sel_before;
    const int g0 = (int)sel_before;
    const int head = min(ns, (4 - (g0 & 3)) & 3);
    const int nbody = (ns - head) >> 2;
    for (int d = 0; d <= npush; ++d) {
      int32_t* di = d == 0 ? t.sel_idx : reinterpret_cast<int32_t*>(t.push_base[d - 1] + 16);
      float* dv = d == 0 ? t.sel_val : reinterpret_cast<float*>(t.push_base[d - 1] + push_voff);
      if (ns > 0) SPARDL_BOUND_CAP(g0 + ns - 1, d == 0 ? t.sel_cap : t.push_cap);
      const bool vec = ((reinterpret_cast<uintptr_t>(di) | reinterpret_cast<uintptr_t>(dv)) & 15) == 0;
      if (!vec) {   // (unaligned destination: plain stores)
        for (int l = tid; l < ns; l += kCoopThreads) {
          di[g0 + l] = geti(l);
          dv[g0 + l] = getv(l);
        }
        continue;
      }
      if (tid < head) {
        di[g0 + tid] = geti(tid);
        dv[g0 + tid] = getv(tid);
      }
      for (int j = tid; j < nbody; j += kCoopThreads) {
        const int l = head + 4 * j;
        reinterpret_cast<int4*>(di + g0 + l)[0] =
            make_int4(geti(l), geti(l + 1), geti(l + 2), geti(l + 3));
        reinterpret_cast<float4*>(dv + g0 + l)[0] =
            make_float4(getv(l), getv(l + 1), getv(l + 2), getv(l + 3));
      }
      for (int l = head + 4 * nbody + tid; l < ns; l += kCoopThreads) {
        di[g0 + l] = geti(l);
        dv[g0 + l] = getv(l);
      }
    }
  }
  stamp(6);
  // the CTA holding the last tie taken knows the cut index (ties in index order)
  cutv = __reduce_max_sync(0xffffffffu, cutv);
  __shared__ int s_cut;
  if (tid == 0) s_cut = -1;
  __syncthreads();
  if (lane == 0 && cutv >= 0) atomicMax(&s_cut, cutv);
  __syncthreads();
  if (tid == 0 && state == kWOk && base_eq < need_eq && need_eq <= base_eq + eq) ws->cut = s_cut;
  // ---- completion: the last CTA records, counts, cleans up and publishes
  __syncthreads();
  if (tid == 0) {
    if (npush > 0) __threadfence_system();
    else __threadfence();
    s_flag = (int)(atomicAdd(&ws->wdone, 1u) == (unsigned)G - 1);
  }
  __syncthreads();
  if (!s_flag) return;
  __threadfence();
  if (SPARDL_STAMPS && tid == 0) {   // the last CTA's completion
    long long ts;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(ts));
    t.scr->tstamp[7] = ts;
  }
  if (state == kWOk) {   // leave the histograms zeroed for the next run
    for (int b = tid; b < kWBins; b += kCoopThreads) {
      ws->hist[b] = 0;
      cs[kCoopH2 + b] = 0;
      cs[kCoopH2g + b] = 0;
    }
    for (int b = tid; b < 512; b += kCoopThreads) cs[kCoopH3 + b] = 0;
  }
  if (tid != 0) return;
  const long long ns = state == kWAll ? total : (state == kWOk ? budget : 0);
  const int32_t cut = state == kWOk ? __ldcg(&ws->cut) : -1;
  *bar = 0;
  ws->wdone = 0;
  ws->state = state;
  ws->T = T;
  ws->total = total;
  ws->total_sel = ns;
  SelScratch* sc = t.scr;
  const int all = state == kWAll ? 1 : (state == kWNone ? 2 : 0);
  sc->mode = 0;
  sc->total = total;
  sc->prefix = state == kWOk ? T : 0;
  sc->cut_idx = cut;
  sc->all = all;
  if (ws->is_div) {
    if (all == 1) {
      sc->all = 0;
      sc->prefix = *t.pre_key_dev;
      sc->cut_idx = INT_MAX;
    }
    if (t.div_hist)
      update_history(t.div_hist, 0, all, state == kWOk ? T : 0u, *t.pre_key_dev, total, budget);
  }
  *t.sel_cnt = (int32_t)ns;
  for (int p = 0; p < npush; ++p) *reinterpret_cast<int32_t*>(t.push_base[p]) = (int32_t)ns;
  if (t.dis_cnt) *t.dis_cnt = (int32_t)(total - ns);
  if (t.total_out) *t.total_out = total;
  peer_publish(t.ps);   // (fences at system scope first)
}

}  // namespace

int wsel_coop_words() { return kCoopWords; }
int wsel_coop_max_seg() { return kCoopMaxSeg; }

// CTAs of the cooperative select resident at once on this device, and the
// entries one CTA can hold
static int coop_table_bytes(int tabn) { return (2 * tabn + 4) * 4; }

static void coop_geometry(int* resident, int* cap, int tabn = kCoopMaxSeg) {
  static int res[kMaxDevices] = {}, cp[kMaxDevices] = {};
  const int dev = cur_device();
  if (!res[dev]) {
    int optin = 0, sms = 0;
    cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    cudaFuncAttributes fa{};
    cudaFuncGetAttributes(&fa, k_wsel_coop);
    const int dyn = optin - (int)fa.sharedSizeBytes - 1024;
    cudaFuncSetAttribute(k_wsel_coop, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn);
    cp[dev] = dyn;   // (dynamic shared memory; the entries follow from the table size)

    int per = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_wsel_coop, kCoopThreads, dyn);
    res[dev] = std::max(1, sms * std::max(1, per));
  }
  *resident = res[dev];
  *cap = std::max(0, (cp[dev] - coop_table_bytes(tabn)) / 8) & ~31;
  // tests: a smaller shared copy per CTA, so that the overflow scratch runs
  if (const char* e = getenv("SPARDL_WSEL_COOP_CAP")) *cap = std::max(32, std::min(*cap, atoi(e)));
}

long long wsel_coop_capacity(int ntask, int max_nseg) {
  int resident = 0, cap = 0;
  coop_geometry(&resident, &cap, std::max(1, max_nseg));
  const int G = std::max(1, std::min(kCoopMaxG, resident / std::max(1, ntask)));
  return (long long)G * cap;
}

int launch_wselect_coop(const SelTask* tasks_dev, int ntask, int max_nseg, cudaStream_t s) {
  if (ntask <= 0) return 0;
  const int tabn = std::max(1, std::min(max_nseg, kCoopMaxSeg));
  int resident = 0, cap = 0;
  coop_geometry(&resident, &cap, tabn);
  const int G = std::max(1, std::min(kCoopMaxG, resident / ntask));
  const size_t smem = (size_t)coop_table_bytes(tabn) + (size_t)cap * 8;
  launch_pdl(k_wsel_coop, dim3(G, ntask), dim3(kCoopThreads), smem, s, tasks_dev, cap, tabn);
  return 1;
}

int launch_wselect(const SelTask* tasks_dev, int ntask, int max_tiles, bool histogram,
                   cudaStream_t s) {
  if (ntask <= 0 || max_tiles <= 0) return 0;
  int n = 0;
  if (histogram) {   // (the dividing selects' histogram comes from k_div_cand)
    launch_pdl(k_wsel_hist, dim3(max_tiles, ntask), dim3(kWThreads), 0, s, tasks_dev);
    ++n;
  }
  launch_pdl(k_wsel_gather, dim3(max_tiles, ntask), dim3(kWThreads), 0, s, tasks_dev);
  launch_pdl(k_wsel_write, dim3(max_tiles, ntask), dim3(kWThreads), 0, s, tasks_dev);
  return n + 2;
}

int wsel_max_group() { return kWMaxGroup; }

}  // namespace sdl
