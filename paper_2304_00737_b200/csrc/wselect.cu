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
#include <climits>
#include <cstdio>

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

}  // namespace

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
