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
//   k_wsel_hist    level-1 histogram of the magnitude keys, 2048 bins of
//                  key >> 20 (the dividing select's window histogram above
//                  its pre-threshold is filled by k_div_cand instead)
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

#include "common.cuh"
#include "kernels.cuh"

namespace sdl {

namespace {

constexpr int kWThreads = 256;
constexpr int kWWarps = kWThreads / 32;
constexpr int kWHistTiles = 16;    // tiles per histogram CTA
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

// level-1 bin of a key: 0..kWBins-1, kWBins = above the window, -1 = below
__device__ __forceinline__ int w_bin(int mode, uint32_t base, uint32_t shift, uint32_t key) {
  if (mode == kWFull) return (int)(key >> 20);
  if (key < base) return -1;
  const uint32_t d = (key - base) >> shift;
  return d >= (uint32_t)kWBins ? kWBins : (int)d;
}

__device__ __forceinline__ unsigned long long w_comp(uint32_t key, int32_t idx) {
  return ((unsigned long long)key << 32) | (unsigned long long)(0x7fffffffu - (uint32_t)idx);
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kWThreads) k_wsel_hist(const SelTask* __restrict__ tasks) {
  pdl_enter();
  const SelTask& t = tasks[blockIdx.y];
  WScratch* __restrict__ ws = t.ws;
  if (ws->mode != kWFull) return;
  peer_wait(t.ps);
  const int nseg = w_nseg(*ws);
  const int G = ws->group;
  const int s0 = blockIdx.x * kWHistTiles * G;
  if (s0 >= nseg) return;
  const int s1 = min(nseg, s0 + kWHistTiles * G);
  __shared__ uint32_t h[kWBins];
  for (int b = threadIdx.x; b < kWBins; b += kWThreads) h[b] = 0;
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  for (int s = s0 + warp; s < s1; s += kWWarps) {
    int off, cnt;
    w_seg(*ws, s, off, cnt);
    const float* vp = ws->val + off;
    for (int j0 = 0; j0 < cnt; j0 += 128) {
      float v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int j = j0 + u * 32 + lane;
        v[u] = j < cnt ? __ldcg(vp + j) : 0.f;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (j0 + u * 32 + lane < cnt) atomicAdd(&h[mag_key(v[u]) >> 20], 1u);
    }
  }
  __syncthreads();
  for (int b = threadIdx.x; b < kWBins; b += kWThreads)
    if (h[b]) atomicAdd(&ws->hist[b], h[b]);
}

// The bin holding the need-th largest key of the level-1 histogram (every
// thread of the CTA gets the result).  Returns false if the histogram (plus
// `above`) holds fewer than `need` entries.  *before = entries in higher bins
// (including `above`).
__device__ bool w_locate(const uint32_t* __restrict__ hist, long long above, long long need,
                         int* bin, long long* before, int* scratch, long long* sh) {
  constexpr int BPT = kWBins / kWThreads;   // 8 bins per thread
  __shared__ int s_bin;
  __shared__ long long s_before;
  const int tid = threadIdx.x;
  const int g = kWThreads - 1 - tid;        // this thread's bin group, top groups first
  uint32_t hb[BPT];
  long long mine = 0;
#pragma unroll
  for (int q = 0; q < BPT; ++q) {
    hb[q] = __ldcg(hist + g * BPT + q);
    mine += hb[q];
  }
  if (tid == 0) {
    s_bin = -1;
    s_before = 0;
  }
  // exclusive scan over descending groups (counts fit in int: < 2^31 entries)
  int tot = 0;
  const long long ex = above + block_exscan((int)mine, scratch, &tot);
  if (ex < need && need <= ex + mine) {
    long long cum = ex;
    for (int q = BPT - 1; q >= 0; --q) {
      if (cum + (long long)hb[q] >= need) {
        s_bin = g * BPT + q;
        s_before = cum;
        break;
      }
      cum += hb[q];
    }
  }
  __syncthreads();
  *bin = s_bin;
  *before = s_before;
  (void)sh;
  return s_bin >= 0;
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
__global__ void __launch_bounds__(kWThreads) k_wsel_gather(const SelTask* __restrict__ tasks) {
  pdl_enter();
  const SelTask& t = tasks[blockIdx.y];
  WScratch* __restrict__ ws = t.ws;
  peer_wait(t.ps);
  __shared__ int scratch[40];
  __shared__ long long lsh[32];
  __shared__ int s_state;
  __shared__ unsigned int s_n, s_na;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int mode = ws->mode;
  const uint32_t base = ws->base, shift = ws->shift;
  const int64_t budget = t.budget_dev ? *t.budget_dev : t.budget;
  const long long above = mode == kWWindow ? (long long)__ldcg(&ws->above) : 0;
  // ---- the run state and the boundary bin (identical in every CTA)
  long long total;
  bool bad = false;
  if (ws->is_div) {
    total = *t.cand_total;
    bad = *t.cand_bad != 0 || total < budget;   // incomplete: dense fallback in k_select
  }
  int bstar = -1;
  long long before = 0;
  {
    long long part = 0;
    for (int b = tid; b < kWBins; b += kWThreads) part += __ldcg(ws->hist + b);
    long long u0 = 0, u1 = 0;
    block_sum3_ll(part, u0, u1, lsh);
    if (!ws->is_div) total = part;
  }
  int state;
  if (bad) state = kWFallback;
  else if (total <= budget) state = kWAll;
  else if (budget <= 0) state = kWNone;
  else if (above >= budget) state = kWFallback;   // threshold above the window
  else state = w_locate(ws->hist, above, budget, &bstar, &before, scratch, lsh) ? kWOk : kWFallback;
  // ---- this tile
  const int nseg = w_nseg(*ws);
  const int G = ws->group;
  const int ntiles = (nseg + G - 1) / G;
  const int q = blockIdx.x;
  if (tid == 0) {
    s_n = 0;
    s_na = 0;
  }
  __syncthreads();
  if (q < ntiles && state != kWFallback) {
    const int s0 = q * G, s1 = min(nseg, s0 + G);
    unsigned int n = 0, na = 0;
    for (int s = s0 + warp; s < s1; s += kWWarps) {
      int off, cnt;
      w_seg(*ws, s, off, cnt);
      n += cnt;
      if (state != kWOk) continue;
      const float* vp = ws->val + off;
      const int32_t* ip = ws->idx + off;
      for (int j0 = 0; j0 < cnt; j0 += 128) {
        float v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = j0 + u * 32 + lane;
          v[u] = j < cnt ? __ldcg(vp + j) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = j0 + u * 32 + lane;
          const uint32_t key = mag_key(v[u]);
          const int b = j < cnt ? w_bin(mode, base, shift, key) : -1;
          na += b > bstar;
          const bool in = b == bstar;
          const uint32_t bal = __ballot_sync(0xffffffffu, in);
          if (bal) {
            int p0 = 0;
            if (lane == 0) p0 = (int)atomicAdd(&ws->bin_n, (unsigned)__popc(bal));
            p0 = __shfl_sync(0xffffffffu, p0, 0);
            if (in) {
              const int p = p0 + __popc(bal & lanemask_lt());
              if (p < ws->bin_cap) {
                ws->bin_c[p] = w_comp(key, __ldcg(ip + j));
                ws->bin_tile[p] = q;
              }
            }
          }
        }
      }
    }
    n = __reduce_add_sync(0xffffffffu, lane == 0 ? n : 0u);   // (segment counts: lane-uniform)
    na = __reduce_add_sync(0xffffffffu, na);
    if (lane == 0) {
      atomicAdd(&s_n, n);
      atomicAdd(&s_na, na);
    }
    __syncthreads();
    if (tid == 0) {
      ws->tile_n[q] = (int)s_n;
      ws->tile_sel[q] = state == kWOk ? (int)s_na : (state == kWAll ? (int)s_n : 0);
    }
  }
  // ---- arrival; the last CTA of the task finishes the selection
  __threadfence();
  __syncthreads();
  if (tid == 0) s_state = (int)(atomicAdd(&ws->arrive, 1u) == gridDim.x - 1);
  __syncthreads();
  if (!s_state) return;
  __threadfence();
  SelScratch* sc = t.scr;
  if (state == kWOk) {
    const long long nb = (long long)__ldcg(&ws->bin_n);
    if (nb > ws->bin_cap || nb != (long long)__ldcg(ws->hist + bstar))
      state = kWFallback;   // bin buffer overflow (massive key ties): k_select
  }
  unsigned long long cstar = 0;
  if (state == kWOk) {
    const int nb = (int)__ldcg(&ws->bin_n);
    cstar = w_select_kth(ws->bin_c, nb, budget - before, scratch);
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
  // ---- the selection record, the dividing history; zero the histogram
  for (int b = tid; b < kWBins; b += kWThreads) ws->hist[b] = 0;
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
    ws->above = 0;
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
          update_history(t.div_hist, 0, all, state == kWOk ? T : 0u, *t.pre_key_dev, total,
                         budget);
      }
    }
  }
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kWThreads) k_wsel_write(const SelTask* __restrict__ tasks) {
  pdl_enter();
  const SelTask& t = tasks[blockIdx.y];
  const WScratch* __restrict__ ws = t.ws;
  const int state = ws->state;
  if (state == kWFallback) return;   // k_select selects this task
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q = blockIdx.x;
  const int ntiles = ws->ntiles;
  const int npush = t.npush;
  __shared__ int segsel[kWMaxGroup], segbase[kWMaxGroup + 1];
  __shared__ int s_last;
  if (q < ntiles) {
    peer_wait(t.ps);
    const uint32_t T = ws->T;
    const int32_t cut = ws->cut;
    auto keep = [&](uint32_t key, int32_t ix) {
      return state == kWAll || (state == kWOk && (key > T || (key == T && ix <= cut)));
    };
    const int nseg = w_nseg(*ws);
    const int G = ws->group;
    const int s0 = q * G, s1 = min(nseg, s0 + G);
    const int nl = s1 - s0;
    // pass A: kept entries per segment
    for (int ls = warp; ls < nl; ls += kWWarps) {
      int off, cnt;
      w_seg(*ws, s0 + ls, off, cnt);
      const float* vp = ws->val + off;
      const int32_t* ip = ws->idx + off;
      int k = 0;
      for (int j0 = 0; j0 < cnt; j0 += 128) {
        float v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = j0 + u * 32 + lane;
          v[u] = j < cnt ? __ldcg(vp + j) : 0.f;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int j = j0 + u * 32 + lane;
          const uint32_t key = mag_key(v[u]);
          bool kp = false;
          if (j < cnt) kp = key == T && state == kWOk ? keep(key, __ldcg(ip + j)) : keep(key, 0);
          k += __popc(__ballot_sync(0xffffffffu, kp));
        }
      }
      if (lane == 0) segsel[ls] = k;
    }
    __syncthreads();
    if (tid == 0) {
      int a = 0;
      for (int ls = 0; ls < nl; ++ls) {
        segbase[ls] = a;
        a += segsel[ls];
      }
      segbase[nl] = a;
    }
    __syncthreads();
    // pass B: ordered writes (segment bases, then warp-ballot ranks)
    int32_t* pidx[kMaxPush];
    float* pval[kMaxPush];
#pragma unroll
    for (int p = 0; p < kMaxPush; ++p) {
      pidx[p] = nullptr;
      pval[p] = nullptr;
      if (p < npush) {
        unsigned char* b = t.push_base[p];
        pidx[p] = reinterpret_cast<int32_t*>(b + 16);
        pval[p] = reinterpret_cast<float*>(b + 16 + 4 * (size_t)t.push_cap);
      }
    }
    const int sel0 = ws->tile_sel_off[q];
    const int dis0 = ws->tile_dis_off[q];
    const bool want_dis = t.dis_idx != nullptr;
    const float w = t.weight;
    const uint32_t lt = lanemask_lt();
    int seg_entry0 = 0;   // entries of the tile before segment ls (for discard ranks)
    for (int ls = 0; ls < nl; ++ls) {
      int off, cnt;
      w_seg(*ws, s0 + ls, off, cnt);
      if (ls % kWWarps == warp) {
        const float* vp = ws->val + off;
        const int32_t* ip = ws->idx + off;
        int ks = sel0 + segbase[ls];
        int kd = dis0 + (seg_entry0 - segbase[ls]);
        for (int j0 = 0; j0 < cnt; j0 += 128) {
          float v[4];
          int32_t ix[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int j = j0 + u * 32 + lane;
            v[u] = j < cnt ? __ldcg(vp + j) : 0.f;
            ix[u] = j < cnt ? __ldcg(ip + j) : 0;
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int j = j0 + u * 32 + lane;
            const bool valid = j < cnt;
            const bool kp = valid && keep(mag_key(v[u]), ix[u]);
            const uint32_t bk = __ballot_sync(0xffffffffu, kp);
            const uint32_t bd = __ballot_sync(0xffffffffu, valid && !kp);
            if (kp) {
              const int p = ks + __popc(bk & lt);
              t.sel_idx[p] = ix[u];
              t.sel_val[p] = v[u];
#pragma unroll
              for (int pp = 0; pp < kMaxPush; ++pp)
                if (pp < npush) {
                  pidx[pp][p] = ix[u];
                  pval[pp][p] = v[u];
                }
            } else if (valid && want_dis) {
              const int p = kd + __popc(bd & lt);
              t.dis_idx[p] = ix[u];
              t.dis_val[p] = __fmul_rn(v[u], w);
            }
            ks += __popc(bk);
            kd += __popc(bd);
          }
        }
      }
      seg_entry0 += cnt;
    }
  }
  // ---- completion: the last CTA of the task writes the counts and publishes
  if (npush > 0) __threadfence_system();
  else __threadfence();
  __syncthreads();
  if (tid == 0) s_last = (int)(atomicAdd(const_cast<uint32_t*>(&ws->wdone), 1u) == gridDim.x - 1);
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
  if (histogram) {
    launch_pdl(k_wsel_hist, dim3((max_tiles + kWHistTiles - 1) / kWHistTiles, ntask),
               dim3(kWThreads), 0, s, tasks_dev);
    ++n;
  }
  launch_pdl(k_wsel_gather, dim3(max_tiles, ntask), dim3(kWThreads), 0, s, tasks_dev);
  launch_pdl(k_wsel_write, dim3(max_tiles, ntask), dim3(kWThreads), 0, s, tasks_dev);
  return n + 2;
}

int wsel_max_group() { return kWMaxGroup; }

}  // namespace sdl
