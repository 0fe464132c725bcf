// The dividing pass: residual add fused with candidate compaction.
//
// Semantics (inc/pipeline.hpp:162-184, inc/residual.hpp:63-92):
//   combined = g + carry            (ResidualStore::apply; this is also G_copy)
//   per block b: top-L of the dense slice combined[lo_b, hi_b) (zeros count)
// Layout: the residual buffer IS G_copy -- `carry` is overwritten in place by
// g + carry, so the pass moves exactly 12 bytes per element (read g, read
// carry, write carry) plus the small candidate stream.
//
// Kernels:
//   k_div_sample   one chunk in `sample_every`: histogram of the top 11 key bits
//                  of g + carry (read only)
//   k_div_prethr   per block: the pre-threshold -- the lower edge of the digit
//                  holding the sample's ~1.25 L-th largest key
//   k_div_cand     every chunk: combined = g + carry written back with 128-bit
//                  stores; entries with key >= pre-threshold compacted, in
//                  index order, into the chunk's candidate segment
// The select that follows (select.cu) checks on the device that the
// candidates are complete (>= L of them, no chunk overflow); otherwise it
// selects from the dense slice instead, so the result never depends on the
// sample.
#include <algorithm>
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"
#include "wsel_common.cuh"

#ifndef SPARDL_DIV_MINB
#define SPARDL_DIV_MINB 3
#endif

namespace sdl {

namespace {

// chunk c of a task covers [max(lo, A + c*kChunk), min(hi, A + (c+1)*kChunk))
// with A = lo rounded down to a multiple of 4, so every chunk is made of
// whole float4 groups of the global array.
__device__ __forceinline__ int64_t chunk_origin(const DivTask& t) { return (int64_t)(t.lo & ~3); }

__global__ void __launch_bounds__(kThreads) k_div_sample(const DivTask* __restrict__ tasks,
                                                         int apply_residual) {
  pdl_enter();
  const DivTask& t = tasks[blockIdx.y];
  if (!t.use_cand || t.hist->valid) return;   // no sample needed: carried threshold
  const int c = blockIdx.x * t.sample_every;
  if (c >= t.nchunks) return;
  // 13-bit key histogram (8 exponent + 5 mantissa bits: 1/32-octave bins)
  extern __shared__ uint32_t h[];
  __shared__ unsigned int bmin, bmax;
  for (int b = threadIdx.x; b < kSampBins; b += blockDim.x) h[b] = 0;
  if (threadIdx.x == 0) {
    bmin = kSampBins;
    bmax = 0;
  }
  __syncthreads();
  const int64_t A = chunk_origin(t) + (int64_t)c * kChunk;
  const int64_t s = A > t.lo ? A : t.lo;
  const int64_t e = (A + kChunk) < t.hi ? (A + kChunk) : t.hi;
  const float* g = apply_residual ? t.g_tab[t.g_id] : nullptr;
  constexpr int PER = kChunk / kThreads;   // elements per thread, all loads issued first
  float vals[PER];
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int64_t i = s + (int64_t)q * kThreads + threadIdx.x;
    vals[q] = 0.f;
    if (i < e) vals[q] = apply_residual ? __fadd_rn(__ldcs(g + i), __ldcs(t.carry + i)) : t.carry[i];
  }
  // 1/32-octave bins spread a warp's keys over many bins: plain shared
  // atomics; the occupied bin range is tracked in registers
  unsigned lo_b = kSampBins, hi_b = 0;
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int64_t i = s + (int64_t)q * kThreads + threadIdx.x;
    if (i < e) {
      const uint32_t bin = mag_key(vals[q]) >> kSampShift;
      atomicAdd(&h[bin], 1u);
      lo_b = min(lo_b, bin);
      hi_b = max(hi_b, bin);
    }
  }
  lo_b = __reduce_min_sync(0xffffffffu, lo_b);
  hi_b = __reduce_max_sync(0xffffffffu, hi_b);
  if ((threadIdx.x & 31) == 0) {
    atomicMin(&bmin, lo_b);
    atomicMax(&bmax, hi_b);
  }
  __syncthreads();
  for (int b = bmin + threadIdx.x; b <= (int)bmax; b += blockDim.x)
    if (h[b]) atomicAdd(&t.samp_hist[b], h[b]);
}

__global__ void __launch_bounds__(kThreads) k_div_prethr(const DivTask* __restrict__ tasks) {
  pdl_enter();
  const DivTask& t = tasks[blockIdx.x];
  constexpr int BPT = kSampBins / kThreads;
  __shared__ long long suf[kThreads];
  __shared__ long long lscr[32];
  // the wide select's histogram window (wselect.cu): 2048 bins from the
  // pre-threshold up, together ~4x the expected distance to the threshold
  auto set_window = [&](uint32_t pre, uint32_t w) {
    if (t.ws) {
      uint32_t s = 0;
      while (s < 31 && ((unsigned long long)kWBins << s) < 4ull * w) ++s;
      t.ws->base = pre;
      t.ws->shift = s;
    }
  };
  if (t.use_cand && t.hist->valid) {   // threshold carried from the last iteration
    if (threadIdx.x == 0) {           // (before touching the histogram: the common case)
      *t.cand_total = 0;
      *t.cand_bad = 0;
      *t.pre_key = t.hist->next_pre;
      set_window(t.hist->next_pre, t.hist->delta);
    }
    return;   // the sample histogram was not touched: still zero
  }
  uint32_t* hist = t.samp_hist + threadIdx.x * BPT;
  long long mine = 0;
  for (int q = 0; q < BPT; ++q) mine += hist[q];
  const long long ns = block_sum_ll(mine, lscr);
  const int64_t nb = (int64_t)t.hi - t.lo;
  if (threadIdx.x == 0) {
    *t.cand_total = 0;
    *t.cand_bad = t.use_cand ? 0 : 1;
    *t.pre_key = 0;
  }
  // target rank inside the sample: 1.25 L scaled to the sample, plus 4 sigma
  const double frac = (double)t.budget / (double)nb;
  const double expect = frac * (double)ns;
  const long long target = (long long)(1.25 * expect + 4.0 * sqrt(expect + 1.0) + 8.0);
  if (!t.use_cand || ns == 0 || target >= ns) {
    if (threadIdx.x == 0) *t.cand_bad = 1;
    for (int q = 0; q < BPT; ++q) hist[q] = 0;   // leave the histogram zeroed
    return;
  }
  // reverse inclusive scan (Hillis-Steele over descending thread order)
  const int r = blockDim.x - 1 - threadIdx.x;
  __shared__ long long vals[kThreads];
  vals[r] = mine;
  __syncthreads();
  suf[threadIdx.x] = vals[threadIdx.x];
  __syncthreads();
  for (int o = 1; o < (int)blockDim.x; o <<= 1) {
    const long long add = threadIdx.x >= (unsigned)o ? suf[threadIdx.x - o] : 0;
    __syncthreads();
    suf[threadIdx.x] += add;
    __syncthreads();
  }
  const long long above = r > 0 ? suf[r - 1] : 0;
  if (above < target && target <= above + mine) {
    long long cum = above;
    for (int q = BPT - 1; q >= 0; --q) {
      const uint32_t cq = hist[q];
      if (cum + (long long)cq >= target) {
        *t.pre_key = (uint32_t)(threadIdx.x * BPT + q) << kSampShift;
        set_window((uint32_t)(threadIdx.x * BPT + q) << kSampShift, 8u << kSampShift);
        break;
      }
      cum += cq;
    }
  }
  for (int q = 0; q < BPT; ++q) hist[q] = 0;   // leave the histogram zeroed
}

// The chunk's candidates (bit (it * 4 + e) of `mask`: element
// (warp * 32 * ITER + it * 32 + lane) * 4 + e of the chunk, value in s_comb)
// compacted in index order into the chunk's candidate segment.
__device__ __forceinline__ void cand_compact(const DivTask& t, int c, int64_t A, uint32_t mask,
                                             const float* s_comb, uint32_t* s_wh = nullptr,
                                             uint32_t* s_wab = nullptr, uint32_t hbase = 0,
                                             uint32_t hshift = 0) {
  constexpr int ITER = kChunk / (kThreads * 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // order: (warp, it, lane, e) == index order inside the chunk
  // per group: a lane's offset = candidates of the lower lanes, from four
  // ballots (one per float4 component)
  int lane_excl[ITER];
  int warp_total = 0;
  const uint32_t lt = lanemask_lt();
#pragma unroll
  for (int it = 0; it < ITER; ++it) {
    int below = 0, all = 0;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const uint32_t b = __ballot_sync(0xffffffffu, (mask >> (it * 4 + e)) & 1u);
      below += __popc(b & lt);
      all += __popc(b);
    }
    lane_excl[it] = warp_total + below;
    warp_total += all;
  }
  __shared__ int wtot[kThreads / 32 + 1];
  if (lane == 0) wtot[warp] = warp_total;
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0;
    for (int w = 0; w < kThreads / 32; ++w) {
      const int x = wtot[w];
      wtot[w] = s;
      s += x;
    }
    wtot[kThreads / 32] = s;
  }
  __syncthreads();
  const int total = wtot[kThreads / 32];
  if (total > t.cap) {   // chunk segment overflow: the select falls back to the dense slice
    if (threadIdx.x == 0) {
      atomicOr(t.cand_bad, 2);
      t.cand_cnt[c] = 0;
    }
    return;
  }
  const int wbase = wtot[warp];
  int32_t* ci = t.cand_idx + (size_t)c * t.cap;
  float* cv = t.cand_val + (size_t)c * t.cap;
#pragma unroll
  for (int it = 0; it < ITER; ++it) {
    int p = wbase + lane_excl[it];
    const int64_t i0 = A + ((int64_t)warp * (32 * ITER) + it * 32 + lane) * 4;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      if (mask & (1u << (it * 4 + e))) {
        const float x = s_comb[(warp * (32 * ITER) + it * 32 + lane) * 4 + e];
        ci[p] = (int32_t)(i0 + e);
        cv[p] = x;
        ++p;
        if (s_wh) {   // the wide select's window histogram (shared, flushed per CTA)
          const uint32_t d = (mag_key(x) - hbase) >> hshift;
          atomicAdd(d < (uint32_t)kWBins ? &s_wh[d] : s_wab, 1u);
        }
      }
    }
  }
  if (threadIdx.x == 0) t.cand_cnt[c] = total;
}

// The dividing select's level-1 histogram, filled by the candidate pass
// itself: every CTA flushes its shared histogram (once, non-empty bins only)
// and the CTA that completes the task decides the wide select's run
// (wsel_common.cuh).  Every CTA of the grid arrives, with or without work.
__device__ void div_wsel_epilogue(const DivTask& t, const uint32_t* s_wh, const uint32_t* s_wab,
                                  bool flush) {
  WScratch* ws = t.ws;
  __shared__ int s_last;
  __shared__ int scratch[40];
  __shared__ long long lsh[3 * 32];
  __syncthreads();
  if (flush) {
    for (int b = threadIdx.x; b < kWBins; b += kThreads)
      if (s_wh[b]) atomicAdd(&ws->hist[b], s_wh[b]);
    if (threadIdx.x == 0 && *s_wab) atomicAdd(&ws->above, *s_wab);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    s_last = (int)(atomicAdd(&ws->harrive, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const long long total = w_hist_total(ws, lsh) + __ldcg(&ws->above);
  const bool bad = (__ldcg(t.cand_bad) & 3) != 0 || total < t.budget;
  w_decide(ws, total, bad, t.budget, kWWindow, ws->base, ws->shift, scratch, lsh);
}

// ---------------------------------------------------------------------------
// Bulk-copy (TMA) form of the candidate pass.  One elected thread streams
// the chunk's carry and gradient into shared memory with cp.async.bulk
// (two 32 KB copies completing on one mbarrier: no registers hold the
// chunk, so every load of the SM is in flight at once); the deferred
// finalize records patch the staged carry; combined = g + carry is written
// back in place in shared memory and streamed out with one bulk store; the
// candidates are compacted from shared memory as in k_div_cand.  The
// unaligned edge elements of a block (lo, hi not multiples of 4) go through
// plain loads and stores.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int APPLY, int FIN>
__global__ void __launch_bounds__(kThreads, SPARDL_DIV_MINB) k_div_cand_bulk(const DivTask* __restrict__ tasks) {
  pdl_enter();
  const DivTask& t = tasks[blockIdx.y];
  const int c = blockIdx.x;
  __shared__ uint32_t s_wh[kWBins];
  __shared__ uint32_t s_wab;
  const bool wf = t.ws != nullptr && t.ws_fused;
  if (c >= t.nchunks) {
    if (wf) div_wsel_epilogue(t, s_wh, &s_wab, false);
    return;
  }
  uint32_t wb = 0, wsh = 0;
  if (wf) {
    for (int b = threadIdx.x; b < kWBins; b += kThreads) s_wh[b] = 0;
    if (threadIdx.x == 0) s_wab = 0;
    wb = t.ws->base;
    wsh = t.ws->shift;
  }
  extern __shared__ __align__(128) unsigned char dsm[];
  float* s_c = reinterpret_cast<float*>(dsm);        // carry -> combined
  float* s_g = s_c + kChunk;                          // gradient
  __shared__ __align__(8) unsigned long long bar;
  const bool cand = !(*t.cand_bad & 1);
  const uint32_t pre = *t.pre_key;
  const int64_t A = chunk_origin(t) + (int64_t)c * kChunk;
  const int64_t lo = t.lo, hi = t.hi;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int ITER = kChunk / (kThreads * 4);
  // the whole-float4 span of the chunk inside [lo, hi)
  const int64_t v0 = max(A, (lo + 3) & ~int64_t(3));
  const int64_t v1 = max(v0, min(A + kChunk, hi & ~int64_t(3)));
  const uint32_t bytes = (uint32_t)((v1 - v0) * 4);
  const float* __restrict__ g = APPLY ? t.g_tab[t.g_id] : nullptr;
  float* __restrict__ carry = t.carry;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    const uint32_t tx = bytes * (APPLY ? 2u : 1u);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)),
                 "r"(tx)
                 : "memory");
    if (bytes) {
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
              "r"(smem_u32(s_c + (v0 - A))),
          "l"(carry + v0), "r"(bytes), "r"(smem_u32(&bar))
          : "memory");
      if (APPLY)
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
                "r"(smem_u32(s_g + (v0 - A))),
            "l"(g + v0), "r"(bytes), "r"(smem_u32(&bar))
            : "memory");
    }
  }
  // the chunk's edge elements (outside the span, inside [lo, hi)) and zeros
  // outside the block
  for (int k = threadIdx.x; k < kChunk; k += kThreads) {
    const int64_t i = A + k;
    if (i >= v0 && i < v1) continue;
    const bool in = i >= lo && i < hi;
    s_c[k] = in ? carry[i] : 0.f;
    if (APPLY) s_g[k] = in ? g[i] : 0.f;
  }
  int r0 = 0, r1 = 0;
  int32_t d_all = 0, d_cut = 0;
  uint32_t d_pre = 0;
  if (FIN && *t.fin_apply) {
    r0 = t.chunk_off[c];
    r1 = t.chunk_off[c + 1];
    d_all = t.prev_sel->all;   // the previous dividing selection (membership)
    d_pre = t.prev_sel->prefix;
    d_cut = t.prev_sel->cut_idx;
  }
  int32_t rj = -1;
  float rv1 = 0.f, rv2 = 0.f;
  if (FIN && r0 + (int)threadIdx.x < r1) {
    const int r = r0 + (int)threadIdx.x;
    rj = t.rec_idx[r];
    rv1 = t.rec_v1[r];
    rv2 = t.rec_v2[r];
  }
  {   // wait for the bulk copies
    uint32_t done = 0;
    do {
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
          : "=r"(done)
          : "r"(smem_u32(&bar))
          : "memory");
    } while (!done);
  }
  __syncthreads();   // (edge elements written by plain stores)
  if (FIN) {   // the previous iteration's deferred finalize
    auto member = [&](uint32_t key, int32_t j) {
      if (d_all == 1) return true;
      if (d_all == 2) return false;
      return key > d_pre || (key == d_pre && j <= d_cut);
    };
    auto patch = [&](int32_t j, float a1, float a2) {
      const int sp = (int)(j - A);
      const float x = s_c[sp];
      s_c[sp] = fin_fold(x, !member(mag_key(x), j), a1, a2);
    };
    if (rj >= 0) patch(rj, rv1, rv2);
    for (int q = r0 + (int)threadIdx.x + kThreads; q < r1; q += kThreads)
      patch(t.rec_idx[q], t.rec_v1[q], t.rec_v2[q]);
    __syncthreads();
  }
  uint32_t mask = 0;
  bool nan = false;
#pragma unroll
  for (int it = 0; it < ITER; ++it) {
    const int q4 = warp * (32 * ITER) + it * 32 + lane;
    const int64_t i0 = A + (int64_t)q4 * 4;
    float4 cc = reinterpret_cast<const float4*>(s_c)[q4];
    if (APPLY) {
      const float4 gg = reinterpret_cast<const float4*>(s_g)[q4];
      cc.x = __fadd_rn(gg.x, cc.x);
      cc.y = __fadd_rn(gg.y, cc.y);
      cc.z = __fadd_rn(gg.z, cc.z);
      cc.w = __fadd_rn(gg.w, cc.w);
      reinterpret_cast<float4*>(s_c)[q4] = cc;
      if (i0 >= v0 && i0 + 4 <= v1) __stcs(reinterpret_cast<float4*>(carry + i0), cc);
    }
    const float ov[4] = {cc.x, cc.y, cc.z, cc.w};
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int64_t i = i0 + e;
      if (i >= lo && i < hi) {
        const uint32_t k = mag_key(ov[e]);
        nan |= k > 0x7f800000u;
        if (k >= pre) mask |= 1u << (it * 4 + e);
        if (APPLY && (i < v0 || i >= v1)) carry[i] = ov[e];   // edge element
      }
    }
  }
  if (nan) *t.err = 1;
  if (cand) cand_compact(t, c, A, mask, s_c, wf ? s_wh : nullptr, &s_wab, wb, wsh);
  if (wf) div_wsel_epilogue(t, s_wh, &s_wab, cand);
}

// FIN: the deferred finalize of the previous iteration (records, see
// FinRecTask) is applied to the chunk's carry before the gradient is added
// (when *t.fin_apply).  The records of the chunk (~1 % of its elements, index
// order) are loaded while the chunk streams in and marked in a bitmap of the
// chunk's positions; the carry stays in registers, and an element whose bit
// is set takes its record (its rank among the set bits) as it is combined.
constexpr int kFinRecMax = 256;    // records per chunk handled in place (else: staged)
#ifndef SPARDL_DIV_FIN_MINB
#define SPARDL_DIV_FIN_MINB 3
#endif

template <int APPLY, int FIN>
__global__ void __launch_bounds__(kThreads, FIN ? SPARDL_DIV_FIN_MINB : SPARDL_DIV_MINB)
    k_div_cand(const DivTask* __restrict__ tasks) {
  pdl_enter();
  const DivTask& t = tasks[blockIdx.y];
  const int c = blockIdx.x;
  // the wide select's window histogram of the candidates (t.ws)
  __shared__ uint32_t s_wh[kWBins];
  __shared__ uint32_t s_wab;
  const bool wf = t.ws != nullptr && t.ws_fused;
  if (c >= t.nchunks) {
    if (wf) div_wsel_epilogue(t, s_wh, &s_wab, false);
    return;
  }
  uint32_t wb = 0, wsh = 0;
  if (wf) {
    for (int b = threadIdx.x; b < kWBins; b += kThreads) s_wh[b] = 0;
    if (threadIdx.x == 0) s_wab = 0;
    wb = t.ws->base;
    wsh = t.ws->shift;
  }
  // participation in the look-back is decided by the pre-threshold kernel
  // only (bit 0), never by an overflow seen later in this kernel (bit 1)
  const bool cand = !(*t.cand_bad & 1);
  const uint32_t pre = *t.pre_key;
  const int64_t A = chunk_origin(t) + (int64_t)c * kChunk;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int ITER = kChunk / (kThreads * 4);   // float4 groups per lane
  // the combined values wait here for the compaction (registers are the
  // occupancy limit: the loads in flight need them)
  __shared__ __align__(16) float s_comb[kChunk];
  uint32_t mask = 0;
  bool nan = false;
  const int64_t lo = t.lo, hi = t.hi;
  // gradient and carry never alias; telling the compiler so lets every load
  // of the chunk issue before the first store (one memory latency per CTA
  // instead of one per float4 group)
  const float* __restrict__ g = APPLY ? t.g_tab[t.g_id] : nullptr;
  float* __restrict__ carry = t.carry;
  float4 gv[ITER], cv4[ITER];
#pragma unroll
  for (int it = 0; it < ITER; ++it) {
    const int64_t i0 = A + ((int64_t)warp * (32 * ITER) + it * 32 + lane) * 4;
    if (i0 >= lo && i0 + 4 <= hi) {
      if (APPLY) gv[it] = __ldcs(reinterpret_cast<const float4*>(g + i0));
      cv4[it] = __ldcs(reinterpret_cast<const float4*>(carry + i0));
    }
  }
  // (every chunk load is issued before anything below waits on memory)
  int r0 = 0, r1 = 0;
  if (FIN && *t.fin_apply) {
    r0 = t.chunk_off[c];
    r1 = t.chunk_off[c + 1];
  }
  // ---- the chunk's finalize records, while the chunk streams in
  __shared__ uint32_t s_bits[kChunk / 32];     // positions with a record
  __shared__ int s_wpre[kChunk / 32];          // records before each word
  __shared__ float s_rv[2][kFinRecMax];
  __shared__ int s_scr[40];
  int32_t d_all = 0, d_cut = 0;
  uint32_t d_pre = 0;
  const bool fin = FIN && r1 > r0;                      // uniform per CTA
  const int nrec = r1 - r0;
  if (fin) {
    d_all = t.prev_sel->all;   // the previous dividing selection (membership)
    d_pre = t.prev_sel->prefix;
    d_cut = t.prev_sel->cut_idx;
    s_bits[threadIdx.x] = 0;   // (kChunk / 32 == kThreads words)
    __syncthreads();
    for (int q = threadIdx.x; q < min(nrec, kFinRecMax); q += kThreads) {
      const int sp = (int)(t.rec_idx[r0 + q] - A);
      atomicOr(&s_bits[sp >> 5], 1u << (sp & 31));
      s_rv[0][q] = t.rec_v1[r0 + q];
      s_rv[1][q] = t.rec_v2[r0 + q];
    }
    __syncthreads();
    int tot;
    s_wpre[threadIdx.x] = block_exscan(__popc(s_bits[threadIdx.x]), s_scr, &tot);
    __syncthreads();
  }
  auto fin_value = [&](int sp, float x) {   // the carry at chunk position sp
    const uint32_t wd = s_bits[sp >> 5];
    if (!((wd >> (sp & 31)) & 1u)) return x;
    const int r = s_wpre[sp >> 5] + __popc(wd & ((1u << (sp & 31)) - 1u));
    const int32_t j = (int32_t)(A + sp);
    const uint32_t key = mag_key(x);
    const bool member = d_all == 1 || (d_all == 0 && (key > d_pre || (key == d_pre && j <= d_cut)));
    return fin_fold(x, !member, s_rv[0][r], s_rv[1][r]);
  };
  const bool big = fin && nrec > kFinRecMax;   // rare: records past the table, patched below
#pragma unroll
  for (int it = 0; it < ITER; ++it) {
    const int64_t i0 = A + ((int64_t)warp * (32 * ITER) + it * 32 + lane) * 4;
    const int sp0 = (warp * (32 * ITER) + it * 32 + lane) * 4;
    if (i0 >= lo && i0 + 4 <= hi) {
      float4 cc = cv4[it];
      if (fin && !big && s_bits[sp0 >> 5]) {
        cc.x = fin_value(sp0, cc.x);
        cc.y = fin_value(sp0 + 1, cc.y);
        cc.z = fin_value(sp0 + 2, cc.z);
        cc.w = fin_value(sp0 + 3, cc.w);
      }
      cv4[it] = cc;
    }
  }
  if (big) {   // every record through shared memory (a dense chunk of records)
#pragma unroll
    for (int it = 0; it < ITER; ++it) {
      const int64_t i0 = A + ((int64_t)warp * (32 * ITER) + it * 32 + lane) * 4;
      const int sp0 = (warp * (32 * ITER) + it * 32 + lane) * 4;
      if (i0 >= lo && i0 + 4 <= hi) {
        reinterpret_cast<float4*>(s_comb)[sp0 >> 2] = cv4[it];
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (i0 + e >= lo && i0 + e < hi) s_comb[sp0 + e] = carry[i0 + e];
      }
    }
    __syncthreads();
    for (int q = r0 + (int)threadIdx.x; q < r1; q += kThreads) {
      const int32_t j = t.rec_idx[q];
      const int sp = (int)(j - A);
      const float x = s_comb[sp];
      const uint32_t key = mag_key(x);
      const bool member =
          d_all == 1 || (d_all == 0 && (key > d_pre || (key == d_pre && j <= d_cut)));
      s_comb[sp] = fin_fold(x, !member, t.rec_v1[q], t.rec_v2[q]);
    }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < ITER; ++it) {
      const int64_t i0 = A + ((int64_t)warp * (32 * ITER) + it * 32 + lane) * 4;
      if (i0 >= lo && i0 + 4 <= hi)
        cv4[it] = reinterpret_cast<const float4*>(s_comb)[warp * (32 * ITER) + it * 32 + lane];
    }
    __syncthreads();
  }
#pragma unroll
  for (int it = 0; it < ITER; ++it) {
    const int64_t i0 = A + ((int64_t)warp * (32 * ITER) + it * 32 + lane) * 4;
    if (i0 >= lo && i0 + 4 <= hi) {
      const float4 cc = cv4[it];
      float4 o;
      if (APPLY) {
        const float4 gg = gv[it];
        o.x = __fadd_rn(gg.x, cc.x);
        o.y = __fadd_rn(gg.y, cc.y);
        o.z = __fadd_rn(gg.z, cc.z);
        o.w = __fadd_rn(gg.w, cc.w);
        __stcs(reinterpret_cast<float4*>(carry + i0), o);
      } else {
        o = cc;
      }
      reinterpret_cast<float4*>(s_comb)[warp * (32 * ITER) + it * 32 + lane] = o;
      const float ov[4] = {o.x, o.y, o.z, o.w};
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const uint32_t k = mag_key(ov[e]);
        nan |= k > 0x7f800000u;
        if (k >= pre) mask |= 1u << (it * 4 + e);
      }
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int64_t i = i0 + e;
        const int sp = (warp * (32 * ITER) + it * 32 + lane) * 4 + e;
        const float staged = big ? s_comb[sp] : 0.f;   // (big: patched in place)
        s_comb[sp] = 0.f;
        if (i >= lo && i < hi) {
          float x = big ? staged : carry[i];
          if (fin && !big) x = fin_value(sp, x);   // an edge element with a record
          if (APPLY) {
            x = __fadd_rn(g[i], x);
            carry[i] = x;
          }
          s_comb[sp] = x;
          const uint32_t k = mag_key(x);
          nan |= k > 0x7f800000u;
          if (k >= pre) mask |= 1u << (it * 4 + e);
        }
      }
    }
  }
  if (nan) *t.err = 1;
  if (cand) cand_compact(t, c, A, mask, s_comb, wf ? s_wh : nullptr, &s_wab, wb, wsh);
  if (wf) div_wsel_epilogue(t, s_wh, &s_wab, cand);
}

// One CTA per task: the work list of the dividing select -- every chunk
// segment cut into tiles of <= kTile candidates, in chunk (= index) order --
// and the candidate total.  Unused tile slots get count 0.
__device__ void div_tiles_body(const DivTask& t, int* scratch) {
  int tile_carry = 0, cand_carry = 0;
  for (int c0 = 0; c0 < t.nchunks; c0 += blockDim.x) {
    const int c = c0 + threadIdx.x;
    const int cnt = c < t.nchunks ? t.cand_cnt[c] : 0;
    const int tl = t.tile_len;
    const int nt = (cnt + tl - 1) / tl;
    int ttot, ctot;
    const int tbase = tile_carry + block_exscan(nt, scratch, &ttot);
    block_exscan(cnt, scratch, &ctot);
    for (int j = 0; j < nt; ++j) {
      const int q = tbase + j;
      if (q < t.max_tiles) {
        t.tile_off[q] = c * t.cap + j * tl;
        t.tile_cnt[q] = min(tl, cnt - j * tl);
      }
    }
    tile_carry += ttot;
    cand_carry += ctot;
  }
  for (int q = tile_carry + threadIdx.x; q < t.max_tiles; q += blockDim.x) t.tile_cnt[q] = 0;
  if (threadIdx.x == 0) {
    *t.cand_total = cand_carry;
    *t.ntiles = min(tile_carry, t.max_tiles);
    if (tile_carry > t.max_tiles) *t.cand_bad |= 4;   // work list capacity: dense fallback
  }
  __syncthreads();
}

// Second chance.  A block whose carried pre-threshold missed -- fewer than L
// candidates, a chunk segment overflowing, or (cluster select) more tiles
// than its work list -- would otherwise go down the exact dense path (a
// select over the whole block: ~270 us per block at C4).  Instead this CTA
// samples the block's combined values (now in the carry) as k_div_sample
// does, puts the pre-threshold at a wider margin (1.5 L + 6 sigma of the
// sample), resets the block's history (the select re-fits it from this run)
// and marks the block (bit 3) for k_div_recand, which recompacts its
// candidates from the carry.  Only a second miss takes the dense path.
__device__ void div_resample(const DivTask& t, uint32_t* h, int* scratch) {
  constexpr int BPT = kSampBins / 1024;   // bins per thread (blockDim.x == 1024)
  for (int b = threadIdx.x; b < kSampBins; b += blockDim.x) h[b] = 0;
  __syncthreads();
  for (int c = 0; c < t.nchunks; c += t.sample_every) {
    const int64_t A = chunk_origin(t) + (int64_t)c * kChunk;
    const int64_t s = A > t.lo ? A : t.lo;
    const int64_t e = (A + kChunk) < t.hi ? (A + kChunk) : t.hi;
    for (int64_t i = s + threadIdx.x; i < e; i += blockDim.x)
      atomicAdd(&h[mag_key(__ldcg(t.carry + i)) >> kSampShift], 1u);
  }
  __syncthreads();
  // thread r holds bins [(1023 - r) * BPT, +BPT): thread order = key order, descending
  const int r = blockDim.x - 1 - threadIdx.x;
  int mine = 0;
  for (int q = 0; q < BPT; ++q) mine += (int)h[r * BPT + q];
  int ns = 0;
  const int above = block_exscan(mine, scratch, &ns);
  const double expect = (double)t.budget / (double)((int64_t)t.hi - t.lo) * (double)ns;
  const long long target = (long long)(1.5 * expect + 6.0 * sqrt(expect + 1.0) + 16.0);
  __shared__ int s_ok;
  if (threadIdx.x == 0) s_ok = 0;
  __syncthreads();
  if (target < ns && above < target && target <= above + mine) {
    long long cum = above;
    for (int q = BPT - 1; q >= 0; --q) {
      const uint32_t cq = h[r * BPT + q];
      if (cum + (long long)cq >= target) {
        const uint32_t pre = (uint32_t)(r * BPT + q) << kSampShift;
        *t.pre_key = pre;
        if (t.ws) {   // the wide select's window (as k_div_prethr sets it)
          uint32_t sh = 0;
          while (sh < 31 && ((unsigned long long)kWBins << sh) < 4ull * (8u << kSampShift)) ++sh;
          t.ws->base = pre;
          t.ws->shift = sh;
        }
        s_ok = 1;
        break;
      }
      cum += cq;
    }
  }
  __syncthreads();
  if (threadIdx.x == 0 && s_ok) {
    *t.cand_bad = 8;
    *t.cand_total = 0;
    t.hist->valid = 0;   // re-fitted by this run's select from the new pre-threshold
    if (t.retries) atomicAdd(t.retries, 1ull);
  }
}

// PHASE 0 (after k_div_cand): the work list, or the second chance on a
// miss.  PHASE 1 (after k_div_recand): the work list of the blocks redone.
template <int PHASE>
__global__ void __launch_bounds__(1024) k_div_tiles(const DivTask* __restrict__ tasks) {
  pdl_enter();
  const DivTask& t = tasks[blockIdx.x];
  __shared__ int scratch[40];
  if (PHASE == 1) {
    if (!(*t.cand_bad & 8)) return;
    div_tiles_body(t, scratch);
    if (threadIdx.x == 0) *t.cand_bad &= ~8;
    return;
  }
  if (*t.cand_bad & 1) return;
  div_tiles_body(t, scratch);
  const int bad = *t.cand_bad;
  const bool miss = t.use_cand &&
                    ((bad & 2) || *t.cand_total < t.budget || (!t.huge && (bad & 4)));
  if (!miss) return;   // (uniform: every thread read the same words after the barrier)
  __shared__ uint32_t h[kSampBins];
  div_resample(t, h, scratch);
}

// The candidates of the blocks marked by the second chance (bit 3),
// recompacted from the carry (the combined values, written by k_div_cand)
// with the new pre-threshold.  A persistent grid over (block, chunk); with
// no block marked -- the normal case -- every CTA exits after reading the
// flags.
__global__ void __launch_bounds__(kThreads) k_div_recand(const DivTask* __restrict__ tasks,
                                                         int ntask, int max_chunks) {
  pdl_enter();
  int any = 0;
  for (int q = threadIdx.x; q < ntask; q += blockDim.x) any |= (*tasks[q].cand_bad & 8);
  if (!__syncthreads_or(any)) return;
  __shared__ __align__(16) float s_comb[kChunk];
  constexpr int ITER = kChunk / (kThreads * 4);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long items = (long long)ntask * max_chunks;
  for (long long w = blockIdx.x; w < items; w += gridDim.x) {
    const DivTask& t = tasks[w / max_chunks];
    const int c = (int)(w % max_chunks);
    if (c >= t.nchunks || !(*t.cand_bad & 8)) continue;   // uniform per CTA
    const uint32_t pre = *t.pre_key;
    const int64_t A = chunk_origin(t) + (int64_t)c * kChunk;
    const int64_t lo = t.lo, hi = t.hi;
    uint32_t mask = 0;
    __syncthreads();   // s_comb of the previous item fully consumed
#pragma unroll
    for (int it = 0; it < ITER; ++it) {
      const int sp0 = (warp * (32 * ITER) + it * 32 + lane) * 4;
      const int64_t i0 = A + sp0;
      float v[4];
      if (i0 >= lo && i0 + 4 <= hi) {
        const float4 x = __ldcg(reinterpret_cast<const float4*>(t.carry + i0));
        v[0] = x.x; v[1] = x.y; v[2] = x.z; v[3] = x.w;
      } else {
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] = (i0 + e >= lo && i0 + e < hi) ? t.carry[i0 + e] : 0.f;
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        s_comb[sp0 + e] = v[e];
        if (i0 + e >= lo && i0 + e < hi && mag_key(v[e]) >= pre) mask |= 1u << (it * 4 + e);
      }
    }
    cand_compact(t, c, A, mask, s_comb);
  }
}

}  // namespace

int launch_divide(const DivTask* tasks_dev, int ntask, int max_chunks, int sample_every,
                  int apply_residual, cudaStream_t s, int part) {
  if (ntask <= 0) return 0;
  int n = 0;
  if (part != 2) {
    // sample_every is uniform across a batch (set by the planner)
    const int sx = (max_chunks + sample_every - 1) / sample_every;
    const int smem = kSampBins * (int)sizeof(uint32_t);
    static bool configured[kMaxDevices] = {};   // per device (benign race: idempotent)
    const int dev = cur_device();
    if (!configured[dev]) {
      cudaFuncSetAttribute(k_div_sample, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      configured[dev] = true;
    }
    launch_pdl(k_div_sample, dim3(sx, ntask), dim3(kThreads), smem, s, tasks_dev, apply_residual);
    launch_pdl(k_div_prethr, dim3(ntask), dim3(kThreads), 0, s, tasks_dev);
    n += 2;
  }
  if (part != 1) {
    static const bool bulk = [] {
      const char* e = getenv("SPARDL_DIV_BULK");   // 1: the bulk-copy (TMA) form
      return e && e[0] == '1';
    }();
    if (bulk) {
      constexpr int smem = 2 * kChunk * (int)sizeof(float);
      static bool configured[kMaxDevices][3] = {};
      const int dev = cur_device();
      auto k = apply_residual == 2 ? k_div_cand_bulk<1, 1>
                                   : (apply_residual ? k_div_cand_bulk<1, 0> : k_div_cand_bulk<0, 0>);
      const int v = apply_residual == 2 ? 2 : (apply_residual ? 1 : 0);
      if (!configured[dev][v]) {
        cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        configured[dev][v] = true;
      }
      launch_pdl(k, dim3(max_chunks, ntask), dim3(kThreads), smem, s, tasks_dev);
    } else if (apply_residual == 2) {   // + the previous iteration's deferred finalize
      launch_pdl(k_div_cand<1, 1>, dim3(max_chunks, ntask), dim3(kThreads), 0, s, tasks_dev);
    } else if (apply_residual) {
      launch_pdl(k_div_cand<1, 0>, dim3(max_chunks, ntask), dim3(kThreads), 0, s, tasks_dev);
    } else {
      launch_pdl(k_div_cand<0, 0>, dim3(max_chunks, ntask), dim3(kThreads), 0, s, tasks_dev);
    }
    launch_pdl(k_div_tiles<0>, dim3(ntask), dim3(1024), 0, s, tasks_dev);
    // the second chance (no-ops unless a block's pre-threshold missed)
    static int recand_grid[kMaxDevices] = {};
    const int dev = cur_device();
    if (!recand_grid[dev]) {
      int sms = 0, per = 0;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_div_recand, kThreads, 0);
      recand_grid[dev] = std::max(1, sms) * std::max(1, per);
    }
    launch_pdl(k_div_recand, dim3(recand_grid[dev]), dim3(kThreads), 0, s, tasks_dev, ntask,
               max_chunks);
    launch_pdl(k_div_tiles<1>, dim3(ntask), dim3(1024), 0, s, tasks_dev);
    n += 4;
  }
  return n;
}

}  // namespace sdl
