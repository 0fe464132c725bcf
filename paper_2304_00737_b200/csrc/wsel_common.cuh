// Level-1 decision of the wide select (wselect.cu), shared with the
// dividing candidate pass (divide.cu), which histograms its candidates
// itself: the CTA that completes a task's histogram fixes the run state,
// the boundary bin and this run's geometry, and zeroes the histogram.
// Whole CTA of kWDecideThreads threads.
#pragma once

#include "common.cuh"
#include "kernels.cuh"

namespace sdl {
namespace {

constexpr int kWDecideThreads = 256;

// level-1 bin of a key: 0..kWBins-1, kWBins = above the window, -1 = below
__device__ __forceinline__ int w_bin(int mode, uint32_t base, uint32_t shift, uint32_t key) {
  if (mode == kWFull) return (int)(key >> 20);
  if (key < base) return -1;
  const uint32_t d = (key - base) >> shift;
  return d >= (uint32_t)kWBins ? kWBins : (int)d;
}

// this run's histogram geometry of a task (identical in every CTA of the
// histogram and gather kernels: the previous threshold is only rewritten by
// the finisher, after every gather CTA has classified its tile)
__device__ __forceinline__ void w_geometry(const SelTask& t, const WScratch& w, int& mode,
                                           uint32_t& base, uint32_t& shift) {
  if (w.mode == kWWindow) {
    mode = kWWindow;
    base = w.base;
    shift = w.shift;
    return;
  }
  const SelScratch* sc = t.scr;
  const uint32_t prev = sc->prefix;
  if (sc->all == 0 && prev != 0) {
    mode = kWWindow;
    shift = kWAutoShift;
    const uint32_t half = (uint32_t)(kWBins / 2) << kWAutoShift;
    base = prev > half ? prev - half : 0u;
  } else {
    mode = kWFull;
    base = 0;
    shift = 20;
  }
}


// The bin holding the need-th largest key of the level-1 histogram (every
// thread of the CTA gets the result).  Returns false if the histogram (plus
// `above`) holds fewer than `need` entries.  *before = entries in higher bins
// (including `above`).
__device__ bool w_locate(const uint32_t* __restrict__ hist, long long above, long long need,
                         int* bin, long long* before, int* scratch, long long* sh) {
  constexpr int BPT = kWBins / kWDecideThreads;   // 8 bins per thread
  __shared__ int s_bin;
  __shared__ long long s_before;
  const int tid = threadIdx.x;
  const int g = kWDecideThreads - 1 - tid;        // this thread's bin group, top groups first
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


// total: entries of this run (candidates for the dividing select); bad: the
// input cannot be selected here (dividing candidates incomplete).
__device__ void w_decide(WScratch* ws, long long total, bool bad, long long budget, int mode,
                         uint32_t base, uint32_t shift, int* scratch, long long* lsh) {
  const int tid = threadIdx.x;
  const long long above = __ldcg(&ws->above);
  int state, bstar = -1;
  long long before = 0;
  if (bad) state = kWFallback;
  else if (total <= budget) state = kWAll;
  else if (budget <= 0) state = kWNone;
  else if (above >= budget) state = kWFallback;   // threshold above the window
  else state = w_locate(ws->hist, above, budget, &bstar, &before, scratch, lsh) ? kWOk : kWFallback;
  const uint32_t expect = bstar >= 0 ? __ldcg(ws->hist + bstar) : 0u;
  __syncthreads();
  for (int b = tid; b < kWBins; b += kWDecideThreads) ws->hist[b] = 0;
  if (tid == 0) {
    ws->state = state;
    ws->run_mode = mode;
    ws->run_base = base;
    ws->run_shift = shift;
    ws->bstar = bstar;
    ws->before = before;
    ws->bin_expect = expect;
    ws->total_in = total;
    ws->above = 0;
    ws->below = 0;
    ws->harrive = 0;
  }
}

// every bin of the task's histogram summed (the CTA's threads)
__device__ __forceinline__ long long w_hist_total(const WScratch* ws, long long* lsh) {
  long long part = 0;
  for (int b = threadIdx.x; b < kWBins; b += kWDecideThreads) part += __ldcg(ws->hist + b);
  long long u0 = 0, u1 = 0;
  block_sum3_ll(part, u0, u1, lsh);
  return part;
}

}  // namespace
}  // namespace sdl
