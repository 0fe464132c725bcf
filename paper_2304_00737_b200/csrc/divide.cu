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
#include "common.cuh"
#include "kernels.cuh"

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
  uint32_t* hist = t.samp_hist + threadIdx.x * BPT;
  long long mine = 0;
  for (int q = 0; q < BPT; ++q) mine += hist[q];
  const long long ns = block_sum_ll(mine, lscr);
  const int64_t nb = (int64_t)t.hi - t.lo;
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
    if (threadIdx.x == 0) {
      *t.cand_total = 0;
      *t.cand_bad = 0;
      *t.pre_key = t.hist->next_pre;
      set_window(t.hist->next_pre, t.hist->delta);
    }
    return;   // the sample histogram was not touched: still zero
  }
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

template <int APPLY>
__global__ void __launch_bounds__(kThreads, SPARDL_DIV_MINB) k_div_cand(const DivTask* __restrict__ tasks) {
  pdl_enter();
  const DivTask& t = tasks[blockIdx.y];
  const int c = blockIdx.x;
  if (c >= t.nchunks) return;
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
        s_comb[(warp * (32 * ITER) + it * 32 + lane) * 4 + e] = 0.f;
        if (i >= lo && i < hi) {
          float x = carry[i];
          if (APPLY) {
            x = __fadd_rn(g[i], x);
            carry[i] = x;
          }
          s_comb[(warp * (32 * ITER) + it * 32 + lane) * 4 + e] = x;
          const uint32_t k = mag_key(x);
          nan |= k > 0x7f800000u;
          if (k >= pre) mask |= 1u << (it * 4 + e);
        }
      }
    }
  }
  if (nan) *t.err = 1;
  if (!cand) return;
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
  // the wide select's level-1 histogram of the candidates (window above the
  // pre-threshold; fire-and-forget reductions)
  WScratch* ws = t.ws;
  const uint32_t wb = ws ? ws->base : 0u, wsh = ws ? ws->shift : 0u;
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
        if (ws) {
          const uint32_t d = (mag_key(x) - wb) >> wsh;
          atomicAdd(d < (uint32_t)kWBins ? &ws->hist[d] : &ws->above, 1u);
        }
      }
    }
  }
  if (threadIdx.x == 0) t.cand_cnt[c] = total;
}

// One CTA per task: the work list of the dividing select -- every chunk
// segment cut into tiles of <= kTile candidates, in chunk (= index) order --
// and the candidate total.  Unused tile slots get count 0.
__global__ void __launch_bounds__(1024) k_div_tiles(const DivTask* __restrict__ tasks) {
  pdl_enter();
  const DivTask& t = tasks[blockIdx.x];
  __shared__ int scratch[40];
  if (*t.cand_bad & 1) return;
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
    if (tile_carry > t.max_tiles) *t.cand_bad |= 2;   // work list capacity: dense fallback
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
    if (apply_residual)
      launch_pdl(k_div_cand<1>, dim3(max_chunks, ntask), dim3(kThreads), 0, s, tasks_dev);
    else
      launch_pdl(k_div_cand<0>, dim3(max_chunks, ntask), dim3(kThreads), 0, s, tasks_dev);
    launch_pdl(k_div_tiles, dim3(ntask), dim3(1024), 0, s, tasks_dev);
    n += 2;
  }
  return n;
}

}  // namespace sdl
