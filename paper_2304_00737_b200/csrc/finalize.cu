// Global-gradient assembly, residual finalize, ledger and the B-SAG
// controller on the device.
#include <algorithm>
#include <climits>

#include "common.cuh"
#include "kernels.cuh"

namespace sdl {

namespace {

// ---------------------------------------------------------------------------
// Assembly: the global gradient is the concatenation of the m reserved
// blocks in position order (inc/pipeline.hpp:279-291); blocks cover
// increasing index ranges, so the result is index-sorted.
// off[] holds m + 1 ints of dynamic shared memory (any team size).
__global__ void __launch_bounds__(kThreads) k_assemble(const AssembleTask* __restrict__ tasks) {
  pdl_enter();
  const AssembleTask& t = tasks[blockIdx.y];
  peer_wait(t.ps);   // the gathered blocks of other GPUs are published
  extern __shared__ int off[];
  __shared__ int s_part[40];   // block_exscan scratch (>= 33 ints)
  {   // block offsets: CTA-wide exclusive scan of the m counts
    int run = 0;
    for (int b0 = 0; b0 < t.m; b0 += kThreads) {
      const int b = b0 + threadIdx.x;
      const int c = b < t.m ? *t.src[b].cnt : 0;
      int tot = 0;
      const int ex = block_exscan(c, s_part, &tot);
      if (b < t.m) off[b] = run + ex;
      run += tot;
    }
    if (threadIdx.x == 0) {
      off[t.m] = run;
      if (blockIdx.x == 0) *t.out_cnt = run;
    }
  }
  __syncthreads();
  const int total = off[t.m];
  unsigned long long h = 0;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < total; p += gridDim.x * blockDim.x) {
    const int b = upper_bound_i32(off, t.m + 1, p) - 1;   // off[b] <= p < off[b + 1]
    const int j = p - off[b];
    const int32_t ix = t.src[b].idx[j];
    const float v = t.src[b].val[j];
    t.out_idx[p] = ix;
    t.out_val[p] = v;
    if (t.out_hash) {
      unsigned long long x = ((unsigned long long)(uint32_t)ix << 32) | __float_as_uint(v);
      x ^= (unsigned long long)p * 0x9E3779B97F4A7C15ull;
      x ^= x >> 33;
      x *= 0xff51afd7ed558ccdull;
      x ^= x >> 33;
      x *= 0xc4ceb9fe1a85ec53ull;
      x ^= x >> 33;
      h += x;
    }
  }
  if (t.out_hash) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) h += __shfl_down_sync(0xffffffffu, h, o);
    if ((threadIdx.x & 31) == 0 && h)
      atomicAdd(reinterpret_cast<unsigned long long*>(t.out_hash), h);
  }
}

// ---------------------------------------------------------------------------
// Residual finalize (inc/residual.hpp:128-160), one task per worker.
//   gres: carry[j] = xi(j) for j in the global gradient; xi(j) starts as
//         combined[j] when the dividing select discarded j (that discard is
//         recorded first, inc/pipeline.hpp:177-180) and then folds every
//         in-procedure discard of j in recording order; absent -> +0.
//   pres: carry[j] = 0 for j in the global gradient.
//   lres: carry = dividing remainder, i.e. combined with the dividing
//         selections zeroed (handled by k_finalize_lres).
// Off the global gradient the carry already holds g_copy (in place).
// Warp-cooperative lower/upper bound over a sorted global array (32-ary
// search: ~log32(n) rounds of one load per lane instead of log2(n)
// dependent loads).  Must be called by a full warp.
__device__ __forceinline__ int warp_bound(const int32_t* a, int n, int32_t x, bool upper) {
  const int lane = threadIdx.x & 31;
  int lo = 0, hi = n;   // answer in [lo, hi]
  while (hi - lo > 32) {
    const int step = (hi - lo + 31) / 32;
    const int p = lo + lane * step;
    const int32_t v = p < hi ? a[p] : INT_MAX;
    const bool below = upper ? (v <= x) : (v < x);
    const int c = __popc(__ballot_sync(0xffffffffu, below && p < hi));
    if (c == 0) {
      hi = lo;
    } else {
      const int nlo = lo + (c - 1) * step + 1;
      const int nhi = lo + c * step;
      lo = nlo;
      hi = nhi < hi ? nhi : hi;
    }
  }
  const int p = lo + lane;
  const int32_t v = p < hi ? a[p] : INT_MAX;
  const bool below = p < hi && (upper ? (v <= x) : (v < x));
  return lo + __popc(__ballot_sync(0xffffffffu, below));
}

// One CTA per (worker, block b, chunk of 256 global entries of block b).
// The dividing-selection membership comes from the dividing select's
// threshold (no search); each in-procedure discard list is joined with the
// chunk through a shared-memory binary search over the chunk's indices.
#ifndef SPARDL_FIN_CHUNK
#define SPARDL_FIN_CHUNK 1024
#endif
constexpr int kFinChunk = SPARDL_FIN_CHUNK;  // global entries per CTA
constexpr int kFinPer = kFinChunk / kThreads;

constexpr int kXiBatch = 4;                  // discard entries per thread per batch
constexpr int kFinLists = 4;                 // discard lists joined before the carry is read
constexpr int kMaxXiLists = kThreads / 64;   // bound searches in parallel (2 warps each)

#ifndef SPARDL_FIN_MINB
#define SPARDL_FIN_MINB 6   // (<= 40 registers, a small spill; C4 one GPU: finalize 0.260 -> 0.224 ms against 4)
#endif
__global__ void __launch_bounds__(kThreads, SPARDL_FIN_MINB)
    k_finalize(const FinalizeTask* __restrict__ tasks, const int32_t* abort) {
  pdl_enter();
  if (err_set(abort)) return;   // void iteration (peer timeout): carry untouched
  const FinalizeTask& t = tasks[blockIdx.z];
  if (t.mode == 2) return;   // lres ignores the global gradient
  peer_wait(t.ps);           // remote blocks of the global gradient published
  const int b = blockIdx.y;
  const GatherSrc G = t.gblk[b];
  const int gn = *G.cnt;
  const int c0 = blockIdx.x * kFinChunk;
  if (c0 >= gn) return;
  const int nloc = min(kFinChunk, gn - c0);
  const int tid = threadIdx.x;
  float* __restrict__ carry = t.carry;
  // audit: this block's place in the assembled global gradient
  __shared__ int s_off;
  if (t.aud_comb) {
    if (tid == 0) {
      int o = 0;
      for (int q = 0; q < b; ++q) o += *t.gblk[q].cnt;
      s_off = o;
    }
    __syncthreads();
  }
  if (t.mode == 1) {   // pres: zero at the global indices
    for (int e = tid; e < nloc; e += kThreads) {
      const int32_t j = G.idx[c0 + e];
      if (t.aud_comb) {
        t.aud_comb[s_off + c0 + e] = carry[j];
        t.aud_carry[s_off + c0 + e] = 0.f;
      }
      carry[j] = 0.f;
    }
    return;
  }
  __shared__ int32_t gi[kFinChunk];
  __shared__ float sv[kFinChunk];
  __shared__ unsigned char sf[kFinChunk];
  __shared__ int range[2 * kMaxXiLists];
  // dividing-select state, read once
  const SelScratch* dsc = t.div_sc[b];
  const int d_all = dsc->all;
  const uint32_t d_pre = dsc->prefix;
  const int32_t d_cut = dsc->cut_idx;
  auto div_member = [&](uint32_t key, int32_t j) {
    if (d_all == 1) return true;
    if (d_all == 2) return false;
    return key > d_pre || (key == d_pre && j <= d_cut);
  };
  int32_t jj[kFinPer];
#pragma unroll
  for (int q = 0; q < kFinPer; ++q) {
    const int e = tid + q * kThreads;
    jj[q] = e < nloc ? G.idx[c0 + e] : INT_MAX;
    gi[e] = jj[q];
  }
  const int x0 = t.xi_off[b], x1 = t.xi_off[b + 1];
  // With <= kFinLists discard lists the join runs first and the carry is
  // read and written back in one go (its sector is still in L2 for the
  // write); otherwise the carry is read first and folded list by list.
  const bool late = x1 - x0 <= kFinLists;
  float x[kFinPer], acc[kFinPer];
  bool present[kFinPer];
  int nd[kFinPer];
#pragma unroll
  for (int q = 0; q < kFinPer; ++q) {
    x[q] = (!late && jj[q] != INT_MAX) ? carry[jj[q]] : 0.f;
    present[q] = !late && jj[q] != INT_MAX && !div_member(mag_key(x[q]), jj[q]);
    acc[q] = present[q] ? x[q] : 0.f;
    nd[q] = 0;
  }
  __shared__ float svl[kFinLists][kFinChunk];   // late mode: list li's value per entry
  __syncthreads();
  const int32_t jlo = gi[0], jhi = gi[nloc - 1];
  // Late mode without the audit: the dividing-selection membership comes from
  // joining the chunk with this worker's dividing selection of block b (the
  // list the select wrote, exactly the entries the threshold test accepts)
  // instead of reading the carry.  The carry is then touched only where the
  // residual changes: a member is overwritten (its residual is its discards,
  // no read), a non-member with discards is read, folded and written, a
  // non-member without discards keeps its combined value (no access) -- most
  // global entries come from other workers' selections.
  const bool join_div = late && !t.aud_comb;
  __shared__ unsigned char s_mem[kFinChunk];
  __shared__ int s_drange[2];
  // with fewer discard lists than bound-search warp pairs, the dividing list's
  // range is searched by a spare pair beside them (one dependent search phase
  // less per CTA)
  const bool d_fused = join_div && x1 > x0 && (x1 - x0) < kMaxXiLists;
  const GatherSrc D = t.div[b];
  if (join_div) {
#pragma unroll
    for (int q = 0; q < kFinPer; ++q) s_mem[tid + q * kThreads] = 0;
  }
  if (join_div && !d_fused) {
    if (tid < 64) {
      const int dn = *D.cnt;
      const bool upper = tid >= 32;
      const int r = warp_bound(D.idx, dn, upper ? jhi : jlo, upper);
      if ((tid & 31) == 0) s_drange[tid >> 5] = r;
    }
    __syncthreads();
    const int r0 = s_drange[0], r1 = s_drange[1];
    for (int p = r0 + tid; p < r1; p += kThreads) {
      const int32_t x = D.idx[p];
      const int ps = lower_bound_i32(gi, nloc, x);
      if (ps < nloc && gi[ps] == x) s_mem[ps] = 1;
    }
    __syncthreads();
  }
  for (int xb = x0; xb < x1; xb += kMaxXiLists) {
    const int nx = min(kMaxXiLists, x1 - xb);
    // the sub-range of each discard list inside [jlo, jhi], in parallel
    {
      const int warp = tid >> 5, li = warp >> 1;
      if (li < nx) {
        const XiList X = t.xi[xb + li];
        const int xn = *X.cnt;
        const bool upper = warp & 1;
        const int r = warp_bound(X.idx, xn, upper ? jhi : jlo, upper);
        if ((tid & 31) == 0) range[warp] = r;
      } else if (d_fused && xb == x0 && li == nx) {
        const bool upper = warp & 1;
        const int r = warp_bound(D.idx, *D.cnt, upper ? jhi : jlo, upper);
        if ((tid & 31) == 0) s_drange[warp & 1] = r;
      }
    }
#pragma unroll
    for (int q = 0; q < kFinPer; ++q) sf[tid + q * kThreads] = 0;
    __syncthreads();
    if (d_fused && xb == x0) {   // the dividing list's entries in this chunk (s_mem only)
      const int r0 = s_drange[0], r1 = s_drange[1];
      for (int p = r0 + tid; p < r1; p += kThreads) {
        const int32_t x = D.idx[p];
        const int ps = lower_bound_i32(gi, nloc, x);
        if (ps < nloc && gi[ps] == x) s_mem[ps] = 1;
      }
    }
    for (int li = 0; li < nx; ++li) {   // fold in recording order
      const XiList X = t.xi[xb + li];
      const int r0 = range[2 * li], r1 = range[2 * li + 1];
      float* dst = late ? svl[xb - x0 + li] : sv;
      for (int p0 = r0; p0 < r1; p0 += kThreads * kXiBatch) {
        int32_t xi[kXiBatch];
        int pos[kXiBatch];
#pragma unroll
        for (int u = 0; u < kXiBatch; ++u) {
          const int p = p0 + u * kThreads + tid;
          xi[u] = p < r1 ? X.idx[p] : INT_MIN;
        }
        float xv[kXiBatch];
#pragma unroll
        for (int u = 0; u < kXiBatch; ++u) {
          pos[u] = -1;
          if (xi[u] != INT_MIN) {
            const int ps = lower_bound_i32(gi, nloc, xi[u]);
            if (ps < nloc && gi[ps] == xi[u]) pos[u] = ps;
          }
          xv[u] = pos[u] >= 0 ? X.val[p0 + u * kThreads + tid] : 0.f;
        }
#pragma unroll
        for (int u = 0; u < kXiBatch; ++u)
          if (pos[u] >= 0) {
            dst[pos[u]] = xv[u];
            sf[pos[u]] = (unsigned char)(sf[pos[u]] | (1u << li));
          }
      }
      if (late) {
        __syncthreads();   // sf[e] is or-ed by list; one list at a time
      } else {
        __syncthreads();
#pragma unroll
        for (int q = 0; q < kFinPer; ++q) {
          const int e = tid + q * kThreads;
          if (e < nloc && sf[e]) {
            acc[q] = present[q] ? __fadd_rn(acc[q], sv[e]) : sv[e];
            present[q] = true;
            sf[e] = 0;
          }
        }
        __syncthreads();
      }
    }
    if (late) {   // bit li of sf[e]: list li holds entry e (all lists of this batch)
      __syncthreads();
#pragma unroll
      for (int q = 0; q < kFinPer; ++q) nd[q] = sf[tid + q * kThreads];
    }
  }
  bool skip[kFinPer];
#pragma unroll
  for (int q = 0; q < kFinPer; ++q) skip[q] = false;
  if (late && join_div) {   // the carry read only where it is kept and folded
#pragma unroll
    for (int q = 0; q < kFinPer; ++q) {
      const int e = tid + q * kThreads;
      const bool mem = jj[q] != INT_MAX && s_mem[e];
      skip[q] = !mem && nd[q] == 0;   // unchanged (or past the chunk)
      x[q] = (jj[q] != INT_MAX && !mem && nd[q] != 0) ? carry[jj[q]] : 0.f;
      present[q] = jj[q] != INT_MAX && !mem;
    }
#pragma unroll
    for (int q = 0; q < kFinPer; ++q) {
      const int e = tid + q * kThreads;
      acc[q] = present[q] ? x[q] : 0.f;
      for (int li = 0; li < x1 - x0; ++li)
        if ((nd[q] >> li) & 1) {
          const float v = svl[li][e];
          acc[q] = present[q] ? __fadd_rn(acc[q], v) : v;
          present[q] = true;
        }
    }
  } else if (late) {   // read, fold and write back each entry's carry together
#pragma unroll
    for (int q = 0; q < kFinPer; ++q) x[q] = jj[q] != INT_MAX ? carry[jj[q]] : 0.f;
#pragma unroll
    for (int q = 0; q < kFinPer; ++q) {
      const int e = tid + q * kThreads;
      present[q] = jj[q] != INT_MAX && !div_member(mag_key(x[q]), jj[q]);
      acc[q] = present[q] ? x[q] : 0.f;
      for (int li = 0; li < x1 - x0; ++li)
        if ((nd[q] >> li) & 1) {
          const float v = svl[li][e];
          acc[q] = present[q] ? __fadd_rn(acc[q], v) : v;
          present[q] = true;
        }
    }
  }
#pragma unroll
  for (int q = 0; q < kFinPer; ++q) {
    const int e = tid + q * kThreads;
    if (e < nloc && !skip[q]) {
      const float r = present[q] ? acc[q] : 0.f;
      SPARDL_BOUND(gi[e], t.n);
      carry[gi[e]] = r;
      if (t.aud_comb) {
        t.aud_comb[s_off + c0 + e] = x[q];
        t.aud_carry[s_off + c0 + e] = r;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// Deferred finalize records (see FinRecTask): one CTA per (task, 1024 global
// entries of block b).  The discard lists are joined with the CTA's indices
// exactly as in k_finalize, but nothing touches the carry: the records and
// the per-chunk record offsets are written in global-gradient order.
__global__ void __launch_bounds__(kThreads) k_fin_records(const FinRecTask* __restrict__ tasks,
                                                          int32_t* apply_flag) {
  pdl_enter();
  const FinRecTask& t = tasks[blockIdx.y];
  peer_wait(t.ps);
  const int gn = *t.g_cnt;
  const int tid = threadIdx.x;
  if (blockIdx.x == 0 && blockIdx.y == 0 && tid == 0) *apply_flag = 1;
  if (blockIdx.x == 0 && tid == 0) *t.rec_n = gn;
  const int c0 = blockIdx.x * kFinChunk;
  auto chunk_of = [&](int32_t j) { return (int)(((int64_t)j - t.origin) / kChunk); };
  if (gn == 0) {
    if (blockIdx.x == 0)
      for (int c = tid; c <= t.nchunks; c += kThreads) t.chunk_off[c] = 0;
    return;
  }
  if (c0 >= gn) return;
  const int nloc = min(kFinChunk, gn - c0);
  __shared__ int32_t gi[kFinChunk];
  __shared__ float sv[2][kFinChunk];
  __shared__ int range[4];
  for (int e = tid; e < kFinChunk; e += kThreads) {
    gi[e] = e < nloc ? t.g_idx[c0 + e] : INT_MAX;
    sv[0][e] = __uint_as_float(kNoRec);
    sv[1][e] = __uint_as_float(kNoRec);
  }
  __syncthreads();
  const int32_t jlo = gi[0], jhi = gi[nloc - 1];
  {   // each list's sub-range inside [jlo, jhi] (warps 0-3: lower/upper bounds)
    const int warp = tid >> 5, li = warp >> 1;
    if (li < t.nxl) {
      const XiList X = t.xl[li];
      const bool upper = warp & 1;
      const int r = warp_bound(X.idx, *X.cnt, upper ? jhi : jlo, upper);
      if ((tid & 31) == 0) range[warp] = r;
    }
  }
  __syncthreads();
  for (int li = 0; li < t.nxl; ++li) {
    const XiList X = t.xl[li];
    const int r0 = range[2 * li], r1 = range[2 * li + 1];
    for (int p = r0 + tid; p < r1; p += kThreads) {
      const int32_t x = X.idx[p];
      const int ps = lower_bound_i32(gi, nloc, x);
      if (ps < nloc && gi[ps] == x) sv[li][ps] = X.val[p];
    }
  }
  __syncthreads();
  for (int e = tid; e < nloc; e += kThreads) {
    const int i = c0 + e;
    const int32_t j = gi[e];
    t.rec_idx[i] = j;
    t.rec_v1[i] = sv[0][e];
    t.rec_v2[i] = sv[1][e];
    // chunk offsets: the chunks between the previous record's and this one's
    const int cj = chunk_of(j);
    const int cp = i == 0 ? -1 : chunk_of(e > 0 ? gi[e - 1] : t.g_idx[i - 1]);
    for (int c = cp + 1; c <= cj; ++c) t.chunk_off[c] = i;
    if (i == gn - 1)
      for (int c = cj + 1; c <= t.nchunks; ++c) t.chunk_off[c] = gn;
  }
}

// The pending records applied to the carry in place (a reader of the carry
// between iterations); the caller clears the apply flag afterwards.
__global__ void __launch_bounds__(kThreads) k_fin_apply(const FinRecTask* __restrict__ tasks,
                                                        const int32_t* apply_flag) {
  pdl_enter();
  if (!*apply_flag) return;
  const FinRecTask& t = tasks[blockIdx.y];
  const int n = *t.rec_n;
  const SelScratch* dsc = t.div_sc;
  for (int i = blockIdx.x * kFinChunk + threadIdx.x; i < min(n, (int)(blockIdx.x + 1) * kFinChunk);
       i += kThreads) {
    const int32_t j = t.rec_idx[i];
    const float x = t.carry[j];
    const bool keep = !sel_member(dsc, mag_key(x), j);
    t.carry[j] = fin_fold(x, keep, t.rec_v1[i], t.rec_v2[i]);
  }
}

__global__ void __launch_bounds__(kThreads)
    k_finalize_lres(const FinalizeTask* __restrict__ tasks, const int32_t* abort) {
  pdl_enter();
  if (err_set(abort)) return;
  const FinalizeTask& t = tasks[blockIdx.y];
  if (t.mode != 2) return;
  for (int b = 0; b < t.m; ++b) {
    const GatherSrc d = t.div[b];
    const int dn = *d.cnt;
    for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < dn; e += gridDim.x * blockDim.x)
      t.carry[d.idx[e]] = 0.f;
  }
}

// ---------------------------------------------------------------------------
__global__ void k_ledger(const LedgerAdd* __restrict__ adds, int n, const int32_t* abort) {
  pdl_enter();
  if (err_set(abort)) return;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const long long v = 2ll * (long long)(*adds[i].cnt);
    if (v) atomicAdd(reinterpret_cast<unsigned long long*>(adds[i].dst), (unsigned long long)v);
  }
}

// ---------------------------------------------------------------------------
// Algorithm 2 (inc/sag.hpp:61-81) in double precision, llround semantics
// (round half away from zero) via CUDA's llround.
__global__ void k_controller(const CtlTask* __restrict__ tasks, int n, int observe,
                             const int32_t* abort) {
  pdl_enter();
  if (err_set(abort)) return;
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  HCtl c = *tasks[i].ctl;
  if (observe) {
    const long long nt = *tasks[i].n_t;
    const bool over = nt > c.target;
    const bool rising = c.step > 0.0;
    if (over != rising) {
      if (c.flag) {
        c.step *= 2.0;
        c.flag = 0;
      } else {
        c.flag = 1;
      }
    } else {
      c.step = -c.step / 2.0;
      c.flag = 0;
    }
    double v = __dadd_rn(c.h, c.step);
    if (v < c.lower) v = c.lower;
    else if (c.upper < v) v = c.upper;
    c.h = v;
    *tasks[i].ctl = c;
  }
  const long long b = llround(c.h);
  *tasks[i].budget = b > 1 ? b : 1;
}

}  // namespace

int launch_assemble(const AssembleTask* tasks_dev, int ntask, int max_m, int64_t max_k,
                    cudaStream_t s) {
  if (ntask <= 0) return 0;
  int gx = (int)((max_k + kThreads - 1) / kThreads);
  gx = gx < 1 ? 1 : (gx > 1184 ? 1184 : gx);
  const size_t smem = sizeof(int) * (static_cast<size_t>(max_m) + 1);
  if (smem > 48 * 1024) {
    static bool configured[kMaxDevices] = {};
    const int dev = cur_device();
    if (!configured[dev]) {
      cudaFuncSetAttribute(k_assemble, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
      configured[dev] = true;
    }
  }
  launch_pdl(k_assemble, dim3(gx, ntask), dim3(kThreads), smem, s, tasks_dev);
  return 1;
}

int launch_finalize(const FinalizeTask* tasks_dev, int ntask, int64_t max_blk, int m,
                    int max_div, const int32_t* abort, cudaStream_t s) {
  if (ntask <= 0) return 0;
  int gx = (int)((max_blk + kFinChunk - 1) / kFinChunk);
  gx = gx < 1 ? 1 : gx;
  launch_pdl(k_finalize, dim3(gx, m, ntask), dim3(kThreads), 0, s, tasks_dev, abort);
  if (max_div > 0) {
    int lx = (max_div + kThreads - 1) / kThreads;
    lx = lx < 1 ? 1 : (lx > 1184 ? 1184 : lx);
    launch_pdl(k_finalize_lres, dim3(lx, ntask), dim3(kThreads), 0, s, tasks_dev, abort);
    return 2;
  }
  return 1;
}

int launch_fin_records(const FinRecTask* tasks_dev, int ntask, int64_t max_blk,
                       int32_t* apply_flag, cudaStream_t s) {
  if (ntask <= 0) return 0;
  const int gx = (int)std::max<int64_t>(1, (max_blk + kFinChunk - 1) / kFinChunk);
  launch_pdl(k_fin_records, dim3(gx, ntask), dim3(kThreads), 0, s, tasks_dev, apply_flag);
  return 1;
}

int launch_fin_apply(const FinRecTask* tasks_dev, int ntask, int64_t max_blk,
                     int32_t* apply_flag, cudaStream_t s) {
  if (ntask <= 0) return 0;
  const int gx = (int)std::max<int64_t>(1, (max_blk + kFinChunk - 1) / kFinChunk);
  launch_pdl(k_fin_apply, dim3(gx, ntask), dim3(kThreads), 0, s, tasks_dev,
             static_cast<const int32_t*>(apply_flag));
  return 1;
}

int launch_ledger(const LedgerAdd* adds_dev, int nadd, const int32_t* abort, cudaStream_t s) {
  if (nadd <= 0) return 0;
  const int gx = (nadd + kThreads - 1) / kThreads;
  launch_pdl(k_ledger, dim3(gx), dim3(kThreads), 0, s, adds_dev, nadd, abort);
  return 1;
}

int launch_controller(const CtlTask* tasks_dev, int ntask, int observe, const int32_t* abort,
                      cudaStream_t s) {
  if (ntask <= 0) return 0;
  launch_pdl(k_controller, dim3((ntask + 127) / 128), dim3(128), 0, s, tasks_dev, ntask, observe,
             abort);
  return 1;
}

}  // namespace sdl
