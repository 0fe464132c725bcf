// r-way index merge with a left fold of the values in list order.
//
// Semantics: acc = l0; for t in 1..r-1: acc = merge_add(acc, l_t)
// (inc/sparse.hpp:182-208, applied as the reference applies it: SRS merges
// received blocks into the held block in arrival order,
// inc/reduce_scatter.hpp:190-202; B-SAG folds the gathered blocks in source
// rank order, inc/sag.hpp:231-236).  For an index present in several lists
// the value is ((v_a + v_b) + v_c) ... in list order -- every add is one
// IEEE round-to-nearest fp32 add (__fadd_rn, never contracted).
//
// Partitioning: every T-th entry of every list is a splitter.  Between two
// consecutive splitters each list contributes at most T entries, all inside
// one "window" of T consecutive entries of that list, so a CTA merges its
// partition from <= r windows staged in shared memory.  The partition output
// is written at the partition's position in concatenation space, so the
// result is a segmented list (one segment per partition, gaps where indices
// coincided) that the select kernels consume directly.
#include <climits>

#include "common.cuh"
#include "kernels.cuh"

namespace sdl {

namespace {

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  const size_t ga = __cvta_generic_to_global(gmem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(ga) : "memory");
}

// Rank all samples of a task; write the sorted splitters and, for each
// splitter, the window of every list that can hold its partition.
__global__ void __launch_bounds__(kThreads) k_merge_rank(const MergeTask* __restrict__ tasks) {
  pdl_enter();
  const MergeTask& t = tasks[blockIdx.y];
  peer_wait(t.ps);   // remote input lists published (k_merge_part follows in order)
  const int r = t.r, T = t.T;
  __shared__ int32_t samp[kMaxSamples];
  __shared__ int base[kMaxR + 1];
  if (threadIdx.x == 0) {
    int b = 0;
    for (int l = 0; l < r; ++l) {
      const int n = *t.in_cnt[l];
      base[l] = b;
      b += (n + T - 1) / T;
    }
    base[r] = b;
  }
  __syncthreads();
  const int S = base[r];
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    t.splitters[S] = INT_MAX;
    *t.nparts = S;
  }
  if ((int)(blockIdx.x * blockDim.x) >= S) return;
  for (int q = threadIdx.x; q < S; q += blockDim.x) {
    int l = 0;
    while (q >= base[l + 1]) ++l;
    samp[q] = t.in_idx[l][(q - base[l]) * T];
  }
  __syncthreads();
  for (int q = blockIdx.x * blockDim.x + threadIdx.x; q < S; q += gridDim.x * blockDim.x) {
    int l = 0;
    while (q >= base[l + 1]) ++l;
    const int j = q - base[l];
    const int32_t v = samp[q];
    int rank = j;
    int win[kMaxR];
    for (int u = 0; u < r; ++u) {
      if (u == l) {
        win[u] = j;
        continue;
      }
      const int32_t* a = samp + base[u];
      const int n = base[u + 1] - base[u];
      const int ub = upper_bound_i32(a, n, v);
      win[u] = ub - 1;
      rank += (u < l) ? ub : lower_bound_i32(a, n, v);
    }
    t.splitters[rank] = v;
    for (int u = 0; u < r; ++u) t.windows[(size_t)rank * r + u] = win[u];
  }
}

#ifndef SPARDL_MERGE_THREADS
#define SPARDL_MERGE_THREADS 256
#endif
constexpr int kMergeThreads = SPARDL_MERGE_THREADS;   // threads per partition CTA

__global__ void __launch_bounds__(kMergeThreads) k_merge_part(const MergeTask* __restrict__ tasks) {
  pdl_enter();
  // grid (task, partition): partitions of every task come first in launch
  // order, so the live ones (q < nparts, usually far fewer than max_parts)
  // all start in the first wave
  const MergeTask& t = tasks[blockIdx.x];
  const int q = blockIdx.y;
  const int S = *t.nparts;
  if (q >= t.max_parts) return;
  if (q >= S) {
    if (threadIdx.x == 0) {
      t.seg_off[q] = 0;
      t.seg_cnt[q] = 0;
    }
    return;
  }
  const int32_t v_lo = t.splitters[q];
  const int32_t v_hi = t.splitters[q + 1];
  if (v_lo == v_hi) {
    if (threadIdx.x == 0) {
      t.seg_off[q] = 0;
      t.seg_cnt[q] = 0;
    }
    return;
  }
  const int r = t.r, T = t.T;
  extern __shared__ __align__(16) unsigned char smem[];
  int32_t* w_idx = reinterpret_cast<int32_t*>(smem);          // [r*T]
  float* w_val = reinterpret_cast<float*>(w_idx + r * T);      // [r*T]
  int32_t* m_idx = reinterpret_cast<int32_t*>(w_val + r * T);  // [r*T]
  float* m_val = reinterpret_cast<float*>(m_idx + r * T);      // [r*T]
  __shared__ int wlen[kMaxR], wstart[kMaxR], a_[kMaxR], b_[kMaxR], sz_pref[kMaxR + 1];
  __shared__ int seg_base;
  __shared__ int scratch[40];
  if (threadIdx.x < r) {
    const int l = threadIdx.x;
    const int w = t.windows[(size_t)q * r + l];
    const int n = *t.in_cnt[l];
    if (w < 0) {
      wstart[l] = 0;
      wlen[l] = 0;
    } else {
      wstart[l] = w * T;
      const int rem = n - w * T;
      wlen[l] = rem < T ? rem : T;
    }
  }
  __syncthreads();
  // stage the windows with asynchronous 16-byte copies: every thread issues
  // all of its copies before waiting once (16-byte aligned windows: block
  // buffers are, and T % 4 == 0); the < 4-entry tail and unaligned lists
  // (component API inputs) are copied with plain loads
  for (int l = 0; l < r; ++l) {
    const int32_t* gi = t.in_idx[l] + wstart[l];
    const float* gv = t.in_val[l] + wstart[l];
    const bool al = ((reinterpret_cast<uintptr_t>(gi) | reinterpret_cast<uintptr_t>(gv)) & 15) == 0;
    const int n4 = al ? (wlen[l] >> 2) : 0;
    for (int j = threadIdx.x; j < n4; j += blockDim.x) {
      cp_async16(w_idx + l * T + 4 * j, gi + 4 * j);
      cp_async16(w_val + l * T + 4 * j, gv + 4 * j);
    }
    for (int j = 4 * n4 + threadIdx.x; j < wlen[l]; j += blockDim.x) {
      w_idx[l * T + j] = gi[j];
      w_val[l * T + j] = gv[j];
    }
  }
  asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();
  if (threadIdx.x < r) {
    const int l = threadIdx.x;
    a_[l] = lower_bound_i32(w_idx + l * T, wlen[l], v_lo);
    b_[l] = lower_bound_i32(w_idx + l * T, wlen[l], v_hi);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    int s = 0, base = 0;
    for (int l = 0; l < r; ++l) {
      sz_pref[l] = s;
      s += b_[l] - a_[l];
      base += wstart[l] + a_[l];
    }
    sz_pref[r] = s;
    seg_base = base;
  }
  __syncthreads();
  const int M = sz_pref[r];
  // stable r-way merge by (index, list): scatter every entry to its rank
  for (int e = threadIdx.x; e < M; e += blockDim.x) {
    int l = 0;
    while (e >= sz_pref[l + 1]) ++l;
    const int i = a_[l] + (e - sz_pref[l]);
    const int32_t x = w_idx[l * T + i];
    int pos = i - a_[l];
    for (int u = 0; u < r; ++u) {
      if (u == l) continue;
      const int32_t* a = w_idx + u * T + a_[u];
      const int n = b_[u] - a_[u];
      pos += (u < l) ? upper_bound_i32(a, n, x) : lower_bound_i32(a, n, x);
    }
    m_idx[pos] = x;
    m_val[pos] = w_val[l * T + i];
  }
  __syncthreads();
  // fold runs of equal index (at most r long, in list order) and compact
  int out = 0;
  for (int e0 = 0; e0 < M; e0 += blockDim.x) {
    const int e = e0 + threadIdx.x;
    const bool head = e < M && (e == 0 || m_idx[e] != m_idx[e - 1]);
    int tot;
    const int rk = out + block_rank(head, scratch, &tot);
    if (head) {
      const int32_t x = m_idx[e];
      float acc = m_val[e];
      for (int f = e + 1; f < M && m_idx[f] == x; ++f) acc = __fadd_rn(acc, m_val[f]);
      t.out_idx[seg_base + rk] = x;
      t.out_val[seg_base + rk] = acc;
    }
    out += tot;
  }
  if (threadIdx.x == 0) {
    t.seg_off[q] = seg_base;
    t.seg_cnt[q] = out;
  }
}

}  // namespace

int launch_merge(const MergeTask* tasks_dev, int ntask, int max_parts, int max_r_T,
                 cudaStream_t s) {
  if (ntask <= 0 || max_parts <= 0) return 0;
  const int rx = (max_parts + kThreads - 1) / kThreads;
  launch_pdl(k_merge_rank, dim3(rx, ntask), dim3(kThreads), 0, s, tasks_dev);
  const size_t smem = (size_t)max_r_T * 16;
  static size_t configured = 0;
  if (smem > 48 * 1024 && smem > configured) {
    cudaFuncSetAttribute(k_merge_part, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)smem);
    configured = smem;
  }
  launch_pdl(k_merge_part, dim3(ntask, max_parts), dim3(kMergeThreads), smem, s, tasks_dev);
  return 2;
}

}  // namespace sdl
