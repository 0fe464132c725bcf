// The fp64 component kernels of the C++ drop-in surface (include/spardl/).
//
// The reference's component API computes in double (inc/sparse.hpp:27-75):
// top_k_select on |value| (a double compare, ties by the smaller index,
// inc/sparse.hpp:122-162) and merge_add summing coinciding indices as
// a.value + b.value (inc/sparse.hpp:182-208).  The all-reduce pipeline runs
// in fp32 (the north star's value type); these one-shot components keep the
// reference's double semantics exactly, so its own unit tests
// (tests/test_sparse.cpp) hold unmodified.  They are small-call paths: one
// CTA selects, two kernels merge.
#include <cstdint>

#include "common.cuh"
#include "kernels.cuh"

namespace sdl {

namespace {

constexpr int kT64 = 1024;

__device__ __forceinline__ unsigned long long mag64(double v) {
  return static_cast<unsigned long long>(__double_as_longlong(v)) & 0x7fffffffffffffffull;
}

// The rank-`need` digit (8 bits at `shift`) among the values x of entries
// passing `in`, counting from the largest digit down; whole CTA.
template <class GetX, class In>
__device__ int digit_select(int n, int shift, long long& need, GetX getx, In in, uint32_t* h,
                            int* scratch) {
  __shared__ int s_d;
  __shared__ long long s_need;
  if (threadIdx.x < 256) h[threadIdx.x] = 0;
  __syncthreads();
  for (int i = threadIdx.x; i < n; i += kT64)
    if (in(i)) atomicAdd(&h[(getx(i) >> shift) & 255ull], 1u);
  __syncthreads();
  const int dgt = 255 - (int)threadIdx.x;
  const int cnt = threadIdx.x < 256 ? (int)h[dgt] : 0;
  int tot = 0;
  const int ex = block_exscan(cnt, scratch, &tot);
  if (threadIdx.x < 256 && ex < need && need <= ex + cnt) {
    s_d = dgt;
    s_need = need - ex;
  }
  __syncthreads();
  const int d = s_d;
  need = s_need;
  __syncthreads();
  return d;
}

// top_k_select in double: flag[i] = 1 for the min(budget, n) entries first
// in (|v| desc, index asc).  One CTA: radix select of the threshold
// magnitude T, then of the cut index among |v| == T.
__global__ void __launch_bounds__(kT64) k_topk64(const int64_t* __restrict__ idx,
                                                 const double* __restrict__ val, int n,
                                                 long long budget, uint8_t* __restrict__ flag) {
  __shared__ uint32_t h[256];
  __shared__ int scratch[40];
  if (budget >= n || budget <= 0) {
    for (int i = threadIdx.x; i < n; i += kT64) flag[i] = budget > 0 ? 1 : 0;
    return;
  }
  // magnitude threshold: 8 digits of the 63-bit magnitude
  long long need = budget;
  unsigned long long T = 0, mask = 0;
  for (int shift = 56; shift >= 0; shift -= 8) {
    const unsigned long long m0 = mask, t0 = T;
    const int d = digit_select(
        n, shift, need, [&](int i) { return mag64(val[i]); },
        [&](int i) { return (mag64(val[i]) & m0) == t0; }, h, scratch);
    T |= static_cast<unsigned long long>(d) << shift;
    mask |= 255ull << shift;
  }
  // `need` entries of magnitude T are kept: the smallest indices among them
  // (the reference's tie rule) -- radix select on the bias-free index
  // ascending: select the need-th largest of ~index
  unsigned long long C = 0, cmask = 0;
  for (int shift = 56; shift >= 0; shift -= 8) {
    const unsigned long long m0 = cmask, c0 = C;
    const int d = digit_select(
        n, shift, need, [&](int i) { return ~static_cast<unsigned long long>(idx[i]); },
        [&](int i) {
          return mag64(val[i]) == T && (~static_cast<unsigned long long>(idx[i]) & m0) == c0;
        },
        h, scratch);
    C |= static_cast<unsigned long long>(d) << shift;
    cmask |= 255ull << shift;
  }
  const long long cut = static_cast<long long>(~C);   // largest kept index among |v| == T
  for (int i = threadIdx.x; i < n; i += kT64) {
    const unsigned long long k = mag64(val[i]);
    flag[i] = (k > T || (k == T && idx[i] <= cut)) ? 1 : 0;
  }
}

// merge_add in double, step 1: every entry's position in the stable merge
// (a before b at equal indices) -- an index present in both lists takes two
// adjacent positions, a's first.
__global__ void k_merge64_rank(const int64_t* __restrict__ ai, const double* __restrict__ av,
                               int na, const int64_t* __restrict__ bi,
                               const double* __restrict__ bv, int nb, int64_t* __restrict__ ti,
                               double* __restrict__ tv) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < na) {
    const int64_t x = ai[e];
    int lo = 0, hi = nb;   // lower_bound in b
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (bi[mid] < x) lo = mid + 1;
      else hi = mid;
    }
    ti[e + lo] = x;
    tv[e + lo] = av[e];
  } else if (e < na + nb) {
    const int j = e - na;
    const int64_t x = bi[j];
    int lo = 0, hi = na;   // upper_bound in a
    while (lo < hi) {
      const int mid = (lo + hi) >> 1;
      if (ai[mid] <= x) lo = mid + 1;
      else hi = mid;
    }
    ti[j + lo] = x;
    tv[j + lo] = bv[j];
  }
}

// step 2 (one CTA): fold each adjacent pair of equal indices (a + b) and
// compact in order.
__global__ void __launch_bounds__(kT64) k_merge64_fold(const int64_t* __restrict__ ti,
                                                       const double* __restrict__ tv, int n,
                                                       int64_t* __restrict__ oi,
                                                       double* __restrict__ ov,
                                                       int64_t* __restrict__ no) {
  __shared__ int scratch[40];
  int carry = 0;
  for (int k0 = 0; k0 < n; k0 += kT64) {
    const int k = k0 + threadIdx.x;
    const bool head = k < n && (k == 0 || ti[k] != ti[k - 1]);
    int tot = 0;
    const int r = carry + block_rank(head, scratch, &tot);
    if (head) {
      double v = tv[k];
      if (k + 1 < n && ti[k + 1] == ti[k]) v = v + tv[k + 1];   // a.value + b.value
      oi[r] = ti[k];
      ov[r] = v;
    }
    carry += tot;
  }
  if (threadIdx.x == 0) *no = carry;
}

}  // namespace

int launch_topk64(const int64_t* idx, const double* val, int n, long long budget, uint8_t* flag,
                  cudaStream_t s) {
  if (n <= 0) return 0;
  k_topk64<<<1, kT64, 0, s>>>(idx, val, n, budget, flag);
  note_launch(cudaGetLastError());
  return 1;
}

int launch_merge64(const int64_t* ai, const double* av, int na, const int64_t* bi,
                   const double* bv, int nb, int64_t* ti, double* tv, int64_t* oi, double* ov,
                   int64_t* no, cudaStream_t s) {
  const int n = na + nb;
  if (n > 0)
    k_merge64_rank<<<(n + 255) / 256, 256, 0, s>>>(ai, av, na, bi, bv, nb, ti, tv);
  k_merge64_fold<<<1, kT64, 0, s>>>(ti, tv, n, oi, ov, no);
  note_launch(cudaGetLastError());
  return 2;
}

}  // namespace sdl
