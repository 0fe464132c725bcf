// Global-gradient assembly, residual finalize, ledger and the B-SAG
// controller on the device.
#include "common.cuh"
#include "kernels.cuh"

namespace sdl {

namespace {

// ---------------------------------------------------------------------------
// Assembly: the global gradient is the concatenation of the m reserved
// blocks in position order (inc/pipeline.hpp:279-291); blocks cover
// increasing index ranges, so the result is index-sorted.
__global__ void __launch_bounds__(kThreads) k_assemble(const AssembleTask* __restrict__ tasks) {
  const AssembleTask& t = tasks[blockIdx.y];
  __shared__ int off[65];
  if (threadIdx.x == 0) {
    int s = 0;
    for (int b = 0; b < t.m; ++b) {
      off[b] = s;
      s += *t.src[b].cnt;
    }
    off[t.m] = s;
    if (blockIdx.x == 0) *t.out_cnt = s;
  }
  __syncthreads();
  const int total = off[t.m];
  unsigned long long h = 0;
  for (int p = blockIdx.x * blockDim.x + threadIdx.x; p < total; p += gridDim.x * blockDim.x) {
    int b = 0;
    while (p >= off[b + 1]) ++b;
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
__device__ __forceinline__ int block_of_dev(int64_t n, int m, int64_t i) {
  const int64_t base = n / m, rem = n % m;
  const int64_t split = rem * (base + 1);
  if (i < split) return (int)(i / (base + 1));
  return (int)(rem + (i - split) / base);
}

__global__ void __launch_bounds__(kThreads) k_finalize(const FinalizeTask* __restrict__ tasks) {
  const FinalizeTask& t = tasks[blockIdx.y];
  if (t.mode == 2) return;   // lres ignores the global gradient
  const int gn = *t.g_cnt;
  for (int e = blockIdx.x * blockDim.x + threadIdx.x; e < gn; e += gridDim.x * blockDim.x) {
    const int32_t j = t.g_idx[e];
    if (t.mode == 1) {
      t.carry[j] = 0.f;
      continue;
    }
    const int b = block_of_dev(t.n, t.m, j);
    const GatherSrc d = t.div[b];
    const int dn = *d.cnt;
    const int p = lower_bound_i32(d.idx, dn, j);
    bool present = !(p < dn && d.idx[p] == j);
    float acc = present ? t.carry[j] : 0.f;
    for (int q = t.xi_off[b]; q < t.xi_off[b + 1]; ++q) {
      const XiList x = t.xi[q];
      const int xn = *x.cnt;
      const int r = lower_bound_i32(x.idx, xn, j);
      if (r < xn && x.idx[r] == j) {
        const float xv = x.val[r];
        acc = present ? __fadd_rn(acc, xv) : xv;
        present = true;
      }
    }
    t.carry[j] = present ? acc : 0.f;
  }
}

__global__ void __launch_bounds__(kThreads) k_finalize_lres(const FinalizeTask* __restrict__ tasks) {
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
__global__ void k_ledger(const LedgerAdd* __restrict__ adds, int n) {
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const long long v = 2ll * (long long)(*adds[i].cnt);
    if (v) atomicAdd(reinterpret_cast<unsigned long long*>(adds[i].dst), (unsigned long long)v);
  }
}

// ---------------------------------------------------------------------------
// Algorithm 2 (inc/sag.hpp:61-81) in double precision, llround semantics
// (round half away from zero) via CUDA's llround.
__global__ void k_controller(const CtlTask* __restrict__ tasks, int n, int observe) {
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
  (void)max_m;
  if (ntask <= 0) return 0;
  int gx = (int)((max_k + kThreads - 1) / kThreads);
  gx = gx < 1 ? 1 : (gx > 1184 ? 1184 : gx);
  k_assemble<<<dim3(gx, ntask), kThreads, 0, s>>>(tasks_dev);
  return 1;
}

int launch_finalize(const FinalizeTask* tasks_dev, int ntask, int64_t max_k, int max_div,
                    cudaStream_t s) {
  if (ntask <= 0) return 0;
  int gx = (int)((max_k + kThreads - 1) / kThreads);
  gx = gx < 1 ? 1 : (gx > 2368 ? 2368 : gx);
  k_finalize<<<dim3(gx, ntask), kThreads, 0, s>>>(tasks_dev);
  if (max_div > 0) {
    int lx = (max_div + kThreads - 1) / kThreads;
    lx = lx < 1 ? 1 : (lx > 1184 ? 1184 : lx);
    k_finalize_lres<<<dim3(lx, ntask), kThreads, 0, s>>>(tasks_dev);
    return 2;
  }
  return 1;
}

int launch_ledger(const LedgerAdd* adds_dev, int nadd, cudaStream_t s) {
  if (nadd <= 0) return 0;
  const int gx = (nadd + kThreads - 1) / kThreads;
  k_ledger<<<gx, kThreads, 0, s>>>(adds_dev, nadd);
  return 1;
}

int launch_controller(const CtlTask* tasks_dev, int ntask, int observe, cudaStream_t s) {
  if (ntask <= 0) return 0;
  k_controller<<<(ntask + 127) / 128, 128, 0, s>>>(tasks_dev, ntask, observe);
  return 1;
}

}  // namespace sdl
