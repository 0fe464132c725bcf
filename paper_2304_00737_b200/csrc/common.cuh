// Small device helpers shared by the kernels.
#pragma once

#include <cstdio>
#include <cstdlib>

#include <cuda_runtime.h>
#include <stdint.h>

#include "kernels.cuh"

namespace sdl {

// Device bounds assertions (the sanitizer stand-in: compute-sanitizer is
// closed on the GPU pool).  Compiled in with make EXTRA=-DSPARDL_CHECKED=1:
// a violated bound prints the site and traps (the launch fails loudly).
#ifndef SPARDL_CHECKED
#define SPARDL_CHECKED 0
#endif
#if SPARDL_CHECKED
#define SPARDL_BOUND(i, n)                                                                  \
  do {                                                                                      \
    const long long i_ = (long long)(i), n_ = (long long)(n);                               \
    if (i_ < 0 || i_ >= n_) {                                                               \
      printf("SPARDL_BOUND %s:%d: %s = %lld outside [0, %s = %lld)\n", __FILE__, __LINE__,  \
             #i, i_, #n, n_);                                                               \
      __trap();                                                                             \
    }                                                                                       \
  } while (0)
#else
#define SPARDL_BOUND(i, n) \
  do {                     \
  } while (0)
#endif
// (a capacity of 0 means "not recorded": unchecked)
#define SPARDL_BOUND_CAP(i, cap) \
  do {                           \
    if ((cap) > 0) SPARDL_BOUND(i, cap); \
  } while (0)

// Magnitude key: |v| ordering == unsigned ordering of the low 31 bits for
// every non-NaN float; +0 and -0 share key 0 (inc/sparse.hpp:122-127 compares
// fabs values, so they tie and the smaller index wins).
__device__ __forceinline__ uint32_t mag_key(float v) {
  return __float_as_uint(v) & 0x7fffffffu;
}

__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// Exclusive prefix count of a predicate over the whole CTA (blockDim.x a
// multiple of 32, <= 1024).  `scratch` holds >= 33 ints.  Returns the
// exclusive rank of this thread; *total receives the CTA-wide count.
__device__ __forceinline__ int block_rank(bool pred, int* scratch, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  const uint32_t b = __ballot_sync(0xffffffffu, pred);
  const int in_warp = __popc(b & lanemask_lt());
  if (lane == 0) scratch[warp] = __popc(b);
  __syncthreads();
  if (threadIdx.x < 32) {
    int v = threadIdx.x < nwarps ? scratch[threadIdx.x] : 0;
    int inc = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int n = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += n;
    }
    if (threadIdx.x < nwarps) scratch[threadIdx.x] = inc - v;
    if (threadIdx.x == 31) scratch[32] = inc;
  }
  __syncthreads();
  const int r = scratch[warp] + in_warp;
  *total = scratch[32];
  __syncthreads();
  return r;
}

// CTA sums of three long longs (two barriers); scratch holds 3 * 32.
__device__ __forceinline__ void block_sum3_ll(long long& a, long long& b, long long& c,
                                              long long* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    a += __shfl_down_sync(0xffffffffu, a, o);
    b += __shfl_down_sync(0xffffffffu, b, o);
    c += __shfl_down_sync(0xffffffffu, c, o);
  }
  if (lane == 0) {
    scratch[3 * warp] = a;
    scratch[3 * warp + 1] = b;
    scratch[3 * warp + 2] = c;
  }
  __syncthreads();
  a = b = c = 0;
  for (int w = 0; w < nwarps; ++w) {
    a += scratch[3 * w];
    b += scratch[3 * w + 1];
    c += scratch[3 * w + 2];
  }
  __syncthreads();
}

// Exclusive prefix sums of three ints over the CTA in one pass (two
// barriers); scratch holds 3 * 33 ints.  e* = exclusive prefix, t* = total.
__device__ __forceinline__ void block_exscan3(int a, int b, int c, int* scratch, int& ea, int& eb,
                                              int& ec, int& ta, int& tb, int& tc) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  int ia = a, ib = b, ic = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int na = __shfl_up_sync(0xffffffffu, ia, o);
    const int nb = __shfl_up_sync(0xffffffffu, ib, o);
    const int nc = __shfl_up_sync(0xffffffffu, ic, o);
    if (lane >= o) {
      ia += na;
      ib += nb;
      ic += nc;
    }
  }
  if (lane == 31) {
    scratch[warp] = ia;
    scratch[33 + warp] = ib;
    scratch[66 + warp] = ic;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    const bool in = threadIdx.x < nwarps;
    int wa = in ? scratch[threadIdx.x] : 0, wb = in ? scratch[33 + threadIdx.x] : 0,
        wc = in ? scratch[66 + threadIdx.x] : 0;
    int xa = wa, xb = wb, xc = wc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int na = __shfl_up_sync(0xffffffffu, xa, o);
      const int nb = __shfl_up_sync(0xffffffffu, xb, o);
      const int nc = __shfl_up_sync(0xffffffffu, xc, o);
      if (lane >= o) {
        xa += na;
        xb += nb;
        xc += nc;
      }
    }
    __syncwarp();
    if (in) {
      scratch[threadIdx.x] = xa - wa;
      scratch[33 + threadIdx.x] = xb - wb;
      scratch[66 + threadIdx.x] = xc - wc;
    }
    if (threadIdx.x == 31) {
      scratch[32] = xa;
      scratch[65] = xb;
      scratch[98] = xc;
    }
  }
  __syncthreads();
  ea = scratch[warp] + ia - a;
  eb = scratch[33 + warp] + ib - b;
  ec = scratch[66 + warp] + ic - c;
  ta = scratch[32];
  tb = scratch[65];
  tc = scratch[98];
  __syncthreads();
}

// Exclusive prefix sum of an int over the CTA.
__device__ __forceinline__ int block_exscan(int v, int* scratch, int* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
  int inc = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int n = __shfl_up_sync(0xffffffffu, inc, o);
    if (lane >= o) inc += n;
  }
  if (lane == 31) scratch[warp] = inc;
  __syncthreads();
  if (threadIdx.x < 32) {
    int w = threadIdx.x < nwarps ? scratch[threadIdx.x] : 0;
    int winc = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int n = __shfl_up_sync(0xffffffffu, winc, o);
      if (lane >= o) winc += n;
    }
    if (threadIdx.x < nwarps) scratch[threadIdx.x] = winc - w;
    if (threadIdx.x == 31) scratch[32] = winc;
  }
  __syncthreads();
  const int r = scratch[warp] + inc - v;
  *total = scratch[32];
  __syncthreads();
  return r;
}

__device__ __forceinline__ long long block_sum_ll(long long v, long long* scratch) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int nwarps = blockDim.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  if (lane == 0) scratch[warp] = v;
  __syncthreads();
  long long t = 0;
  if (threadIdx.x == 0)
    for (int w = 0; w < nwarps; ++w) t += scratch[w];
  __syncthreads();
  if (threadIdx.x == 0) scratch[0] = t;
  __syncthreads();
  t = scratch[0];
  __syncthreads();
  return t;
}

#ifndef SPARDL_DIV_EXTRAP
#define SPARDL_DIV_EXTRAP 0.75
#endif
#ifndef SPARDL_DIV_TARGET
#define SPARDL_DIV_TARGET 1.15
#endif
// Dividing select epilogue: the pre-threshold of the next iteration.
__device__ inline void update_history(DivHistory* h, int mode, int all, uint32_t T, uint32_t pre,
                               long long cand, long long budget) {
  constexpr uint32_t kMinDelta = 1u << 12, kMaxDelta = 1u << 26;
  constexpr double kTarget = SPARDL_DIV_TARGET;   // wanted candidates / L
  if (mode != 0 || all != 0 || budget <= 0) {   // dense fallback (or trivial): sample again
    if (h->valid) h->delta = h->delta < kMaxDelta / 2 ? h->delta * 2 : kMaxDelta;
    h->valid = 0;
    h->has_T = all == 0 && budget > 0;
    h->last_T = T;
    return;
  }
  // secant in (key, log count): count(pre) = cand, count(T) = budget
  const double span = (double)(T - pre);
  const double ratio = (double)cand / (double)budget;
  double d;
  if (ratio > 1.02 && span > 0) d = span * log(kTarget) / log(ratio);
  else d = 2.0 * (span > 0 ? span : (double)kMinDelta);
  if (h->valid) {   // at most x2 / x0.5 per run
    const double old = (double)h->delta;
    d = d > 2 * old ? 2 * old : (d < old / 2 ? old / 2 : d);
  }
  d = d < kMinDelta ? kMinDelta : (d > kMaxDelta ? kMaxDelta : d);
  // a threshold that grows from run to run (residual accumulation) is
  // extrapolated in magnitude, by a fraction of the last growth: with fresh
  // gradients every run T also fluctuates, and a full linear step would
  // overshoot after every upward fluctuation (fewer than L candidates: the
  // dense fallback)
  const float tv = __uint_as_float(T), tp = __uint_as_float(h->last_T);
  const float grown = h->has_T && tv > tp ? tv + (float)SPARDL_DIV_EXTRAP * (tv - tp) : tv;
  const uint32_t Tn = grown < 3.0e38f ? __float_as_uint(grown) : T;
  long long next = (long long)Tn - (long long)d;
  h->delta = (uint32_t)d;
  h->next_pre = next < 0 ? 0u : (uint32_t)next;
  // the first threshold after a (re)start only seeds the trend: trust the
  // carried pre-threshold from the second sampled run on
  h->valid = h->has_T;
  h->last_T = T;
  h->has_T = 1;
}


// Residual finalize of one global index (inc/residual.hpp:128-150, gres):
// xi(j) starts as combined[j] = x when the dividing select discarded j
// (keep), then folds the in-procedure discards in recording order; no
// contribution at all -> +0.  Used by k_finalize's deferred form (records
// applied in the next candidate pass or by k_fin_apply).
__device__ __forceinline__ float fin_fold(float x, bool keep, float v1, float v2) {
  bool has = keep;
  float acc = keep ? x : 0.f;
  if (__float_as_uint(v1) != kNoRec) {
    acc = has ? __fadd_rn(acc, v1) : v1;
    has = true;
  }
  if (__float_as_uint(v2) != kNoRec) {
    acc = has ? __fadd_rn(acc, v2) : v2;
    has = true;
  }
  return has ? acc : 0.f;
}

// lower_bound over a sorted int array [a, a+n)
__device__ __forceinline__ int lower_bound_i32(const int32_t* a, int n, int32_t x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] < x) lo = mid + 1; else hi = mid;
  }
  return lo;
}
__device__ __forceinline__ int upper_bound_i32(const int32_t* a, int n, int32_t x) {
  int lo = 0, hi = n;
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (a[mid] <= x) lo = mid + 1; else hi = mid;
  }
  return lo;
}


// ---------------------------------------------------------------------------
// Programmatic dependent launch.  Every kernel of the path is launched with
// programmatic stream serialization (launch_pdl) and waits for its
// predecessor's completion and memory at pdl_enter() (griddepcontrol.wait;
// a no-op without the attribute).  Measured on B200: it shortens the
// non-graph path (launch latency overlaps the predecessor's tail) and is
// neutral inside the CUDA graph; triggering dependents early
// (SPARDL_PDL_TRIGGER=1) lets waiting CTAs take SM slots from the running
// kernel and costs ~1 % per step, so the trigger is implicit (CTA exit).
// SPARDL_PDL=0 disables the attribute.
#ifndef SPARDL_PDL_TRIGGER
#define SPARDL_PDL_TRIGGER 0
#endif
__device__ __forceinline__ void pdl_enter() {
  asm volatile("griddepcontrol.wait;" ::: "memory");
#if SPARDL_PDL_TRIGGER
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
#endif
}

inline bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("SPARDL_PDL");
    on = (e && e[0] == '0') ? 0 : 1;
  }
  return on == 1;
}

// Kernel attributes (dynamic shared memory opt-in, cluster permissions) are
// per device: the launchers cache them per current device.
constexpr int kMaxDevices = 64;
inline int cur_device() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess) d = 0;
  return d < 0 ? 0 : (d >= kMaxDevices ? kMaxDevices - 1 : d);
}

template <typename... KArgs, typename... Args>
inline cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                              cudaStream_t s, Args... args) {
  cudaLaunchConfig_t lc{};
  lc.gridDim = grid;
  lc.blockDim = block;
  lc.dynamicSmemBytes = smem;
  lc.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  lc.attrs = at;
  lc.numAttrs = pdl_enabled() ? 1 : 0;
  const cudaError_t e = cudaLaunchKernelEx(&lc, kernel, static_cast<KArgs>(args)...);
  note_launch(e);
  return e;
}


// ---------------------------------------------------------------------------
// Peer-transport flags (transport.cu): system-scope acquire/release on
// per-block readiness flags; bounded spins report through *err.

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ long long ld_acquire_sys(const long long* p) {
  long long v;
  asm volatile("ld.acquire.sys.global.b64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_release_sys(long long* p, long long v) {
  asm volatile("st.release.sys.global.b64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// Spins until *flag >= target.  Gives up after `timeout_ns`, or as soon as
// another waiter of this GPU has given up (*err set): the iteration then
// drains quickly on stale (but in-bounds: every count ever stored is within
// its buffer's capacity) data, the writers of persistent state skip their
// stores (err_set), and the host poisons the context at the next sync().
__device__ __forceinline__ bool err_set(const int32_t* err) {
  return err && *reinterpret_cast<const volatile int32_t*>(err) != 0;
}

__device__ inline bool spin_until(const long long* flag, long long target, int32_t* err,
                                  unsigned long long timeout_ns) {
  if (ld_acquire_sys(flag) >= target) return true;
  const unsigned long long t0 = gtime();
  unsigned ns = 32;
  while (ld_acquire_sys(flag) < target) {
    __nanosleep(ns);
    if (ns < 1024) ns <<= 1;
    if (err_set(err)) return false;
    if (gtime() - t0 > timeout_ns) {
      atomicExch(err, 1);
      return false;
    }
  }
  return true;
}

// a whole CTA: wait until the task's remote inputs are published
__device__ inline void peer_wait(const PeerSync& ps) {
  if (ps.nwait <= 0) return;   // uniform per task
  const long long e = *ps.epoch;
  for (int i = threadIdx.x; i < ps.nwait; i += blockDim.x)
    spin_until(ps.wait[i], e, ps.err, ps.timeout_ns);
  __syncthreads();
}

// one thread, after the task's output is complete: publish it to its consumers
__device__ inline void peer_publish(const PeerSync& ps) {
  if (ps.npub <= 0) return;
  const long long e = *ps.epoch;
  __threadfence_system();
  for (int i = 0; i < ps.npub; ++i) st_release_sys(ps.pub[i], e);
}

}  // namespace sdl
