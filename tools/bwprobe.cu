// Bandwidth probe for the dividing pass's access mix (2 reads : 1 write,
// in place).  Standalone: nvcc -gencode arch=compute_100a,code=sm_100a -O3
// tools/bwprobe.cu -o /tmp/bwprobe && /tmp/bwprobe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s\n", cudaGetErrorString(e)); return 1; } } while (0)

__global__ void k_copy(const float4* __restrict__ a, float4* __restrict__ b, int64_t n4) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x)
    b[i] = __ldcs(a + i);
}

__global__ void k_add_gs(const float4* __restrict__ g, float4* __restrict__ c, int64_t n4) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    float4 x = __ldcs(g + i), y = __ldcs(c + i);
    y.x += x.x; y.y += x.y; y.z += x.z; y.w += x.w;
    __stcs(c + i, y);
  }
}

template <int ITER, int TH>
__global__ void __launch_bounds__(TH) k_add_chunk(const float4* __restrict__ g, float4* __restrict__ c, int64_t n4) {
  const int64_t base = (int64_t)blockIdx.x * ITER * TH;
  float4 x[ITER], y[ITER];
#pragma unroll
  for (int it = 0; it < ITER; ++it) {
    const int64_t i = base + it * TH + threadIdx.x;
    if (i < n4) { x[it] = __ldcs(g + i); y[it] = __ldcs(c + i); }
  }
#pragma unroll
  for (int it = 0; it < ITER; ++it) {
    const int64_t i = base + it * TH + threadIdx.x;
    if (i < n4) {
      y[it].x += x[it].x; y[it].y += x[it].y; y[it].z += x[it].z; y[it].w += x[it].w;
      __stcs(c + i, y[it]);
    }
  }
}

// TMA-bulk persistent pipeline: each CTA streams tiles of g and c into
// shared memory with cp.async.bulk, S stages deep, adds, stores from smem
// with cp.async.bulk (smem -> global).
template <int S, int TILE>
__global__ void __launch_bounds__(256) k_add_bulk(const float* __restrict__ g, float* __restrict__ c, int64_t ntiles) {
  extern __shared__ __align__(128) unsigned char sm[];
  float* bg = reinterpret_cast<float*>(sm);
  float* bc = bg + S * TILE;
  __shared__ __align__(8) unsigned long long bar[S];
  const int nct = gridDim.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < S; ++s)
      asm volatile("mbarrier.init.shared.b64 [%0], 1;" :: "r"((unsigned)__cvta_generic_to_shared(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  __syncthreads();
  auto issue = [&](int64_t tile, int s) {
    const unsigned b = (unsigned)__cvta_generic_to_shared(&bar[s]);
    const unsigned bytes = TILE * 4;
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" :: "r"(b), "r"(2 * bytes));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"((unsigned)__cvta_generic_to_shared(bg + s * TILE)), "l"(g + tile * TILE), "r"(bytes), "r"(b) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 :: "r"((unsigned)__cvta_generic_to_shared(bc + s * TILE)), "l"(c + tile * TILE), "r"(bytes), "r"(b) : "memory");
  };
  int64_t my = (ntiles - blockIdx.x + nct - 1) / nct;
  if (threadIdx.x == 0)
    for (int s = 0; s < S && s < my; ++s) issue(blockIdx.x + (int64_t)s * nct, s);
  for (int64_t j = 0; j < my; ++j) {
    const int s = j % S;
    const unsigned ph = (j / S) & 1;
    const unsigned b = (unsigned)__cvta_generic_to_shared(&bar[s]);
    asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W;\n}" :: "r"(b), "r"(ph) : "memory");
    const int64_t tile = blockIdx.x + j * nct;
    float4* xg = reinterpret_cast<float4*>(bg + s * TILE);
    float4* xc = reinterpret_cast<float4*>(bc + s * TILE);
    float4* out = reinterpret_cast<float4*>(c + tile * TILE);
    for (int q = threadIdx.x; q < TILE / 4; q += 256) {
      float4 x = xg[q], y = xc[q];
      y.x += x.x; y.y += x.y; y.z += x.z; y.w += x.w;
      __stcs(out + q, y);
    }
    __syncthreads();
    if (threadIdx.x == 0 && j + S < my) issue(tile + (int64_t)S * nct, s);
  }
}

int main() {
  const int64_t n = 204800000;  // 8 x 25.6M floats
  float *a, *b;
  CK(cudaMalloc(&a, n * 4));
  CK(cudaMalloc(&b, n * 4));
  cudaMemset(a, 0, n * 4);
  cudaMemset(b, 0, n * 4);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int nsm = 0;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
  auto timeit = [&](const char* name, double bytes, auto fn) {
    float best = 1e9;
    for (int r = 0; r < 12; ++r) {
      cudaEventRecord(e0);
      fn();
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (r >= 2 && ms < best) best = ms;
    }
    printf("%-28s %8.1f us  %7.1f GB/s  (%s)\n", name, best * 1e3, bytes / (best * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
  };
  const int64_t n4 = n / 4;
  timeit("copy gs 148x8x256", 8.0 * n, [&] { k_copy<<<nsm * 8, 256>>>((const float4*)a, (float4*)b, n4); });
  timeit("copy gs 148x16x256", 8.0 * n, [&] { k_copy<<<nsm * 16, 256>>>((const float4*)a, (float4*)b, n4); });
  timeit("add gs 148x8x256", 12.0 * n, [&] { k_add_gs<<<nsm * 8, 256>>>((const float4*)a, (float4*)b, n4); });
  timeit("add gs 148x16x256", 12.0 * n, [&] { k_add_gs<<<nsm * 16, 256>>>((const float4*)a, (float4*)b, n4); });
  timeit("add chunk 8x256 (ours)", 12.0 * n, [&] { k_add_chunk<8, 256><<<(n4 + 2047) / 2048, 256>>>((const float4*)a, (float4*)b, n4); });
  timeit("add chunk 4x256", 12.0 * n, [&] { k_add_chunk<4, 256><<<(n4 + 1023) / 1024, 256>>>((const float4*)a, (float4*)b, n4); });
  timeit("add chunk 2x256", 12.0 * n, [&] { k_add_chunk<2, 256><<<(n4 + 511) / 512, 256>>>((const float4*)a, (float4*)b, n4); });
  timeit("add chunk 4x512", 12.0 * n, [&] { k_add_chunk<4, 512><<<(n4 + 2047) / 2048, 512>>>((const float4*)a, (float4*)b, n4); });
  {
    constexpr int S = 4, TILE = 8192;
    const int smem = 2 * S * TILE * 4;
    cudaFuncSetAttribute(k_add_bulk<S, TILE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    timeit("bulk S4 T8192 x148", 12.0 * n, [&] { k_add_bulk<S, TILE><<<nsm, 256, smem>>>(a, b, n / TILE); });
  }
  {
    constexpr int S = 3, TILE = 4096;
    const int smem = 2 * S * TILE * 4;
    cudaFuncSetAttribute(k_add_bulk<S, TILE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    timeit("bulk S3 T4096 x296", 12.0 * n, [&] { k_add_bulk<S, TILE><<<nsm * 2, 256, smem>>>(a, b, n / TILE); });
  }
  {
    constexpr int S = 6, TILE = 4096;
    const int smem = 2 * S * TILE * 4;
    cudaFuncSetAttribute(k_add_bulk<S, TILE>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    timeit("bulk S6 T4096 x148", 12.0 * n, [&] { k_add_bulk<S, TILE><<<nsm, 256, smem>>>(a, b, n / TILE); });
  }
  return 0;
}
