// extern "C" boundary of libspardl_cuda.so (declared in include/spardl_cuda.h).
// Every entry point catches the internal exceptions and returns the status
// code of the reference exception class; the message is kept per thread.
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>
#include <vector>
#include <thread>
#include <exception>
#include <algorithm>

#include "divplan.hpp"
#include "engine.hpp"
#include "host.hpp"
#include "kernels.cuh"
#include "spardl_cuda.h"

#define EXPORT extern "C" __attribute__((visibility("default")))

namespace {

thread_local std::string g_msg;

template <class F>
int guarded(F&& f) {
  try {
    g_msg.clear();
    f();
    return SPARDL_OK;
  } catch (const sdlh::Error& e) {
    g_msg = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_msg = "host out of memory";
    return SPARDL_E_ERROR;
  } catch (const std::exception& e) {
    g_msg = e.what();
    return SPARDL_E_ERROR;
  }
}

#define CK(x)                                                                            \
  do {                                                                                   \
    cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess)                                                               \
      sdlh::fail(SPARDL_E_CUDA, std::string(#x) + ": " + cudaGetErrorString(e_));        \
  } while (0)

void need(const void* p, const char* what) {
  if (!p) sdlh::fail(SPARDL_E_ARG, std::string("null argument: ") + what);
}

// scoped device allocations for the one-shot component entry points; the
// zero fill is ordered on the caller's stream (a torch side stream is
// non-blocking: a legacy-stream memset would race the uploads on it)
struct DevBuf {
  explicit DevBuf(cudaStream_t st) : s(st) {}
  cudaStream_t s;
  std::vector<void*> ptrs;
  ~DevBuf() {
    for (void* p : ptrs) cudaFree(p);
  }
  template <class T>
  T* get(size_t n) {
    void* p = nullptr;
    CK(cudaMalloc(&p, std::max<size_t>(n * sizeof(T), 16)));
    CK(cudaMemsetAsync(p, 0, std::max<size_t>(n * sizeof(T), 16), s));
    ptrs.push_back(p);
    return static_cast<T*>(p);
  }
};

// The component entry points run on the device that owns their inputs
// (restored on return), so a caller on cuda:1 needs no cudaSetDevice.
struct DeviceOf {
  int prev = -1;
  explicit DeviceOf(const void* p) {
    cudaPointerAttributes a{};
    if (p && cudaPointerGetAttributes(&a, p) == cudaSuccess && a.type == cudaMemoryTypeDevice) {
      int cur = 0;
      cudaGetDevice(&cur);
      if (cur != a.device) {
        prev = cur;
        CK(cudaSetDevice(a.device));
      }
    }
    cudaGetLastError();
  }
  ~DeviceOf() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

void require_device() {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0)
    sdlh::fail(SPARDL_E_CUDA, "no CUDA device: the SparDL device path has no CPU fallback");
}

bool wide_enabled() {   // the one-shot components: as the engine (opt-in)
  const char* e = std::getenv("SPARDL_WSEL");
  return e && (e[0] == '1' || e[0] == 'a');
}

// The wide-select scratch of a one-shot select (the same layout the engine
// plans, wselect.cu); t.ws points at its device copy.
sdl::WScratch* attach_wide(sdl::SelTask& t, DevBuf& buf, cudaStream_t s, const int32_t* idx,
                           const float* val, const int32_t* seg_off, const int32_t* seg_cnt,
                           const int32_t* count, int stride, int nseg, int group, int mode,
                           int is_div, int64_t bin_cap) {
  sdl::WScratch w{};
  w.idx = idx;
  w.val = val;
  w.seg_off = seg_off;
  w.seg_cnt = seg_cnt;
  w.count = count;
  w.stride = stride;
  w.nseg = nseg;
  w.group = std::max(1, std::min(group, 64));
  w.max_tiles = (nseg + w.group - 1) / w.group;
  w.mode = mode;
  w.is_div = is_div;
  w.bin_cap = static_cast<int32_t>(std::max<int64_t>(1, bin_cap));
  w.bin_c = buf.get<unsigned long long>(static_cast<size_t>(w.bin_cap));
  w.bin_tile = buf.get<int32_t>(static_cast<size_t>(w.bin_cap));
  const size_t nt = static_cast<size_t>(std::max(1, w.max_tiles));
  w.tile_n = buf.get<int32_t>(nt);
  w.tile_sel = buf.get<int32_t>(nt);
  w.tile_sel_off = buf.get<int32_t>(nt);
  w.tile_dis_off = buf.get<int32_t>(nt);
  sdl::WScratch* d = buf.get<sdl::WScratch>(1);
  CK(cudaMemcpyAsync(d, &w, sizeof(w), cudaMemcpyHostToDevice, s));
  CK(cudaStreamSynchronize(s));   // (w is a host temporary)
  t.ws = d;
  return d;
}

// One select over prepared inputs, with its scratch: the wide path (when
// t.ws is set), then the cluster select for a task it hands back.
void run_select(sdl::SelTask t, cudaStream_t s, DevBuf& buf, int max_tiles = 0,
                bool dividing = false) {
  sdl::sel_prepare(t, t.stride);
  if (t.nseg > sdl::kMaxSegPerTask || t.dnseg > sdl::kMaxSegPerTask)
    sdlh::fail(SPARDL_E_UNSUPPORTED, "selection larger than the device work-item bound");
  t.scr = buf.get<sdl::SelScratch>(1);
  const int nck = std::max(1, sdl::sel_chunk_capacity(t));
  int32_t* segs = buf.get<int32_t>(6 * static_cast<size_t>(nck));
  t.seg_gt = segs;
  t.seg_eq = segs + nck;
  t.seg_sel_off = segs + 2 * nck;
  t.seg_dis_off = segs + 3 * nck;
  t.seg_take = segs + 4 * nck;
  t.seg_valid = segs + 5 * nck;
  sdl::SelTask* td = buf.get<sdl::SelTask>(1);
  CK(cudaMemcpyAsync(td, &t, sizeof(t), cudaMemcpyHostToDevice, s));
  (void)dividing;   // (the one-shot slice histograms in the histogram pass)
  if (t.ws) sdl::launch_wselect(td, 1, max_tiles, true, s);
  sdl::launch_select(td, 1, std::max(1, sdl::sel_scratch_segments(t)), s);
  CK(sdl::take_launch_error());
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(s));   // (t is a host temporary)
}

}  // namespace

EXPORT const char* spardl_last_error(void) { return g_msg.c_str(); }

EXPORT int spardl_device_count(int32_t* n) {
  return guarded([&] {
    need(n, "n");
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) {
      cudaGetLastError();
      c = 0;
    }
    *n = c;
  });
}
EXPORT int spardl_abi_version(void) { return SPARDL_ABI_VERSION; }

// ---------------------------------------------------------------------------
// host schedule logic
EXPORT int spardl_validate(const spardl_config* cfg) {
  return guarded([&] {
    need(cfg, "cfg");
    sdlh::validate(*cfg);
  });
}

EXPORT int spardl_partition(int64_t n, int32_t count, int64_t* lo, int64_t* hi) {
  return guarded([&] {
    const auto p = sdlh::partition(n, count);
    for (int b = 0; b < count; ++b) {
      lo[b] = p.lo[static_cast<size_t>(b)];
      hi[b] = p.hi[static_cast<size_t>(b)];
    }
  });
}

EXPORT int spardl_block_of(int64_t n, int32_t count, int64_t i, int32_t* block) {
  return guarded([&] {
    const auto p = sdlh::partition(n, count);
    if (i < 0 || i >= n) sdlh::fail(SPARDL_E_ARG, "index outside [0, N)");
    *block = p.block_of(i);
  });
}

EXPORT int spardl_build_bags(int32_t m, int32_t rank, int32_t* l, int32_t* remainder,
                             int32_t* bag_size, int32_t* positions) {
  return guarded([&] {
    const auto s = sdlh::build_bags(m, rank);
    *l = s.l;
    *remainder = s.remainder;
    int o = 0;
    for (size_t j = 0; j < s.bags.size(); ++j) {
      bag_size[j] = static_cast<int32_t>(s.bags[j].size());
      for (int p : s.bags[j]) positions[o++] = p;
    }
  });
}

EXPORT int spardl_expected_cost_srs(int64_t m, int64_t k, int64_t* rounds, int64_t* scalars) {
  return guarded([&] {   // inc/reduce_scatter.hpp:257-262
    if (m < 1) sdlh::fail(SPARDL_E_CONFIG, "expected_cost_srs: m >= 1 required");
    if (k % m != 0) sdlh::fail(SPARDL_E_CONFIG, "expected_cost_srs: m must divide k");
    if (m == 1) {
      *rounds = 0;
      *scalars = 0;
    } else {
      *rounds = sdlh::ceil_log2(m);
      *scalars = 2 * (k / m) * (m - 1);
    }
  });
}

EXPORT int spardl_expected_cost_sag(int64_t P, int64_t k, int64_t d, int32_t mode,
                                    int64_t* rounds, int64_t* low, int64_t* high) {
  return guarded([&] { sdlh::expected_cost_sag(P, k, d, mode, rounds, low, high); });
}

EXPORT int spardl_bsag_phase_cost(int64_t P, int64_t k, int64_t d, int64_t* rounds,
                                  int64_t* low, int64_t* high) {
  return guarded([&] {   // inc/sag.hpp:332-340
    if (d < 2 || P % d != 0 || k % P != 0)
      sdlh::fail(SPARDL_E_CONFIG, "bsag_phase_cost: invalid (P, k, d)");
    const int64_t c = k / P;
    *rounds = sdlh::ceil_log2(d);
    *low = 2 * c * (d - 1);
    *high = 2 * c * d * (d - 1);
  });
}

EXPORT int spardl_topka_cost(int64_t P, int64_t k, int64_t* rounds, int64_t* low,
                             int64_t* high) {
  return guarded([&] {   // inc/sag.hpp:343-346
    const int64_t sc = 2 * (P - 1) * k;
    *rounds = sdlh::ceil_log2(P);
    *low = *high = sc;
  });
}

EXPORT int spardl_dyadic_shares(int32_t count, double* out) {
  return guarded([&] {
    const auto s = sdlh::dyadic_shares(count);
    for (size_t i = 0; i < s.size(); ++i) out[i] = s[i];
  });
}

EXPORT int spardl_hctrl_init(spardl_hctrl* c, int64_t P, int64_t k, int64_t d) {
  return guarded([&] {
    need(c, "controller");
    sdlh::hctrl_init(c, P, k, d);
  });
}

EXPORT int spardl_hctrl_observe(spardl_hctrl* c, int64_t n_t) {
  return guarded([&] {
    need(c, "controller");
    sdlh::hctrl_observe(c, n_t);
  });
}

EXPORT int spardl_hctrl_budget(const spardl_hctrl* c, int64_t* budget) {
  return guarded([&] {
    need(c, "controller");
    *budget = sdlh::hctrl_budget(c);
  });
}

// ---------------------------------------------------------------------------
// device components
EXPORT int spardl_topk_select(const int32_t* idx, const float* val, int64_t n, int64_t budget,
                              int32_t* sel_idx, float* sel_val, int64_t* n_sel,
                              int32_t* dis_idx, float* dis_val, int64_t* n_dis, void* stream) {
  return guarded([&] {   // inc/sparse.hpp:136-162
    require_device();
    if (budget < 0) sdlh::fail(SPARDL_E_ERROR, "top_k_select: negative budget");
    if (n < 0 || n >= (int64_t(1) << 31)) sdlh::fail(SPARDL_E_ARG, "n out of range");
    DeviceOf on(val);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    DevBuf buf(s);
    int32_t* cnt = buf.get<int32_t>(3);
    const int32_t n32 = static_cast<int32_t>(n);
    CK(cudaMemcpyAsync(cnt, &n32, sizeof(n32), cudaMemcpyHostToDevice, s));
    sdl::SelTask t{};
    t.mode = 0;
    t.idx = idx;
    t.val = val;
    t.count = cnt;
    int64_t stride = sdl::kTile;
    while ((n + stride - 1) / stride > sdl::kMaxSegPerTask) stride += sdl::kTile;
    t.stride = static_cast<int32_t>(stride);
    t.nseg = static_cast<int32_t>((n + stride - 1) / stride);
    t.budget = budget;
    t.sel_idx = sel_idx;
    t.sel_val = sel_val;
    t.sel_cnt = cnt + 1;
    t.dis_idx = dis_idx;
    t.dis_val = dis_val;
    t.dis_cnt = dis_idx ? cnt + 2 : nullptr;
    t.weight = 1.f;
    int tiles = 0;
    if (n > 0 && wide_enabled()) {
      constexpr int kStride = 8192;
      const int ns = static_cast<int>((n + kStride - 1) / kStride);
      attach_wide(t, buf, s, idx, val, nullptr, nullptr, cnt, kStride, ns, 1, sdl::kWAuto, 0,
                  std::max<int64_t>(16384, n / 8));
      tiles = ns;
    }
    if (n > 0) run_select(t, s, buf, tiles);
    int32_t out[3] = {0, 0, 0};
    CK(cudaMemcpyAsync(out, cnt, sizeof(out), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    *n_sel = out[1];
    if (n_dis) *n_dis = dis_idx ? out[2] : n - out[1];
  });
}

EXPORT int spardl_topk_select_slice(const float* g, int64_t lo, int64_t hi, int64_t budget,
                                    int32_t* sel_idx, float* sel_val, int64_t* n_sel,
                                    void* stream) {
  return guarded([&] {   // inc/sparse.hpp:167-177, through the dividing kernels
    require_device();
    if (budget < 0) sdlh::fail(SPARDL_E_ERROR, "top_k_select: negative budget");
    if (lo < 0 || hi < lo || hi >= (int64_t(1) << 31)) sdlh::fail(SPARDL_E_ARG, "bad range");
    if (reinterpret_cast<uintptr_t>(g) % 16 != 0)
      sdlh::fail(SPARDL_E_ARG, "slice base must be 16-byte aligned");
    DeviceOf on(g);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    const int64_t nb = hi - lo;
    if (nb == 0) {
      *n_sel = 0;
      return;
    }
    DevBuf buf(s);
    sdl::DivTask dt{};
    sdl::SelTask t{};
    sdl::div_plan(dt, t, lo, hi, budget,
                  [&](size_t n) { return static_cast<void*>(buf.get<unsigned char>(n)); });
    dt.carry = const_cast<float*>(g);   // read only when apply_residual == 0
    dt.err = buf.get<int32_t>(1);
    int tiles = 0;
    if (dt.use_cand && wide_enabled()) {
      dt.ws = attach_wide(t, buf, s, dt.cand_idx, dt.cand_val, nullptr, dt.cand_cnt, nullptr,
                          dt.cap, dt.nchunks, 64, sdl::kWWindow, 1,
                          std::max<int64_t>(16384, budget / 8));
      tiles = (dt.nchunks + 63) / 64;
    }
    sdl::DivTask* dtd = buf.get<sdl::DivTask>(1);
    CK(cudaMemcpyAsync(dtd, &dt, sizeof(dt), cudaMemcpyHostToDevice, s));
    sdl::launch_divide(dtd, 1, dt.nchunks, dt.sample_every, 0, s);
    int32_t* cnt = buf.get<int32_t>(1);
    t.dval = g + lo;
    t.sel_idx = sel_idx;
    t.sel_val = sel_val;
    t.sel_cnt = cnt;
    run_select(t, s, buf, tiles, true);
    int32_t out = 0, err = 0;
    CK(cudaMemcpyAsync(&out, cnt, sizeof(out), cudaMemcpyDeviceToHost, s));
    CK(cudaMemcpyAsync(&err, dt.err, sizeof(err), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    if (err) sdlh::fail(SPARDL_E_ARG, "gradient contains NaN (selection order undefined)");
    *n_sel = out;
  });
}

EXPORT int spardl_merge_add(int32_t r, const int32_t* const* idx, const float* const* val,
                            const int64_t* n, int32_t* out_idx, float* out_val, int64_t* n_out,
                            void* stream) {
  return guarded([&] {   // inc/sparse.hpp:182-208 folded left over r lists
    require_device();
    if (r < 1 || r > sdl::kMaxR) sdlh::fail(SPARDL_E_ARG, "merge_add: 1 <= r <= 16 lists");
    DeviceOf on(out_idx);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    DevBuf buf(s);
    int32_t* cnts = buf.get<int32_t>(static_cast<size_t>(r) + 1);
    std::vector<int32_t> hc(static_cast<size_t>(r));
    int64_t capsum = 0, capmax = 1;
    for (int q = 0; q < r; ++q) {
      hc[static_cast<size_t>(q)] = static_cast<int32_t>(n[q]);
      capsum += n[q];
      capmax = std::max<int64_t>(capmax, n[q]);
    }
    CK(cudaMemcpyAsync(cnts, hc.data(), sizeof(int32_t) * r, cudaMemcpyHostToDevice, s));
    sdl::MergeTask mt{};
    mt.r = r;
    for (int q = 0; q < r; ++q) {
      mt.in_idx[q] = idx[q];
      mt.in_val[q] = val[q];
      mt.in_cnt[q] = cnts + q;
    }
    int64_t T = std::max<int64_t>(2048 / r, (capsum + sdl::kMaxSamples - 1) / sdl::kMaxSamples);
    T = (std::max<int64_t>(T, 32) + 3) & ~int64_t(3);
    if (static_cast<int64_t>(r) * T > 12800)
      sdlh::fail(SPARDL_E_UNSUPPORTED, "merge of this size exceeds the shared-memory envelope");
    mt.T = static_cast<int32_t>(T);
    int64_t parts = 0;
    for (int q = 0; q < r; ++q) parts += (n[q] + T - 1) / T;
    parts = std::max<int64_t>(parts, 1);
    mt.max_parts = static_cast<int32_t>(parts);
    mt.splitters = buf.get<int32_t>(parts + 1);
    mt.windows = buf.get<int32_t>(parts * r);
    mt.nparts = buf.get<int32_t>(1);
    mt.out_idx = buf.get<int32_t>(std::max<int64_t>(capsum, 1));
    mt.out_val = buf.get<float>(std::max<int64_t>(capsum, 1));
    mt.out_cap = std::max<int64_t>(capsum, 1);
    mt.seg_off = buf.get<int32_t>(parts);
    mt.seg_cnt = buf.get<int32_t>(parts);
    sdl::MergeTask* mtd = buf.get<sdl::MergeTask>(1);
    CK(cudaMemcpyAsync(mtd, &mt, sizeof(mt), cudaMemcpyHostToDevice, s));
    sdl::launch_merge(mtd, 1, static_cast<int>(parts), static_cast<int>(r * T), static_cast<int>(r), s);
    sdl::SelTask t{};
    t.mode = 0;
    t.idx = mt.out_idx;
    t.val = mt.out_val;
    t.seg_off = mt.seg_off;
    t.seg_cnt = mt.seg_cnt;
    t.nseg = static_cast<int32_t>(parts);
    t.stride = static_cast<int32_t>(r * T);
    t.budget = INT64_MAX;   // identity selection == ordered compaction
    t.sel_idx = out_idx;
    t.sel_val = out_val;
    t.sel_cnt = cnts + r;
    t.weight = 1.f;
    int tiles = 0;
    if (wide_enabled()) {
      const int grp = std::max(1, 8192 / static_cast<int>(T));
      attach_wide(t, buf, s, mt.out_idx, mt.out_val, mt.seg_off, mt.seg_cnt, nullptr,
                  static_cast<int>(r * T), static_cast<int>(parts), grp, sdl::kWAuto, 0, 16384);
      tiles = static_cast<int>((parts + grp - 1) / grp);
    }
    run_select(t, s, buf, tiles);
    int32_t out = 0;
    CK(cudaMemcpyAsync(&out, cnts + r, sizeof(out), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    *n_out = out;
  });
}

// ---------------------------------------------------------------------------
// host-buffer variants: stage through the device, run the device kernels
namespace {
template <class T>
T* to_dev(DevBuf& buf, const T* host, size_t n) {
  T* d = buf.get<T>(std::max<size_t>(n, 1));
  if (n) CK(cudaMemcpy(d, host, sizeof(T) * n, cudaMemcpyHostToDevice));
  return d;
}
template <class T>
void to_host(T* host, const T* dev, size_t n) {
  if (n) CK(cudaMemcpy(host, dev, sizeof(T) * n, cudaMemcpyDeviceToHost));
}
}  // namespace

EXPORT int spardl_topk_select_hostbuf(const int32_t* idx, const float* val, int64_t n,
                                      int64_t budget, int32_t* sel_idx, float* sel_val,
                                      int64_t* n_sel, int32_t* dis_idx, float* dis_val,
                                      int64_t* n_dis) {
  int rc = SPARDL_OK;
  const int outer = guarded([&] {
    require_device();
    DevBuf buf(nullptr);
    const size_t un = static_cast<size_t>(n < 0 ? 0 : n);
    int32_t* di = to_dev(buf, idx, un);
    float* dv = to_dev(buf, val, un);
    int32_t* si = buf.get<int32_t>(un + 1);
    float* sv = buf.get<float>(un + 1);
    int32_t* xi = dis_idx ? buf.get<int32_t>(un + 1) : nullptr;
    float* xv = dis_idx ? buf.get<float>(un + 1) : nullptr;
    int64_t ns = 0, nd = 0;
    rc = spardl_topk_select(di, dv, n, budget, si, sv, &ns, xi, xv, &nd, nullptr);
    if (rc != SPARDL_OK) return;
    to_host(sel_idx, si, static_cast<size_t>(ns));
    to_host(sel_val, sv, static_cast<size_t>(ns));
    if (dis_idx) {
      to_host(dis_idx, xi, static_cast<size_t>(nd));
      to_host(dis_val, xv, static_cast<size_t>(nd));
    }
    *n_sel = ns;
    if (n_dis) *n_dis = nd;
  });
  return rc != SPARDL_OK ? rc : outer;
}

EXPORT int spardl_topk_select_slice_hostbuf(const float* g, int64_t lo, int64_t hi,
                                            int64_t budget, int32_t* sel_idx, float* sel_val,
                                            int64_t* n_sel) {
  int rc = SPARDL_OK;
  const int outer = guarded([&] {
    require_device();
    if (hi < lo || lo < 0) sdlh::fail(SPARDL_E_ARG, "bad range");
    DevBuf buf(nullptr);
    float* dg = to_dev(buf, g, static_cast<size_t>(hi));
    const size_t cap = static_cast<size_t>(hi - lo) + 1;
    int32_t* si = buf.get<int32_t>(cap);
    float* sv = buf.get<float>(cap);
    int64_t ns = 0;
    rc = spardl_topk_select_slice(dg, lo, hi, budget, si, sv, &ns, nullptr);
    if (rc != SPARDL_OK) return;
    to_host(sel_idx, si, static_cast<size_t>(ns));
    to_host(sel_val, sv, static_cast<size_t>(ns));
    *n_sel = ns;
  });
  return rc != SPARDL_OK ? rc : outer;
}

EXPORT int spardl_merge_add_hostbuf(int32_t r, const int32_t* const* idx, const float* const* val,
                                    const int64_t* n, int32_t* out_idx, float* out_val,
                                    int64_t* n_out) {
  int rc = SPARDL_OK;
  const int outer = guarded([&] {
    require_device();
    if (r < 1 || r > sdl::kMaxR) sdlh::fail(SPARDL_E_ARG, "merge_add: 1 <= r <= 16 lists");
    DevBuf buf(nullptr);
    std::vector<const int32_t*> di(static_cast<size_t>(r));
    std::vector<const float*> dv(static_cast<size_t>(r));
    size_t total = 0;
    for (int q = 0; q < r; ++q) {
      di[static_cast<size_t>(q)] = to_dev(buf, idx[q], static_cast<size_t>(n[q]));
      dv[static_cast<size_t>(q)] = to_dev(buf, val[q], static_cast<size_t>(n[q]));
      total += static_cast<size_t>(n[q]);
    }
    int32_t* oi = buf.get<int32_t>(total + 1);
    float* ov = buf.get<float>(total + 1);
    int64_t no = 0;
    rc = spardl_merge_add(r, di.data(), dv.data(), n, oi, ov, &no, nullptr);
    if (rc != SPARDL_OK) return;
    to_host(out_idx, oi, static_cast<size_t>(no));
    to_host(out_val, ov, static_cast<size_t>(no));
    *n_out = no;
  });
  return rc != SPARDL_OK ? rc : outer;
}

// ---------------------------------------------------------------------------
// fp64 components (the C++ drop-in surface keeps the reference's double
// semantics for its one-shot component calls; components64.cu)
EXPORT int spardl_topk_select_f64(const int64_t* idx, const double* val, int64_t n,
                                  int64_t budget, uint8_t* flag, void* stream) {
  return guarded([&] {   // inc/sparse.hpp:136-162
    require_device();
    if (budget < 0) sdlh::fail(SPARDL_E_ERROR, "top_k_select: negative budget");
    if (n < 0 || n >= (int64_t(1) << 31)) sdlh::fail(SPARDL_E_ARG, "n out of range");
    DeviceOf on(val);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    sdl::launch_topk64(idx, val, static_cast<int>(n), budget, flag, s);
    CK(sdl::take_launch_error());
    CK(cudaStreamSynchronize(s));
  });
}

EXPORT int spardl_merge_add_f64(const int64_t* ai, const double* av, int64_t na,
                                const int64_t* bi, const double* bv, int64_t nb, int64_t* oi,
                                double* ov, int64_t* n_out, void* stream) {
  return guarded([&] {   // inc/sparse.hpp:182-208
    require_device();
    if (na < 0 || nb < 0 || na + nb >= (int64_t(1) << 31)) sdlh::fail(SPARDL_E_ARG, "n out of range");
    DeviceOf on(oi);
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    DevBuf buf(s);
    const size_t n = static_cast<size_t>(na + nb) + 1;
    int64_t* ti = buf.get<int64_t>(n);
    double* tv = buf.get<double>(n);
    int64_t* no = buf.get<int64_t>(1);
    sdl::launch_merge64(ai, av, static_cast<int>(na), bi, bv, static_cast<int>(nb), ti, tv, oi,
                        ov, no, s);
    CK(sdl::take_launch_error());
    CK(cudaMemcpyAsync(n_out, no, sizeof(int64_t), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
  });
}

EXPORT int spardl_topk_select_f64_hostbuf(const int64_t* idx, const double* val, int64_t n,
                                          int64_t budget, uint8_t* flag) {
  int rc = SPARDL_OK;
  const int outer = guarded([&] {
    require_device();
    DevBuf buf(nullptr);
    const size_t un = static_cast<size_t>(n < 0 ? 0 : n);
    const int64_t* di = to_dev(buf, idx, un);
    const double* dv = to_dev(buf, val, un);
    uint8_t* df = buf.get<uint8_t>(un + 1);
    rc = spardl_topk_select_f64(di, dv, n, budget, df, nullptr);
    if (rc != SPARDL_OK) return;
    to_host(flag, df, un);
  });
  return rc != SPARDL_OK ? rc : outer;
}

EXPORT int spardl_merge_add_f64_hostbuf(const int64_t* ai, const double* av, int64_t na,
                                        const int64_t* bi, const double* bv, int64_t nb,
                                        int64_t* oi, double* ov, int64_t* n_out) {
  int rc = SPARDL_OK;
  const int outer = guarded([&] {
    require_device();
    DevBuf buf(nullptr);
    const int64_t* dai = to_dev(buf, ai, static_cast<size_t>(na));
    const double* dav = to_dev(buf, av, static_cast<size_t>(na));
    const int64_t* dbi = to_dev(buf, bi, static_cast<size_t>(nb));
    const double* dbv = to_dev(buf, bv, static_cast<size_t>(nb));
    int64_t* doi = buf.get<int64_t>(static_cast<size_t>(na + nb) + 1);
    double* dov = buf.get<double>(static_cast<size_t>(na + nb) + 1);
    int64_t no = 0;
    rc = spardl_merge_add_f64(dai, dav, na, dbi, dbv, nb, doi, dov, &no, nullptr);
    if (rc != SPARDL_OK) return;
    to_host(oi, doi, static_cast<size_t>(no));
    to_host(ov, dov, static_cast<size_t>(no));
    *n_out = no;
  });
  return rc != SPARDL_OK ? rc : outer;
}

// ---------------------------------------------------------------------------
// pipeline context
struct spardl_ctx {
  std::unique_ptr<sdle::Engine> eng;
  std::vector<float*> staging;     // device copies of host gradients (allreduce_host)
  std::vector<const float*> staging_c;
  cudaEvent_t ev_up = nullptr, ev_up2 = nullptr;   // upload fork / join
  ~spardl_ctx() {
    if (ev_up) cudaEventDestroy(ev_up);
    if (ev_up2) cudaEventDestroy(ev_up2);
  }
};

EXPORT int spardl_nccl_unique_id(void* out128) {
  return guarded([&] {
    need(out128, "out");
    ncclUniqueId id;
    const ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) sdlh::fail(SPARDL_E_NCCL, ncclGetErrorString(r));
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(out128, &id, sizeof(id));
  });
}

EXPORT int spardl_ctx_create(const spardl_config* cfg, int32_t device, int32_t world_size,
                             int32_t rank, const void* nccl_id, void* stream, spardl_ctx** out) {
  return guarded([&] {
    need(cfg, "cfg");
    need(out, "out");
    *out = nullptr;
    auto c = std::make_unique<spardl_ctx>();
    c->eng = std::make_unique<sdle::Engine>(*cfg, device, world_size, rank, nccl_id,
                                            static_cast<cudaStream_t>(stream));
    *out = c.release();
  });
}

EXPORT int spardl_plan_ops(const spardl_config* cfg, int32_t world_size, int32_t rank,
                           int64_t* ops, int64_t cap, int64_t* n_ops) {
  return guarded([&] {
    need(cfg, "cfg");
    need(n_ops, "n_ops");
    sdle::Engine e(*cfg, 0, world_size, rank, nullptr, nullptr, /*plan_only=*/true);
    const auto v = e.plan_ops();
    *n_ops = static_cast<int64_t>(v.size());
    if (ops) {
      if (cap < *n_ops) sdlh::fail(SPARDL_E_ARG, "ops capacity too small");
      for (size_t i = 0; i < v.size(); ++i) {
        ops[5 * i + 0] = v[i].round;
        ops[5 * i + 1] = v[i].peer;
        ops[5 * i + 2] = v[i].is_send;
        ops[5 * i + 3] = v[i].uid;
        ops[5 * i + 4] = v[i].bytes;
      }
    }
  });
}

EXPORT int spardl_ctx_destroy(spardl_ctx* ctx) {
  return guarded([&] {
    if (!ctx) return;
    for (float* p : ctx->staging) cudaFree(p);
    delete ctx;
  });
}

EXPORT int spardl_ctx_local_workers(const spardl_ctx* ctx, int32_t* first, int32_t* count) {
  return guarded([&] {
    need(ctx, "ctx");
    *first = ctx->eng->first_worker();
    *count = ctx->eng->local_workers();
  });
}

EXPORT int spardl_ctx_transport(const spardl_ctx* ctx, int32_t* peer) {
  return guarded([&] {
    need(ctx, "ctx");
    need(peer, "peer");
    *peer = ctx->eng->peer_transport() ? 1 : 0;
  });
}

EXPORT int spardl_ctx_set_graph(spardl_ctx* ctx, int32_t enable) {
  return guarded([&] {
    need(ctx, "ctx");
    ctx->eng->set_graph(enable != 0);
  });
}

EXPORT int spardl_ctx_set_audit(spardl_ctx* ctx, int32_t enable) {
  return guarded([&] {
    need(ctx, "ctx");
    ctx->eng->set_audit(enable != 0);
  });
}

EXPORT int spardl_allreduce(spardl_ctx* ctx, const float* const* grads_dev) {
  return guarded([&] {
    need(ctx, "ctx");
    need(grads_dev, "grads");
    ctx->eng->run(grads_dev);
  });
}

EXPORT int spardl_allreduce_host(spardl_ctx* ctx, const float* const* grads_host,
                                 int64_t* g_idx, float* g_val, int64_t cap, int64_t* nnz) {
  return guarded([&] {
    need(ctx, "ctx");
    need(grads_host, "grads");
    auto& e = *ctx->eng;
    const int wl = e.local_workers();
    const size_t bytes = sizeof(float) * static_cast<size_t>(e.dimension());
    if (ctx->staging.empty()) {
      for (int i = 0; i < wl; ++i) {
        float* p = nullptr;
        CK(cudaMalloc(&p, bytes));
        ctx->staging.push_back(p);
        ctx->staging_c.push_back(p);
      }
    }
    cudaStream_t s = e.stream();
    // the uploads alternate between two streams (two copy engines on the
    // link) and join before the iteration
    cudaStream_t s2 = e.side_stream();
    if (!ctx->ev_up) {
      CK(cudaEventCreateWithFlags(&ctx->ev_up, cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&ctx->ev_up2, cudaEventDisableTiming));
    }
    CK(cudaEventRecord(ctx->ev_up, s));
    CK(cudaStreamWaitEvent(s2, ctx->ev_up, 0));
    for (int i = 0; i < wl; ++i) {
      need(grads_host[i], "grads[i]");
      CK(cudaMemcpyAsync(ctx->staging[static_cast<size_t>(i)], grads_host[i], bytes,
                         cudaMemcpyHostToDevice, (i & 1) ? s2 : s));
    }
    CK(cudaEventRecord(ctx->ev_up2, s2));
    CK(cudaStreamWaitEvent(s, ctx->ev_up2, 0));
    e.run(ctx->staging_c.data());
    const int32_t* di = nullptr;
    const float* dv = nullptr;
    int64_t n = 0;
    e.global(0, &di, &dv, &n);   // synchronises
    *nnz = n;
    if (g_idx && g_val) {
      if (cap < n) sdlh::fail(SPARDL_E_ARG, "output capacity below the global nnz");
      std::vector<int32_t> tmp(static_cast<size_t>(n));
      CK(cudaMemcpyAsync(tmp.data(), di, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s));
      CK(cudaMemcpyAsync(g_val, dv, sizeof(float) * n, cudaMemcpyDeviceToHost, s));
      CK(cudaStreamSynchronize(s));
      for (int64_t q = 0; q < n; ++q) g_idx[q] = tmp[static_cast<size_t>(q)];
    }
  });
}

EXPORT int spardl_profile(spardl_ctx* ctx, const float* const* grads_dev, int32_t iters,
                          double* phase_ms) {
  return guarded([&] {
    need(ctx, "ctx");
    need(grads_dev, "grads");
    need(phase_ms, "phase_ms");
    ctx->eng->profile(grads_dev, iters, phase_ms);
  });
}

EXPORT int spardl_sync(spardl_ctx* ctx) {
  return guarded([&] {
    need(ctx, "ctx");
    ctx->eng->sync();
  });
}

EXPORT int spardl_get_run_info(spardl_ctx* ctx, spardl_run_info* out) {
  return guarded([&] {
    need(ctx, "ctx");
    *out = ctx->eng->run_info();
  });
}

EXPORT int spardl_get_global(spardl_ctx* ctx, int32_t local_worker, const int32_t** idx,
                             const float** val, int64_t* nnz) {
  return guarded([&] {
    need(ctx, "ctx");
    if (local_worker < 0 || local_worker >= ctx->eng->local_workers())
      sdlh::fail(SPARDL_E_ARG, "local worker out of range");
    ctx->eng->global(local_worker, idx, val, nnz);
  });
}

EXPORT int spardl_get_carry(spardl_ctx* ctx, int32_t local_worker, float** carry_dev) {
  return guarded([&] {
    need(ctx, "ctx");
    if (local_worker < 0 || local_worker >= ctx->eng->local_workers())
      sdlh::fail(SPARDL_E_ARG, "local worker out of range");
    *carry_dev = ctx->eng->carry(local_worker);
  });
}

EXPORT int spardl_carry_to_host(spardl_ctx* ctx, int32_t local_worker, float* host) {
  return guarded([&] {
    need(ctx, "ctx");
    need(host, "host");
    if (local_worker < 0 || local_worker >= ctx->eng->local_workers())
      sdlh::fail(SPARDL_E_ARG, "local worker out of range");
    ctx->eng->sync();
    CK(cudaMemcpy(host, ctx->eng->carry(local_worker),
                  sizeof(float) * static_cast<size_t>(ctx->eng->dimension()),
                  cudaMemcpyDeviceToHost));
  });
}

EXPORT int spardl_carry_from_host(spardl_ctx* ctx, int32_t local_worker, const float* host) {
  return guarded([&] {
    need(ctx, "ctx");
    need(host, "host");
    if (local_worker < 0 || local_worker >= ctx->eng->local_workers())
      sdlh::fail(SPARDL_E_ARG, "local worker out of range");
    ctx->eng->sync();
    CK(cudaMemcpy(ctx->eng->carry(local_worker), host,
                  sizeof(float) * static_cast<size_t>(ctx->eng->dimension()),
                  cudaMemcpyHostToDevice));
  });
}

EXPORT int spardl_set_controller(spardl_ctx* ctx, int32_t local_worker, const spardl_hctrl* c) {
  return guarded([&] {
    need(ctx, "ctx");
    need(c, "controller");
    ctx->eng->set_controller(local_worker, *c);
  });
}

EXPORT int spardl_ctx_reset_state(spardl_ctx* ctx) {
  return guarded([&] {
    need(ctx, "ctx");
    ctx->eng->reset_state();
  });
}

EXPORT int spardl_get_ledger(spardl_ctx* ctx, int64_t* rounds, int64_t* scalars) {
  return guarded([&] {
    need(ctx, "ctx");
    ctx->eng->ledger(rounds, scalars);
  });
}

EXPORT int spardl_get_union_sizes(spardl_ctx* ctx, int64_t* out) {
  return guarded([&] {
    need(ctx, "ctx");
    ctx->eng->union_sizes(out);
  });
}

EXPORT int spardl_get_controller(spardl_ctx* ctx, int32_t local_worker, spardl_hctrl* out) {
  return guarded([&] {
    need(ctx, "ctx");
    ctx->eng->controller(local_worker, out);
  });
}

EXPORT int spardl_dense_fallbacks(spardl_ctx* ctx, int64_t* count) {
  return guarded([&] {
    need(ctx, "ctx");
    *count = ctx->eng->dense_fallbacks();
  });
}

EXPORT int spardl_dense_fallbacks_total(spardl_ctx* ctx, int64_t* count) {
  return guarded([&] {
    need(ctx, "ctx");
    need(count, "count");
    *count = ctx->eng->dense_fallbacks_total();
  });
}

EXPORT int spardl_candidate_retries(spardl_ctx* ctx, int64_t* count) {
  return guarded([&] {
    need(ctx, "ctx");
    need(count, "count");
    *count = ctx->eng->candidate_retries();
  });
}

EXPORT int spardl_wide_handed_back(spardl_ctx* ctx, int64_t* count) {
  return guarded([&] {
    need(ctx, "ctx");
    need(count, "count");
    *count = ctx->eng->wide_handed_back();
  });
}

EXPORT int spardl_div_diag(spardl_ctx* ctx, int32_t task, int64_t* out9) {
  return guarded([&] {
    need(ctx, "ctx");
    ctx->eng->div_diag(task, out9);
  });
}

EXPORT int spardl_debug_select_timestamps(spardl_ctx* ctx, int32_t step, int32_t task,
                                          int64_t* out12) {
  return guarded([&] {
    need(ctx, "ctx");
    ctx->eng->select_timestamps(step, task, out12);
  });
}

EXPORT int spardl_kernel_launches(const spardl_ctx* ctx, int64_t* per_iteration) {
  return guarded([&] {
    need(ctx, "ctx");
    *per_iteration = ctx->eng->launches_per_iter();
  });
}

EXPORT int spardl_ctx_stream(const spardl_ctx* ctx, void** stream) {
  return guarded([&] {
    need(ctx, "ctx");
    *stream = static_cast<void*>(ctx->eng->stream());
  });
}

// ---------------------------------------------------------------------------
// One process, one host thread, every local GPU (inc/fabric.hpp:47-53: one
// call advances all P workers).  One engine per device, ranks 0..ndev-1 of
// one NCCL clique; peers in this process read each other's buffers through
// direct peer access (no IPC).  Calls that are collective across the
// engines (creation, the run-info / ledger gathers) run one host thread per
// device; an iteration is enqueued on all devices from the caller's thread.
struct spardl_mctx {
  std::vector<std::unique_ptr<sdle::Engine>> eng;
  std::vector<int> dev;
  std::vector<float*> staging;        // allreduce_host: device copies, worker order
  int wloc = 1;
  ~spardl_mctx() {
    for (size_t i = 0; i < staging.size(); ++i) {
      cudaSetDevice(dev[i / static_cast<size_t>(wloc)]);
      cudaFree(staging[i]);
    }
  }
};

namespace {
// f(i) on one host thread per engine; the first exception is rethrown
template <class F>
void each_engine(spardl_mctx& m, F&& f) {
  std::vector<std::exception_ptr> errs(m.dev.size());
  std::vector<std::thread> th;
  for (size_t i = 0; i < m.dev.size(); ++i)
    th.emplace_back([&, i] {
      try {
        if (cudaSetDevice(m.dev[i]) != cudaSuccess) sdlh::fail(SPARDL_E_CUDA, "cudaSetDevice");
        f(static_cast<int>(i));
      } catch (...) {
        errs[i] = std::current_exception();
      }
    });
  for (auto& t : th) t.join();
  for (auto& e : errs)
    if (e) std::rethrow_exception(e);
}
}  // namespace

EXPORT int spardl_mctx_create(const spardl_config* cfg, int32_t ndev, const int32_t* devs,
                              spardl_mctx** out) {
  return guarded([&] {
    need(cfg, "cfg");
    need(out, "out");
    require_device();
    sdlh::validate(*cfg);
    int avail = 0;
    CK(cudaGetDeviceCount(&avail));
    if (ndev < 1) sdlh::fail(SPARDL_E_ARG, "ndev must be >= 1");
    if (cfg->workers % ndev != 0)
      sdlh::fail(SPARDL_E_UNSUPPORTED, "P must be a positive multiple of the device count");
    auto m = std::make_unique<spardl_mctx>();
    for (int i = 0; i < ndev; ++i) {
      const int d = devs ? devs[i] : i;
      if (d < 0 || d >= avail) sdlh::fail(SPARDL_E_ARG, "device index out of range");
      m->dev.push_back(d);
    }
    m->wloc = static_cast<int>(cfg->workers / ndev);
    ncclUniqueId id{};
    if (ndev > 1) {
      const ncclResult_t r = ncclGetUniqueId(&id);
      if (r != ncclSuccess) sdlh::fail(SPARDL_E_NCCL, ncclGetErrorString(r));
    }
    m->eng.resize(static_cast<size_t>(ndev));
    each_engine(*m, [&](int i) {
      m->eng[static_cast<size_t>(i)] = std::make_unique<sdle::Engine>(
          *cfg, m->dev[static_cast<size_t>(i)], ndev, i, ndev > 1 ? &id : nullptr, nullptr);
    });
    *out = m.release();
  });
}

EXPORT int spardl_mctx_destroy(spardl_mctx* m) {
  return guarded([&] { delete m; });
}

EXPORT int spardl_mctx_devices(const spardl_mctx* m, int32_t* ndev, int32_t* transport_peer) {
  return guarded([&] {
    need(m, "mctx");
    if (ndev) *ndev = static_cast<int32_t>(m->dev.size());
    if (transport_peer) *transport_peer = m->eng[0]->peer_transport() ? 1 : 0;
  });
}

// grads_dev[w]: worker w's gradient on device dev[w / (P / ndev)]
EXPORT int spardl_mctx_allreduce(spardl_mctx* m, const float* const* grads_dev) {
  return guarded([&] {
    need(m, "mctx");
    need(grads_dev, "grads");
    for (size_t i = 0; i < m->eng.size(); ++i)
      m->eng[i]->run(grads_dev + i * static_cast<size_t>(m->wloc));
  });
}

EXPORT int spardl_mctx_sync(spardl_mctx* m) {
  return guarded([&] {
    need(m, "mctx");
    for (auto& e : m->eng) e->sync();
  });
}

// host gradients in (worker order), the global sparse gradient out
EXPORT int spardl_mctx_allreduce_host(spardl_mctx* m, const float* const* grads_host,
                                      int64_t* g_idx, float* g_val, int64_t cap, int64_t* nnz) {
  return guarded([&] {
    need(m, "mctx");
    need(grads_host, "grads");
    const size_t P = m->eng.size() * static_cast<size_t>(m->wloc);
    const size_t bytes = sizeof(float) * static_cast<size_t>(m->eng[0]->dimension());
    if (m->staging.empty())
      for (size_t w = 0; w < P; ++w) {
        CK(cudaSetDevice(m->dev[w / static_cast<size_t>(m->wloc)]));
        float* p = nullptr;
        CK(cudaMalloc(&p, bytes));
        m->staging.push_back(p);
      }
    for (size_t w = 0; w < P; ++w) {
      need(grads_host[w], "grads[w]");
      const auto& e = m->eng[w / static_cast<size_t>(m->wloc)];
      CK(cudaSetDevice(m->dev[w / static_cast<size_t>(m->wloc)]));
      CK(cudaMemcpyAsync(m->staging[w], grads_host[w], bytes, cudaMemcpyHostToDevice, e->stream()));
    }
    std::vector<const float*> sp(m->staging.begin(), m->staging.end());
    for (size_t i = 0; i < m->eng.size(); ++i)
      m->eng[i]->run(sp.data() + i * static_cast<size_t>(m->wloc));
    for (auto& e : m->eng) e->sync();
    const int32_t* di = nullptr;
    const float* dv = nullptr;
    int64_t n = 0;
    m->eng[0]->global(0, &di, &dv, &n);
    *nnz = n;
    if (g_idx && g_val) {
      if (cap < n) sdlh::fail(SPARDL_E_ARG, "output capacity below the global nnz");
      std::vector<int32_t> tmp(static_cast<size_t>(n));
      CK(cudaSetDevice(m->dev[0]));
      CK(cudaMemcpy(tmp.data(), di, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(g_val, dv, sizeof(float) * n, cudaMemcpyDeviceToHost));
      for (int64_t q = 0; q < n; ++q) g_idx[q] = tmp[static_cast<size_t>(q)];
    }
  });
}

EXPORT int spardl_mctx_get_run_info(spardl_mctx* m, spardl_run_info* out) {
  return guarded([&] {
    need(m, "mctx");
    need(out, "out");
    std::vector<spardl_run_info> ri(m->eng.size());
    each_engine(*m, [&](int i) { ri[static_cast<size_t>(i)] = m->eng[static_cast<size_t>(i)]->run_info(); });
    *out = ri[0];
  });
}

EXPORT int spardl_mctx_get_ledger(spardl_mctx* m, int64_t* rounds, int64_t* scalars) {
  return guarded([&] {
    need(m, "mctx");
    const size_t P = m->eng.size() * static_cast<size_t>(m->wloc);
    std::vector<std::vector<int64_t>> r(m->eng.size(), std::vector<int64_t>(P)),
        sc(m->eng.size(), std::vector<int64_t>(P));
    each_engine(*m, [&](int i) {
      m->eng[static_cast<size_t>(i)]->ledger(r[static_cast<size_t>(i)].data(),
                                             sc[static_cast<size_t>(i)].data());
    });
    std::copy(r[0].begin(), r[0].end(), rounds);
    std::copy(sc[0].begin(), sc[0].end(), scalars);
  });
}

EXPORT int spardl_mctx_get_union_sizes(spardl_mctx* m, int64_t* out) {
  return guarded([&] {
    need(m, "mctx");
    const size_t n = static_cast<size_t>(m->eng.size() * m->wloc);   // >= m
    std::vector<std::vector<int64_t>> u(m->eng.size(), std::vector<int64_t>(n, 0));
    each_engine(*m, [&](int i) { m->eng[static_cast<size_t>(i)]->union_sizes(u[static_cast<size_t>(i)].data()); });
    std::copy(u[0].begin(), u[0].end(), out);
  });
}

// the global sparse gradient as held by worker w (host copy)
EXPORT int spardl_mctx_get_global(spardl_mctx* m, int32_t worker, int64_t* g_idx, float* g_val,
                                  int64_t cap, int64_t* nnz) {
  return guarded([&] {
    need(m, "mctx");
    const int i = worker / m->wloc;
    if (worker < 0 || i >= static_cast<int>(m->eng.size())) sdlh::fail(SPARDL_E_ARG, "worker out of range");
    CK(cudaSetDevice(m->dev[static_cast<size_t>(i)]));
    const int32_t* di = nullptr;
    const float* dv = nullptr;
    int64_t n = 0;
    m->eng[static_cast<size_t>(i)]->global(worker % m->wloc, &di, &dv, &n);
    *nnz = n;
    if (g_idx && g_val) {
      if (cap < n) sdlh::fail(SPARDL_E_ARG, "output capacity below the global nnz");
      std::vector<int32_t> tmp(static_cast<size_t>(n));
      CK(cudaMemcpy(tmp.data(), di, sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
      CK(cudaMemcpy(g_val, dv, sizeof(float) * n, cudaMemcpyDeviceToHost));
      for (int64_t q = 0; q < n; ++q) g_idx[q] = tmp[static_cast<size_t>(q)];
    }
  });
}

EXPORT int spardl_mctx_carry_to_host(spardl_mctx* m, int32_t worker, float* host) {
  return guarded([&] {
    need(m, "mctx");
    need(host, "host");
    const int i = worker / m->wloc;
    if (worker < 0 || i >= static_cast<int>(m->eng.size())) sdlh::fail(SPARDL_E_ARG, "worker out of range");
    auto& e = *m->eng[static_cast<size_t>(i)];
    CK(cudaSetDevice(m->dev[static_cast<size_t>(i)]));
    e.sync();
    CK(cudaMemcpy(host, e.carry(worker % m->wloc), sizeof(float) * e.dimension(),
                  cudaMemcpyDeviceToHost));
  });
}

EXPORT int spardl_mctx_carry_from_host(spardl_mctx* m, int32_t worker, const float* host) {
  return guarded([&] {
    need(m, "mctx");
    need(host, "host");
    const int i = worker / m->wloc;
    if (worker < 0 || i >= static_cast<int>(m->eng.size())) sdlh::fail(SPARDL_E_ARG, "worker out of range");
    auto& e = *m->eng[static_cast<size_t>(i)];
    CK(cudaSetDevice(m->dev[static_cast<size_t>(i)]));
    e.sync();
    CK(cudaMemcpy(e.carry(worker % m->wloc), host, sizeof(float) * e.dimension(),
                  cudaMemcpyHostToDevice));
  });
}

EXPORT int spardl_mctx_set_controller(spardl_mctx* m, int32_t worker, const spardl_hctrl* c) {
  return guarded([&] {
    need(m, "mctx");
    need(c, "controller");
    const int i = worker / m->wloc;
    if (worker < 0 || i >= static_cast<int>(m->eng.size())) sdlh::fail(SPARDL_E_ARG, "worker out of range");
    CK(cudaSetDevice(m->dev[static_cast<size_t>(i)]));
    m->eng[static_cast<size_t>(i)]->set_controller(worker % m->wloc, *c);
  });
}

EXPORT int spardl_mctx_get_controller(spardl_mctx* m, int32_t worker, spardl_hctrl* c) {
  return guarded([&] {
    need(m, "mctx");
    need(c, "controller");
    const int i = worker / m->wloc;
    if (worker < 0 || i >= static_cast<int>(m->eng.size())) sdlh::fail(SPARDL_E_ARG, "worker out of range");
    CK(cudaSetDevice(m->dev[static_cast<size_t>(i)]));
    m->eng[static_cast<size_t>(i)]->controller(worker % m->wloc, c);
  });
}

EXPORT int spardl_mctx_reset_state(spardl_mctx* m) {
  return guarded([&] {
    need(m, "mctx");
    for (size_t i = 0; i < m->eng.size(); ++i) {
      CK(cudaSetDevice(m->dev[i]));
      m->eng[i]->reset_state();
    }
  });
}
