// Host-side sizing and wiring of one dividing task (residual add + candidate
// pass) and of the select that consumes it, shared by the pipeline planner
// (engine.cpp) and the top_k_select_slice component entry point (abi.cpp).
#pragma once

#include <algorithm>
#include <cstdint>

#include "kernels.cuh"

namespace sdl {

// alloc(bytes) returns zeroed device memory that outlives the task.
template <class Alloc>
void div_plan(DivTask& dt, SelTask& t, int64_t lo, int64_t hi, int64_t budget, Alloc&& alloc) {
  const int64_t nb = hi - lo;
  const int64_t A = lo & ~int64_t(3);
  const int nch = static_cast<int>((hi - A + kChunk - 1) / kChunk);
  const double frac = static_cast<double>(budget) / static_cast<double>(nb > 0 ? nb : 1);
  // per-chunk candidate segment: ~8x the expected candidates of a chunk; the
  // select's work list holds up to 4 L candidates (the pre-threshold aims at
  // ~1.4-2.3 L) before the dense fallback takes over
  int cap = static_cast<int>(std::min<double>(kChunk, std::max(1024.0, 8.0 * kChunk * frac)));
  cap = (cap + kTile - 1) / kTile * kTile;
  // work-list tiles: as small as kTile while the list fits the select's
  // per-task work-item bound
  const int64_t cand_cap = std::min<int64_t>(nb, 4 * budget + 4096);
  int tile_len = kTile;
  int max_tiles;
  if (nch + 1 < kMaxSegPerTask) {
    while (nch + (cand_cap + tile_len - 1) / tile_len > kMaxSegPerTask) tile_len += kTile;
    max_tiles = nch + static_cast<int>((cand_cap + tile_len - 1) / tile_len);
  } else {
    // more chunks than the cluster select's work items (a block of > 64M
    // elements): the work list overflows (bit 2 of cand_bad: the cluster
    // select takes the dense path) and the wide select, which reads the
    // chunk segments directly, selects the candidates
    tile_len = kTile * 64;
    max_tiles = kMaxSegPerTask;
  }
  dt.huge = nch + 1 >= kMaxSegPerTask ? 1 : 0;
  dt.tile_len = tile_len;
  dt.lo = static_cast<int32_t>(lo);
  dt.hi = static_cast<int32_t>(hi);
  dt.nchunks = nch;
  dt.cap = cap;
  dt.budget = budget;
  dt.use_cand = frac <= 0.25 ? 1 : 0;
  const size_t ncand = dt.use_cand ? static_cast<size_t>(nch) * cap : 4;
  dt.cand_idx = static_cast<int32_t*>(alloc(sizeof(int32_t) * ncand));
  dt.cand_val = static_cast<float*>(alloc(sizeof(float) * ncand));
  dt.cand_cnt = static_cast<int32_t*>(alloc(sizeof(int32_t) * nch));
  dt.max_tiles = max_tiles;
  dt.tile_off = static_cast<int32_t*>(alloc(sizeof(int32_t) * max_tiles));
  dt.tile_cnt = static_cast<int32_t*>(alloc(sizeof(int32_t) * max_tiles));
  dt.ntiles = static_cast<int32_t*>(alloc(sizeof(int32_t)));
  t.nseg_dev = dt.ntiles;
  dt.cand_total = static_cast<int64_t*>(alloc(sizeof(int64_t)));
  dt.cand_bad = static_cast<int32_t*>(alloc(sizeof(int32_t)));
  dt.pre_key = static_cast<uint32_t*>(alloc(sizeof(uint32_t)));
  dt.samp_hist = static_cast<uint32_t*>(alloc(sizeof(uint32_t) * kSampBins));
  dt.hist = static_cast<DivHistory*>(alloc(sizeof(DivHistory)));
  // ~8 sampled chunks (65k elements) per block: ~650 expected top-L samples
  // at 1% density whatever the block size
  dt.sample_every = std::max(1, nch / 8);

  t.mode_from_cand = dt.use_cand;
  t.mode = dt.use_cand ? 0 : 1;   // no candidate path: a static dense select
  t.idx = dt.cand_idx;
  t.val = dt.cand_val;
  t.seg_off = dt.tile_off;
  t.seg_cnt = dt.tile_cnt;
  t.stride = tile_len;
  t.nseg = dt.use_cand ? max_tiles : 1;
  t.dbase = static_cast<int32_t>(lo);
  t.dn = static_cast<int32_t>(nb);
  t.cand_total = dt.cand_total;
  t.cand_bad = dt.cand_bad;
  t.div_hist = dt.use_cand ? dt.hist : nullptr;
  t.pre_key_dev = dt.pre_key;
  t.budget = budget;
  t.weight = 1.f;
}

}  // namespace sdl
