// filter.cuh — the append-only threshold filter of the two-pass main pass
// (DESIGN.md §5 "Two-pass candidate selection"; operator fusion of cdist and
// topk), shared by the single-SM (knn_tc3.cu) and CTA-pair
// (knn_tc4.cu) kernels.
//
// One filter warp owns 32 query rows (its TMEM lane quarter) and a part of
// BH columns of every tile.  Each 8-column group's minimum w~ that is below the
// row's threshold tau is appended, as (key, group index), to the lane's pending
// run in shared memory.  Appends are rare (C3: ~0.7 % of the (row, 64-column
// part) pairs), so the part minimum is tested first with one warp vote and the
// per-group compares run only when some lane of the warp has a candidate.
#pragma once
#include "ptx.cuh"

namespace tod {

constexpr int kPendRun = 16;          // pending slots per lane (flush checked every 8 groups)
constexpr uint32_t kPendSlot = 32 * 8;  // bytes between a lane's consecutive pending slots

__device__ __forceinline__ float min8(const float* v) {
  return fminf(fminf(fminf(v[0], v[1]), v[2]),
               fminf(fminf(v[3], v[4]), fminf(fminf(v[5], v[6]), v[7])));
}

// v: this lane's BH accumulators of the tile (masked); gbase: global index of
// the part's first group.  `flush` moves the pending run to HBM.
// vote: test the part minimum first (worth it when appends are rare: large n;
// at n = 1e5 most warps hold a candidate in most parts and the test only adds work).
// COL: append each COLUMN below tau of the groups whose minimum is below it, as
// (w~, column index), instead of (group minimum, group index): the re-rank then
// evaluates only those columns (DESIGN.md §5 "Column candidates"); every column
// not appended still has w~ >= tau, so the certificate is unchanged.  Used with
// the vote (rare appends).  In this mode the caller has NOT released the
// accumulator yet: it is released here right after the vote when no lane has a
// candidate (the common case), else after the passing groups' columns are re-read
// from TMEM (reload(gg, c8): a warp-collective tcgen05.ld of the group's 8
// columns, masked as v was) and appended -- so v, like in the group mode, dies
// with the min tree and the filter keeps its register budget.
template <int BH, bool COL, class Flush, class Reload, class Release>
__device__ __forceinline__ void filter_part(const float* v, float tau, int gbase, uint32_t& pa,
                                            uint32_t pbase, bool vote, Flush&& flush,
                                            Reload&& reload, Release&& release) {
  float m[BH / 8];
#pragma unroll
  for (int g = 0; g < BH / 8; ++g) m[g] = min8(v + 8 * g);
  if (vote || COL) {
    float pm = m[0];
#pragma unroll
    for (int g = 1; g + 1 < BH / 8; g += 2) pm = fminf(pm, fminf(m[g], m[g + 1]));
    if constexpr ((BH / 8) % 2 == 0) pm = fminf(pm, m[BH / 8 - 1]);
    if (!__any_sync(0xffffffffu, pm < tau)) {
      if constexpr (COL) release();
      return;
    }
  }
  static_assert(BH % 8 == 0, "parts hold whole 8-column groups");
  if constexpr (COL) {
#pragma unroll 1
    for (int gg = 0; gg < BH / 8; ++gg) {
      if (!__any_sync(0xffffffffu, m[gg] < tau)) continue;
      if (__any_sync(0xffffffffu, pa > pbase + (kPendRun - 8) * kPendSlot)) flush();
      float c8[8];
      reload(gg, c8);  // warp-collective
      if (m[gg] < tau) {
#pragma unroll
        for (int e = 0; e < 8; ++e)
          if (c8[e] < tau) {
            sts_kv(pa, c8[e], (gbase + gg) * 8 + e);
            pa += kPendSlot;
          }
      }
    }
    release();
    return;
  }
#pragma unroll
  for (int g0 = 0; g0 < BH / 8; g0 += 8) {
    if (__any_sync(0xffffffffu, pa > pbase + (kPendRun - 8) * kPendSlot)) flush();
#pragma unroll
    for (int gg = g0; gg < g0 + 8 && gg < BH / 8; ++gg) {
      if (m[gg] < tau) {
        sts_kv(pa, m[gg], gbase + gg);
        pa += kPendSlot;
      }
    }
  }
}

// Tiles of reference chunk c of S: [bt*c/S, bt*(c+1)/S), minus the sample tiles
// (t % R == 0; R a power of two, 0 = none) when SKIP; the sample pass (SMP)
// visits only the sample tiles t = si*R, si in [bs*c/S, bs*(c+1)/S).  (A
// staggered per-CTA start was measured no faster: CTAs sweeping one L2-resident
// chunk in lockstep share its tiles.)
template <int SMP, int SKIP>
struct TileSeq {
  int t, end, R, mask;
  bool on;
  __device__ __forceinline__ void begin(int64_t bt, int S, int R_, int c) {
    R = R_;
    on = SKIP && R > 0;
    mask = R - 1;
    if constexpr (SMP) {
      const int64_t bs = (bt + R - 1) / R;
      t = (int)(bs * c / S) * R;
      end = (int)(bs * (c + 1) / S) * R;
      if (end > bt) end = (int)bt;
      return;
    }
    t = (int)(bt * c / S);
    end = (int)(bt * (c + 1) / S);
    skip();
  }
  __device__ __forceinline__ void skip() {
    if (on && (t & mask) == 0) ++t;
  }
  __device__ __forceinline__ bool more() const { return t < end; }
  __device__ __forceinline__ void next() {
    if constexpr (SMP) {
      t += R;
      return;
    }
    ++t;
    skip();
  }
};

// Runtime-mode tile sequence of chunk c of S over bt tiles (no rotation):
// smode 0: every tile, minus the sample tiles t % R == 0 when R > 0 (R a power
// of two); smode 1: only the sample tiles t = si * R, si in [bs*c/S, bs*(c+1)/S).
struct TileSeqRT {
  int t, end, step, mask;
  bool skip_on;
  __device__ __forceinline__ void begin(int64_t bt, int S, int R, int c, int smode) {
    if (smode) {
      const int64_t bs = (bt + R - 1) / R;
      t = (int)(bs * c / S) * R;
      end = (int)(bs * (c + 1) / S) * R;
      if (end > bt) end = (int)bt;
      step = R;
      skip_on = false;
    } else {
      t = (int)(bt * c / S);
      end = (int)(bt * (c + 1) / S);
      step = 1;
      skip_on = R > 0;
    }
    mask = R - 1;
    skip();
  }
  __device__ __forceinline__ void skip() {
    if (skip_on && (t & mask) == 0) ++t;
  }
  __device__ __forceinline__ bool more() const { return t < end; }
  __device__ __forceinline__ void next() {
    t += step;
    skip();
  }
};

}  // namespace tod
