// topk_list.cuh — per-row running top-K' (K' smallest keys with their column
// indices) kept by ONE thread for ONE query row, inside the fused
// distance epilogue.  This is the "topk on each cdist batch, local candidates
// merged so the result is still exact" of operator fusion (§6.1,
// P:452-455), re-derived for a thread-per-row TMEM/register layout.
//
// Storage: shared memory, column-per-thread ([slot][NT] with NT threads), so a
// warp touching "its" slot e hits 32 consecutive words (conflict-free).
//   slots [0, kp)        the kept list, sorted ascending by key
//   slots [kp, kp+P)     an append-only pending buffer
// The fast path (per distance) is one compare against `thr` (the current
// K'-th smallest key, +inf while the list is not full).  Hits are appended to
// the pending buffer; when any lane of the warp fills its buffer the whole
// warp merges in lock step: bitonic-sort the P pending entries in registers,
// then an in-place backward merge into the sorted list, truncated at kp.
//
// Invariant used by the certificate: every column
// offered to a row and not in its final list has key >= v, where v = the final
// thr (the K'-th kept key, or +inf when fewer than K' were ever offered).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <math_constants.h>

namespace tod {

constexpr int kPend = 16;  // P: pending slots per row

// Merge one row's pending buffer into its sorted list (see header comment).
// Returns (new fill, new thr).  A free __noinline__ function with scalar
// arguments so that the caller's RowTopK state stays in registers.
template <int NT>
__device__ __noinline__ float2 merge_row(float* lv, int* li, int kp, int fill, int pcnt) {
  if (pcnt == 0) {
    const float t = (fill == kp) ? lv[(kp - 1) * NT] : CUDART_INF_F;
    return make_float2(__int_as_float(fill), t);
  }
  float pv[kPend];
  int pi[kPend];
#pragma unroll
  for (int p = 0; p < kPend; ++p) {
    const bool live = p < pcnt;
    pv[p] = live ? lv[(kp + p) * NT] : CUDART_INF_F;
    pi[p] = live ? li[(kp + p) * NT] : -1;
  }
  // Bitonic sort ascending (fully unrolled: stays in registers).
#pragma unroll
  for (int k = 2; k <= kPend; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
#pragma unroll
      for (int i = 0; i < kPend; ++i) {
        const int l = i ^ j;
        if (l > i) {
          const bool up = (i & k) == 0;
          const bool sw = up ? (pv[i] > pv[l]) : (pv[i] < pv[l]);
          const float tv = pv[i];
          const int ti = pi[i];
          pv[i] = sw ? pv[l] : pv[i];
          pi[i] = sw ? pi[l] : pi[i];
          pv[l] = sw ? tv : pv[l];
          pi[l] = sw ? ti : pi[l];
        }
      }
    }
  }
#pragma unroll
  for (int p = 0; p < kPend; ++p) {
    if (p < pcnt) {
      lv[(kp + p) * NT] = pv[p];
      li[(kp + p) * NT] = pi[p];
    }
  }
  // Backward in-place merge of list[0,fill) and pending[0,pcnt) (both
  // ascending) into list[0, min(fill+pcnt, kp)).  Once the pending run is
  // exhausted the remaining list prefix is already in place (o == i).
  int i = fill - 1, j = pcnt - 1;
  int o = fill + pcnt - 1;
  float Lv = i >= 0 ? lv[i * NT] : -CUDART_INF_F;
  int Li = i >= 0 ? li[i * NT] : -1;
  float Pv = lv[(kp + j) * NT];
  int Pi = li[(kp + j) * NT];
  while (j >= 0) {
    const bool takeL = (i >= 0) && (Lv > Pv);
    if (o < kp) {
      lv[o * NT] = takeL ? Lv : Pv;
      li[o * NT] = takeL ? Li : Pi;
    }
    if (takeL) {
      --i;
      if (i >= 0) {
        Lv = lv[i * NT];
        Li = li[i * NT];
      }
    } else {
      --j;
      if (j >= 0) {
        Pv = lv[(kp + j) * NT];
        Pi = li[(kp + j) * NT];
      }
    }
    --o;
  }
  fill = min(fill + pcnt, kp);
  const float t = (fill == kp) ? lv[(kp - 1) * NT] : CUDART_INF_F;
  return make_float2(__int_as_float(fill), t);
}

template <int NT>
struct RowTopK {
  float* lv;  // &vals[0][t]
  int* li;    // &idx[0][t]
  int kp;
  int fill;
  int pcnt;
  float thr;

  __device__ __forceinline__ void init(float* vals, int* idxs, int t, int kprime) {
    lv = vals + t;
    li = idxs + t;
    kp = kprime;
    fill = 0;
    pcnt = 0;
    thr = CUDART_INF_F;
  }
  __device__ __forceinline__ void reset() {
    fill = 0;
    pcnt = 0;
    thr = CUDART_INF_F;
  }
  __device__ __forceinline__ void append(float v, int j) {
    lv[(kp + pcnt) * NT] = v;
    li[(kp + pcnt) * NT] = j;
    ++pcnt;
  }

  // Whole warp must call (lanes with pcnt == 0 participate as no-ops).
  __device__ __forceinline__ void merge() {
    const float2 r = merge_row<NT>(lv, li, kp, fill, pcnt);
    fill = __float_as_int(r.x);
    thr = r.y;
    pcnt = 0;
  }

  // Offer (key, column) unless column == self; merge when any lane is full.
  // Whole warp must call with uniform control flow.
  __device__ __forceinline__ void offer(float key, int col, int self) {
    if (key < thr && col != self) append(key, col);
    if (__any_sync(0xffffffffu, pcnt == kPend)) merge();
  }

  // Flush pending and write the list: out_idx[0..kp) (-1 for empty slots) and
  // returns v (the certificate threshold).  Whole warp must call.
  __device__ __forceinline__ float finish(int* out_idx, bool write) {
    if (__any_sync(0xffffffffu, pcnt > 0)) merge();
    if (write) {
      for (int e = 0; e < kp; ++e) out_idx[e] = e < fill ? li[e * NT] : -1;
    }
    return thr;
  }
};

}  // namespace tod
