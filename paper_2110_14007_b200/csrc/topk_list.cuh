// topk_list.cuh — per-row running top-K' (K' smallest keys with their column
// indices) kept by ONE thread for ONE query row, inside the fused distance
// epilogue.  This is the "topk on each cdist batch, local candidates merged so
// the result is still exact" of operator fusion (§6.1),
// re-derived for a thread-per-row TMEM/register layout.
//
// Storage: shared memory, column-per-thread: slot e of thread t is the 8-byte
// (key, index) pair at base + (e*NT + t)*8, so 32 lanes touching their own
// slots (any e per lane) hit distinct bank pairs (the slot stride NT*8 bytes
// is a multiple of 256).
//   slots [0, kp)          the kept list, sorted ascending by key
//   slots [kp, kp+P)       an append-only pending buffer
// The fast path compares keys against `thr` (the current K'-th smallest key,
// +inf while the list is not full); hits are appended with one predicated
// 64-bit store.  When any lane's pending buffer might overflow, the warp
// merges in lock step: bitonic sort of the pending entries in registers, then
// an in-place backward merge into the sorted list, truncated at kp.
//
// Invariant used by the certificate: every column
// offered to a row and not in its final list has key >= v, where v is the final
// thr (the K'-th kept key, or +inf when fewer than K' were ever offered).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include <math_constants.h>

#include "ptx.cuh"

namespace tod {

constexpr int kPendGroup = 8;   // appends per group between overflow checks

// Merge one row's pending buffer into its sorted list.  `base` is the shared
// address of this thread's slot 0.  Returns (new fill as int bits, new thr).
// __noinline__ with scalar arguments so the caller's state stays in registers.
template <int NT, int kPend>
__device__ __noinline__ float2 merge_row(uint32_t base, int kp, int fill, int pcnt) {
  constexpr uint32_t S = NT * 8;  // byte stride between slots
  if (pcnt == 0) {
    const float t = (fill == kp) ? lds_kv(base + (kp - 1) * S).x : CUDART_INF_F;
    return make_float2(__int_as_float(fill), t);
  }
  const uint32_t pb = base + kp * S;
  // the bitonic network needs a power-of-two width: pad with +inf
  constexpr int NP = kPend <= 8 ? 8 : (kPend <= 16 ? 16 : (kPend <= 32 ? 32 : 64));
  float pv[NP];
  int pi[NP];
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    const bool live = p < kPend && p < pcnt;
    const float2 e = live ? lds_kv(pb + p * S) : make_float2(CUDART_INF_F, __int_as_float(-1));
    pv[p] = e.x;
    pi[p] = __float_as_int(e.y);
  }
  // Bitonic sort ascending (fully unrolled: stays in registers).
#pragma unroll
  for (int k = 2; k <= NP; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
#pragma unroll
      for (int i = 0; i < NP; ++i) {
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
  for (int p = 0; p < kPend; ++p)
    if (p < pcnt) sts_kv(pb + p * S, pv[p], pi[p]);
  static_assert(NP >= kPend, "network narrower than the pending run");
  // Backward in-place merge of list[0,fill) and pending[0,pcnt) (both
  // ascending) into list[0, min(fill+pcnt, kp)).  Once the pending run is
  // exhausted the remaining list prefix is already in place (o == i).
  int i = fill - 1, j = pcnt - 1;
  int o = fill + pcnt - 1;
  float2 L = i >= 0 ? lds_kv(base + i * S) : make_float2(-CUDART_INF_F, 0.f);
  float2 P = lds_kv(pb + j * S);
  while (j >= 0) {
    const bool takeL = (i >= 0) && (L.x > P.x);
    if (o < kp) {
      const float2 t = takeL ? L : P;
      sts_kv(base + o * S, t.x, __float_as_int(t.y));
    }
    if (takeL) {
      --i;
      if (i >= 0) L = lds_kv(base + i * S);
    } else {
      --j;
      if (j >= 0) P = lds_kv(pb + j * S);
    }
    --o;
  }
  fill = min(fill + pcnt, kp);
  const float t = (fill == kp) ? lds_kv(base + (kp - 1) * S).x : CUDART_INF_F;
  return make_float2(__int_as_float(fill), t);
}

// Register-network merge for short lists (kp <= 32, P <= 32): load the sorted
// list and the pending run into registers, bitonic-sort the pending run, take
// the lower half of a half-cleaner between the list and the reversed pending
// run (= the 32 smallest, bitonic) and sort it with five merge stages.  No
// dependent shared-memory chains: ~350 compare-exchanges with full ILP.
template <int NT, int kPend, int W>
__device__ __noinline__ float2 merge_row_net(uint32_t base, int kp, int fill, int pcnt) {
  constexpr uint32_t S = NT * 8;
  static_assert(kPend <= W, "pending run longer than the network");
  if (pcnt == 0) {
    const float t = (fill == kp) ? lds_kv(base + (kp - 1) * S).x : CUDART_INF_F;
    return make_float2(__int_as_float(fill), t);
  }
  float lk[W], pk[W];
  int li[W], pi[W];
#pragma unroll
  for (int e = 0; e < W; ++e) {
    const bool liv = e < fill;
    const float2 a = liv ? lds_kv(base + e * S) : make_float2(CUDART_INF_F, __int_as_float(-1));
    lk[e] = a.x;
    li[e] = __float_as_int(a.y);
    const bool piv = e < kPend && e < pcnt;
    const float2 b = piv ? lds_kv(base + (kp + e) * S) : make_float2(CUDART_INF_F, __int_as_float(-1));
    pk[e] = b.x;
    pi[e] = __float_as_int(b.y);
  }
  auto cas = [](float& ka, int& ia, float& kb, int& ib, bool up) {
    const bool sw = up ? (ka > kb) : (ka < kb);
    const float tk = ka;
    const int ti = ia;
    ka = sw ? kb : ka;
    ia = sw ? ib : ia;
    kb = sw ? tk : kb;
    ib = sw ? ti : ib;
  };
#pragma unroll
  for (int k = 2; k <= W; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
      for (int i = 0; i < W; ++i) {
        const int l = i ^ j;
        if (l > i) cas(pk[i], pi[i], pk[l], pi[l], (i & k) == 0);
      }
  // half-cleaner: lower half = elementwise min of list and reversed pending
#pragma unroll
  for (int i = 0; i < W; ++i) {
    const bool take = pk[W - 1 - i] < lk[i];
    lk[i] = take ? pk[W - 1 - i] : lk[i];
    li[i] = take ? pi[W - 1 - i] : li[i];
  }
#pragma unroll
  for (int j = W >> 1; j > 0; j >>= 1)
#pragma unroll
    for (int i = 0; i < W; ++i) {
      const int l = i ^ j;
      if (l > i) cas(lk[i], li[i], lk[l], li[l], true);
    }
  fill = min(fill + pcnt, kp);
  float t = CUDART_INF_F;
#pragma unroll
  for (int e = 0; e < W; ++e) {
    if (e < fill) sts_kv(base + e * S, lk[e], li[e]);
    t = (e == kp - 1 && fill == kp) ? lk[e] : t;
  }
  return make_float2(__int_as_float(fill), t);
}

// NT: rows (threads) sharing the slot array; P: pending slots per row.
template <int NT, int P = 32>
struct RowTopK {
  static constexpr int kPend = P;
  static constexpr uint32_t S = NT * 8;
  uint32_t base;  // shared address of slot 0 of this thread
  uint32_t pa;    // shared address of the next pending slot
  int kp;
  int fill;
  float thr;

  // `pairs` is the [(kp + kPend) * NT] array of 8-byte (key, index) pairs.
  __device__ __forceinline__ void init(uint2* pairs, int t, int kprime) {
    base = smem_u32(pairs + t);
    kp = kprime;
    reset();
  }
  __device__ __forceinline__ void reset() {
    fill = 0;
    pa = base + kp * S;
    thr = CUDART_INF_F;
  }
  __device__ __forceinline__ int pcnt() const { return (int)((pa - base) / S) - kp; }
  __device__ __forceinline__ void append(float v, int j) {
    sts_kv(pa, v, j);
    pa += S;
  }
  // Whole warp must call (lanes with no pending entries are no-ops).
  __device__ __forceinline__ void merge() {
    float2 r;
    if (P <= 16 && kp <= 16)
      r = merge_row_net<NT, (P <= 16 ? P : 16), 16>(base, kp, fill, pcnt());
    else if (P <= 32 && kp <= 32)
      r = merge_row_net<NT, (P <= 32 ? P : 32), 32>(base, kp, fill, pcnt());
    else
      r = merge_row<NT, P>(base, kp, fill, pcnt());
    fill = __float_as_int(r.x);
    thr = r.y;
    pa = base + kp * S;
  }
  // Make room for up to kPendGroup appends.  Whole warp, uniform control flow.
  __device__ __forceinline__ void reserve_group() { reserve(kPendGroup); }
  // Make room for up to `r` appends.  Whole warp, uniform control flow.
  __device__ __forceinline__ void reserve(int r) {
    const uint32_t limit = base + (kp + kPend - r) * S;
    if (__any_sync(0xffffffffu, pa > limit)) merge();
  }
  // Predicated append (branch-free in SASS).
  __device__ __forceinline__ void append_if(bool p, float v, int j) {
    if (p) append(v, j);
  }
  // Offer up to kPendGroup (key, column) pairs: keys below thr and columns !=
  // self are appended (predicated stores, no branches on the data).
  __device__ __forceinline__ void offer_group(const float (&w)[kPendGroup], int col0, int self) {
#pragma unroll
    for (int e = 0; e < kPendGroup; ++e)
      if (w[e] < thr && col0 + e != self) append(w[e], col0 + e);
  }
  // Flush pending and write the list: out_idx[0..kp) (-1 for empty slots);
  // returns v (the certificate threshold).  Whole warp must call.
  __device__ __forceinline__ float finish(int* out_idx, bool write, float* out_key = nullptr) {
    if (__any_sync(0xffffffffu, pa != base + kp * S)) merge();
    if (write) {
      for (int e = 0; e < kp; ++e) {
        const float2 kv = e < fill ? lds_kv(base + e * S) : make_float2(CUDART_INF_F, 0.f);
        out_idx[e] = e < fill ? __float_as_int(kv.y) : -1;
        if (out_key) out_key[e] = kv.x;
      }
    }
    return thr;
  }
};

}  // namespace tod
