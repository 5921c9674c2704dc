// rerank.cu — K3 re-rank + certificate (provable quantization step (iii),
// "verification", §5.2) and K4 fallback ("recalculate ...
// only on the subset of X where the verification fails").
//
// K3, one warp per query row: the K' (x lists) candidates of pass 1 are
// re-ranked with the EXACT fp64 distance of the oracle's definition
// (O1: sequential sum over c of fl64(x_ic - x_jc)^2, explicit
// __dsub_rn/__dmul_rn/__dadd_rn so nvcc cannot contract to FMA), sorted by
// (D64, index) (reading A4).  The row is CERTIFIED when the k-th re-ranked
// distance is strictly below a rigorous lower bound on the exact distance of
// every candidate pass 1 did not keep; then the
// oracle's top-k lies inside the kept set and the output is exact, indices
// bit-identical.  Uncertified rows are queued for K4.
//
// K4, one block per failing row: fp64 brute force over all references with
// the same formula, per-thread sorted top-k lists, block k-way merge.
#include <math_constants.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>

#include <cuda_fp16.h>

#include "internal.h"

namespace tod {

namespace {

constexpr int kRerankWarps = 8;
constexpr int kMaxCands = 256;   // lists * K' per row
constexpr int kMaxK = 128;

// O1, bit-identical to the oracle (no FMA, ascending c, from +0.0).
__device__ __forceinline__ double d64_row(const float* __restrict__ a, const float* __restrict__ b,
                                          int d) {
  double acc = 0.0;
  for (int c = 0; c < d; ++c) {
    const double t = __dsub_rn((double)a[c], (double)b[c]);
    acc = __dadd_rn(acc, __dmul_rn(t, t));
  }
  return acc;
}

__device__ __forceinline__ bool key_less(double ka, int ia, double kb, int ib) {
  return ka < kb || (ka == kb && ia < ib);
}

// gamma_m(u) = m u / (1 - m u), rounded up generously.
__device__ __forceinline__ double gamma_up(double m, double u) {
  return (m * u) / (1.0 - m * u) * (1.0 + 1e-10);
}

// Tensor-core accumulation model (reading A9), valid for ANY internal
// order and width >= 24 bits: each tcgen05 K-step adds 17 addends (its 16 exact
// fp16/bf16 products and the fp32 accumulator).  Worst case, the hardware aligns
// all of them to the largest exponent and truncates each to 24 bits (error
// < 2^-23 |max| for each of the 16 non-maximal addends), then truncates the
// exact aligned sum S to fp32 (< 2^-23 |S|): per step < 17 * 2^-23 * sum|addends|.
// |acc| <= sum of the earlier |A B| (times 1 + tiny), so with T = ceil(K/16)
// steps, K = dpad + 16:
//   |w~ - w| <= 17 T 2^-23 (1 + 1e-3) sum_k |A_ik B_jk|.
// (Round 1 used a per-operation model, 5T + 2 roundings, which alignment
// truncation can exceed: ADVICE r01.)  Measured on B200 on the library's own
// kernels (tools/cert_check.py): see DESIGN.md A9.
__device__ __forceinline__ double acc_gamma(int dpad) {
  const double T = (double)((dpad + 16 + 15) / 16);
  return 17.0 * T * 1.1920928955078125e-07 /*2^-23*/ * (1.0 + 1e-3);
}

// Writes the k outputs of one row from ascending (key, id) arrays (fp64
// squared distances).  Lane-parallel over m; lane 0 does the sequential sums.
__device__ void write_row(const KnnOutDev& out, int64_t r, int k, const double* keys,
                          const int* ids, int lane, int nlanes) {
  // Called by one full warp (nlanes == 32).  Each square root is taken once,
  // by the lane that owns the rank; the mean is summed in rank order through
  // shuffles (the oracle's sequential order, O3).
  (void)nlanes;
  double acc = 0.0;
  for (int m0 = 0; m0 < k; m0 += 32) {
    const int m = m0 + lane;
    double dd = 0.0;
    if (m < k) {
      dd = __dsqrt_rn(keys[m]);
      if (out.idx) out.idx[r * k + m] = ids[m];
      if (out.dist64) out.dist64[r * k + m] = dd;
      if (out.dist) out.dist[r * k + m] = __double2float_rn(dd);
      if (m == k - 1) {
        if (out.kdist64) out.kdist64[r] = dd;
        if (out.score_kth) out.score_kth[r] = __double2float_rn(dd);
      }
    }
    if (out.score_mean) {
      const int cnt = k - m0 < 32 ? k - m0 : 32;
      for (int t = 0; t < cnt; ++t) acc = __dadd_rn(acc, __shfl_sync(0xffffffffu, dd, t));
    }
  }
  if (lane == 0 && out.score_mean) out.score_mean[r] = __double2float_rn(__ddiv_rn(acc, (double)k));
}

// Lower bound, in original units, on the exact squared distance rho^2 of row r
// to ANY reference column whose pass-1 key is >= w.  Returns a
// value <= 0 when no positive bound exists.  *err receives the pass-1 error
// term (diagnostics).
__device__ double lb2_from_key(const CertParams& cp, int64_t r, double w, double* err) {
  const double u53 = 1.1102230246251565e-16;
  if (cp.kind == PASS_TC) {
    // Tensor-core pass (fp16/bf16 operands, fp32 accumulation; the norm
    // ||xhat_j||^2 enters as pieces p_jq times constants c_q in an extra K
    // block).  With w_ij = ||xhat_j||^2 - 2 xhat_i.xhat_j exact: every product
    // is exact in fp32, so
    //   |w~_ij - w_ij| <= gamma_m(u) sum_k |A_ik B_jk| + rep_j
    //                  <= gamma (2 a_i a_max + 1.002 amax2) + repmax  =: E_i
    // (Cauchy-Schwarz on the dot part; sum_q |c_q p_jq| <= 1.002 ||xhat_j||^2).
    // A9: accumulation model acc_gamma (17 ceil(K/16) units of 2^-23: alignment truncation).
    // w~_ij >= w gives ||xhat_i - xhat_j||^2 >= a_i^2 + w - E_i; the residuals
    // e_i, e_j <= emax then bound the exact distance (triangle inequality).
    const double a2i = cp.qa2[r];
    const double ei = cp.qe[r];
    const double amax2 = cp.g->amax2;
    const double emax = cp.g->emax;
    const double rep = cp.g->repmax;
    const double ai = sqrt(a2i) * (1.0 + 4 * u53);
    const double am = sqrt(amax2) * (1.0 + 4 * u53);
    const double gam = acc_gamma(cp.dpad);
    const double E = (gam * (2.0 * ai * am + 1.002 * amax2) + rep) * (1.0 + 1e-6) + 1e-300;
    const double slack = (cp.d + 8) * 2.0 * u53 * (fabs(a2i) + fabs(w) + E);
    // (1) with a_j <= a_max:  R^2 = ||xhat_i - xhat_j||^2 = a_i^2 + w_ij >= a_i^2 + w - E
    const double R2 = a2i + w - E - slack;
    *err = E + slack;
    double Rh = R2 > 0.0 ? sqrt(R2) * (1.0 - 2.0 * u53) : 0.0;
    // (2) with a_j <= a_i + R (triangle inequality), the column's own error term
    //   E_ij <= gam (3.002 a_i^2 + 4.004 a_i R + 1.002 R^2) + rep
    // turns R^2 >= a_i^2 + w - E_ij into a quadratic in R:
    //   (1 + 1.002 gam) R^2 + 4.004 gam a_i R - C >= 0,  C = a_i^2 + w - 3.002 gam a_i^2 - rep,
    // so R >= 2C / (b + sqrt(b^2 + 4 a C)).  Much tighter than (1) when a_max is far
    // above a_i + R (outlying rows set a_max); the larger of the two bounds holds.
    {
      const double g2 = gam * (1.0 + 1e-6);
      const double qa = 1.0 + 1.002 * g2;
      const double qb = 4.004 * g2 * ai;
      const double C = a2i + w - 3.002 * g2 * a2i * (1.0 + 4.0 * u53) - rep * (1.0 + 1e-6) - slack;
      if (C > 0.0) {
        const double Rb = 2.0 * C / (qb + sqrt(qb * qb + 4.0 * qa * C) * (1.0 + 4.0 * u53)) *
                           (1.0 - 1e-12);
        Rh = fmax(Rh, Rb);
      }
    }
    if (!(Rh > 0.0)) return -1.0;
    const double LB = (Rh - ei - emax) * (1.0 - 8.0 * u53);
    if (!(LB > 0.0)) return -1.0;
    const double lbo = LB / cp.g->s;  // s = 2^e: exact
    return lbo * lbo * (1.0 - 8.0 * u53);
  }
  // fp32 difference-form pass: D~ <= rho^2 (1 + gamma_{d+2}(2^-24)) + tiny.
  const double g32 = gamma_up(cp.d + 2, 5.9604644775390625e-08);
  *err = w * g32;
  return (w - (cp.d + 2) * 1.1754943508222875e-38 /*2^-126*/) / (1.0 + g32) * (1.0 - 8.0 * u53);
}

// The certificate: true iff every reference the pass did not keep has oracle
// distance D64 > dk (the k-th re-ranked D64), so the oracle's top-k lies inside
// the kept set.  `vmin` is the key threshold below which pass 1 kept
// everything it was offered.  D64 >= rho^2 (1 - gamma_{d+2}(2^-53)).
__device__ bool row_certified(const CertParams& cp, int64_t r, float vmin, double dk, double* err) {
  if (vmin == CUDART_INF_F) return true;  // every reference was offered and kept
  const double lb2 = lb2_from_key(cp, r, (double)vmin, err);
  return lb2 > 0.0 && dk < lb2 * (1.0 - gamma_up(cp.d + 2, 1.1102230246251565e-16));
}

__global__ void __launch_bounds__(kRerankWarps * 32)
    k_rerank(const float* __restrict__ Q, int64_t q_begin, int64_t q_count,
             const float* __restrict__ X, int64_t n, int d, int k, int self_join,
             const int32_t* __restrict__ cand_idx, const float* __restrict__ cand_v, int kp, int S,
             CertParams cp, KnnOutDev out, int32_t* __restrict__ fail_rows,
             double* __restrict__ fail_ub, int32_t* __restrict__ fail_count,
             unsigned long long* __restrict__ max_err_bits) {
  __shared__ double s_key[kRerankWarps][kMaxCands];
  __shared__ int s_id[kRerankWarps][kMaxCands];
  __shared__ double s_sk[kRerankWarps][kMaxK];
  __shared__ int s_si[kRerankWarps][kMaxK];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * kRerankWarps + w;
  if (r >= q_count) return;
  const int64_t gi = q_begin + r;
  const float* xi = self_join ? X + gi * d : Q + r * d;
  const int C = S * kp;
  double* keys = s_key[w];
  int* ids = s_id[w];
  for (int e = lane; e < C; e += 32) {
    const int j = cand_idx[r * C + e];
    ids[e] = j;
    keys[e] = j >= 0 ? d64_row(xi, X + (int64_t)j * d, d) : CUDART_INF;
  }
  float vmin = CUDART_INF_F;
  for (int c = 0; c < S; ++c) vmin = fminf(vmin, cand_v[r * S + c]);
  __syncwarp();
  // Rank every valid candidate by (key, id); ids are distinct, so ranks are a
  // permutation of [0, nv).  Keep the first k.
  int nv_local = 0;
  for (int e = lane; e < C; e += 32) {
    const int ie = ids[e];
    if (ie < 0) continue;
    ++nv_local;
    const double ke = keys[e];
    int rank = 0;
    for (int f = 0; f < C; ++f) {
      const int jf = ids[f];
      rank += (jf >= 0) && key_less(keys[f], jf, ke, ie);
    }
    if (rank < k) {
      s_sk[w][rank] = ke;
      s_si[w][rank] = ie;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) nv_local += __shfl_xor_sync(0xffffffffu, nv_local, o);
  __syncwarp();
  double err = 0.0;
  bool cert = nv_local >= k && row_certified(cp, r, vmin, s_sk[w][k - 1], &err);
  if (cp.force_fail) cert = false;
  if (lane == 0 && err > 0.0 && (r & 31) == 0)  // sampled: same-address atomics serialise
    atomicMax(max_err_bits, (unsigned long long)__double_as_longlong(err));
  if (cert) {
    write_row(out, r, k, s_sk[w], s_si[w], lane, 32);
  } else if (lane == 0) {
    const int slot = atomicAdd(fail_count, 1);
    fail_rows[slot] = (int32_t)r;
    // the k-th exact distance among kept columns bounds the true k-th from above
    fail_ub[slot] = nv_local >= k ? s_sk[w][k - 1] : CUDART_INF;
  }
}


// ------------------------------------------------------- group candidates
// Tensor-core pass candidates are 8-column groups (list entries hold the
// group index g = column / 8 and the group's minimum w).  Every column of every
// kept group is re-ranked; columns outside kept groups have w~ >= v (their
// group's minimum is >= v), so the same certificate applies.
constexpr int kGrpWarps = 4;

// Per-row terms of the pass-1 bounds (tensor-core pass): a_i^2, e_i and the
// accumulation error E_i = gamma (2 a_i a_max + 1.002 a_max^2) + rep (lb2_from_key).
struct RowBound {
  double a2i, ei, E;
};
__device__ __forceinline__ RowBound row_bound(const CertParams& cp, int64_t r) {
  const double u53 = 1.1102230246251565e-16;
  RowBound b;
  b.a2i = cp.qa2[r];
  b.ei = cp.qe[r];
  const double amax2 = cp.g->amax2;
  const double ai = sqrt(b.a2i) * (1.0 + 4 * u53);
  const double am = sqrt(amax2) * (1.0 + 4 * u53);
  b.E = (acc_gamma(cp.dpad) * (2.0 * ai * am + 1.002 * amax2) + cp.g->repmax) * (1.0 + 1e-6) + 1e-300;
  return b;
}

// Upper bound, in original units, on the exact squared distance D64 of row r
// to the best column of a group whose pass-1 key is w (the group's minimum w~)
// and whose rows have residual bounds <= ej: that column has w_ij <= w + E_i, so
// ||xhat_i - xhat_j||^2 <= a_i^2 + w + E_i, and the residuals e_i, e_j bound the
// exact distance from above.  (Mirror image of lb2_from_key; tensor-core pass only.)
__device__ double ub2_key_e(const CertParams& cp, const RowBound& b, double w, double ej) {
  const double u53 = 1.1102230246251565e-16;
  const double slack = (cp.d + 8) * 2.0 * u53 * (fabs(b.a2i) + fabs(w) + b.E);
  double R2 = b.a2i + w + b.E + slack;
  if (!(R2 > 0.0)) R2 = 0.0;
  const double Rh = sqrt(R2) * (1.0 + 2.0 * u53);
  const double UB = (Rh + b.ei + ej) * (1.0 + 8.0 * u53);
  const double ubo = UB / cp.g->s;  // s = 2^e: exact
  return ubo * ubo * (1.0 + 8.0 * u53) * (1.0 + gamma_up(cp.d + 2, u53));
}
__device__ double ub2_from_key(const CertParams& cp, int64_t r, double w) {
  return ub2_key_e(cp, row_bound(cp, r), w, cp.g->emax);
}

// Key cut (DESIGN.md §5 "Re-rank"): the largest pass-1 key w (rounded up to
// fp32) for which lb2_from_key(w)(1-gamma) -- with the group's residual bound ej
// in place of e_max -- could still be <= UB.  lb2_from_key is increasing in w,
// so inverting it with every rounding pushed upward gives a cutoff above which a
// group provably holds no column at distance <= UB.  (A larger cutoff only
// visits more groups.)  Ts = cut_scaled(UB) is the row's part.
__device__ double cut_scaled(const CertParams& cp, double UB) {
  const double u53 = 1.1102230246251565e-16;
  const double g64 = gamma_up(cp.d + 2, u53);
  const double T = sqrt(UB / ((1.0 - 8.0 * u53) * (1.0 - g64))) * (1.0 + 4 * u53);
  return T * cp.g->s / (1.0 - 8.0 * u53);
}
__device__ float key_cut_e(const CertParams& cp, const RowBound& b, double Ts, double ej) {
  const double u53 = 1.1102230246251565e-16;
  const double Z = (Ts + b.ei + ej) * (1.0 + 4 * u53);
  const double Zr = Z / (1.0 - 2.0 * u53) * (1.0 + 4 * u53);
  const double w0 = Zr * Zr - b.a2i + b.E;
  const double slack = (cp.d + 8) * 2.0 * u53 * (fabs(b.a2i) + fabs(w0) + b.E);
  const double w = w0 + 2.0 * slack + 1e-9 * (fabs(b.a2i) + fabs(w0) + b.E);
  return __double2float_ru(w);
}
__device__ float key_cut_from_ub(const CertParams& cp, int64_t r, double UB) {
  if (!(UB < CUDART_INF)) return CUDART_INF_F;
  return key_cut_e(cp, row_bound(cp, r), cut_scaled(cp, UB), cp.g->emax);
}

// Group candidates (DESIGN.md §5 "Re-rank").  A row's kept groups come from its
// pass-1 lists (idx/key, -1 = empty slot) and, in the two-pass mode, from the
// main pass's append buffers; they are staged unsorted in shared memory.
//  1. kappa = a key with >= k staged groups at or below it (bisection on the
//     ordered key bits); each of those groups holds a distinct column with
//     D64 <= UB := ub2_from_key(kappa), so the k-th exact distance is <= UB.
//  2. Only groups whose lower bound lb2_from_key(key)(1-gamma) <= UB can hold
//     a top-k column; they are expanded to their 8 columns and evaluated with
//     the oracle formula (O1); columns with D64 <= UB are kept.
//  3. The k smallest by (D64, index) are selected once: a warp bitonic sort
//     when <= 64 columns survive, else k rounds of warp argmin.
constexpr int kSelMax = 512;    // staged groups per row
constexpr int kColMax = 256;    // surviving columns per row

__device__ __forceinline__ uint32_t f2ord(float f) {  // order-preserving float -> uint
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float ord2f(uint32_t o) {
  return __uint_as_float((o & 0x80000000u) ? (o & 0x7FFFFFFFu) : ~o);
}

// Warp bitonic sort of 32 (key, id) pairs, one per lane, ascending by (key, id).
__device__ __forceinline__ void warp_sort32(double& key, int& id, int lane) {
#pragma unroll
  for (int kk = 2; kk <= 32; kk <<= 1) {
#pragma unroll
    for (int j = kk >> 1; j > 0; j >>= 1) {
      const double ok = __shfl_xor_sync(0xffffffffu, key, j);
      const int oi = __shfl_xor_sync(0xffffffffu, id, j);
      const bool up = (lane & kk) == 0;
      const bool lower = (lane & j) == 0;
      const bool other_less = key_less(ok, oi, key, id);
      if ((lower == up) ? other_less : !other_less) {
        key = ok;
        id = oi;
      }
    }
  }
}

// Warp bitonic sort of 64 (key, id) pairs, 2 per lane (element p = 2*lane + e),
// ascending by (key, id); empty slots carry (+inf, INT32_MAX).
__device__ __forceinline__ void warp_sort64(double (&k)[2], int (&id)[2], int lane) {
#pragma unroll
  for (int kk = 2; kk <= 64; kk <<= 1) {
#pragma unroll
    for (int j = kk >> 1; j > 0; j >>= 1) {
      if (j == 1) {
        const int p = 2 * lane;
        const bool up = (p & kk) == 0;
        const bool sw = up ? key_less(k[1], id[1], k[0], id[0]) : key_less(k[0], id[0], k[1], id[1]);
        if (sw) {
          const double tk = k[0];
          const int ti = id[0];
          k[0] = k[1];
          id[0] = id[1];
          k[1] = tk;
          id[1] = ti;
        }
      } else {
        const int lm = j >> 1;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int p = 2 * lane + e;
          const double ok = __shfl_xor_sync(0xffffffffu, k[e], lm);
          const int oi = __shfl_xor_sync(0xffffffffu, id[e], lm);
          const bool up = (p & kk) == 0;
          const bool lower = (p & j) == 0;
          const bool other_less = key_less(ok, oi, k[e], id[e]);
          if ((lower == up) ? other_less : !other_less) {
            k[e] = ok;
            id[e] = oi;
          }
        }
      }
    }
  }
}

// A value h (ordered bits) with count(arr[e] <= h, e < G) >= k, at most ~64 ulps
// above the k-th smallest (bisection on the ordered key bits; G >= k).  Stopping
// within 64 ulps (relative 2^-17, far below the bounds' own slack) saves the last
// halvings; any h with count >= k gives a valid upper bound.
__device__ __forceinline__ uint32_t kth_from_above(const float* arr, int G, int k, int lane) {
  uint32_t lo = 0xFFFFFFFFu, hi = 0u;
  uint32_t ok[8];  // this lane's ordered keys (G <= 256), 0xFFFFFFFF = none
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int e = lane + 32 * u;
    ok[u] = (e < G) ? f2ord(arr[e]) : 0xFFFFFFFFu;
    if (e < G) {
      lo = min(lo, ok[u]);
      hi = max(hi, ok[u]);
    }
  }
  for (int e = lane + 256; e < G; e += 32) {
    const uint32_t o = f2ord(arr[e]);
    lo = min(lo, o);
    hi = max(hi, o);
  }
  lo = __reduce_min_sync(0xffffffffu, lo);
  hi = __reduce_max_sync(0xffffffffu, hi);
  if (lo < hi) --lo;  // count(key <= lo) < k unless lo is the minimum itself
  int chi = G;
  for (int it = 0; it < 32 && hi - lo > 64 && chi > k; ++it) {
    const uint32_t mid = lo + ((hi - lo) >> 1);
    int c = 0;
#pragma unroll
    for (int u = 0; u < 8; ++u) c += ok[u] <= mid;
    for (int e = lane + 256; e < G; e += 32) c += f2ord(arr[e]) <= mid;
    c = __reduce_add_sync(0xffffffffu, c);  // one REDUX instead of a 5-step shuffle tree
    if (c >= k) {
      hi = mid;
      chi = c;
    } else {
      lo = mid;
    }
  }
  return hi;
}

// Staged candidates are 8-column groups (list entries; main-pass appends in group
// mode) or single columns (main-pass appends in column mode, MainPass.colmode),
// told apart by bit 30 of the staged index (column mode needs n < 2^30).
constexpr int kColFlag = 1 << 30;

// Steps 1-2 of a row's re-rank (one warp; DESIGN.md §5 "Re-rank") over its G
// staged candidates (keys gk, tagged indices gid):
//  1. UB >= the k-th exact distance.  Each staged group holds a distinct column
//     with D64 <= ub (ub2_key_e with the candidate's residual bound: a column's
//     own e_j, a group's e_g = max over its rows, or e_max when those arrays are
//     null), so UB = the k-th smallest ub.  (With e_max everywhere the ub order is
//     the key order: UB = ub2_from_key(kappa), kappa the k-th key.)
//  2. Only candidates whose lower bound can be <= UB are visited (key_cut_e with
//     the same residual bound).
// The visited groups are compacted to visg[0, nvg) (visg may alias gid) and the
// visited columns to visc[i * cstride], i < nvc; the caller checks the counts
// against its capacities (entries beyond them are dropped).  gu: G floats of scratch
// (free again on return: visc may alias it).
__device__ __forceinline__ void plan_row(const CertParams& cp, int64_t r, int k, const float* gk,
                                         int* gid, float* gu, int G, int* visg, int capg, int* visc,
                                         int capc, int cstride, double& UB, int& nvg, int& nvc,
                                         int lane) {
  UB = CUDART_INF;
  const RowBound b = row_bound(cp, r);
  const double emax = cp.g->emax;
  auto ej_of = [&](int t) {
    if (t & kColFlag) return cp.ecol ? cp.ecol[t & (kColFlag - 1)] : emax;
    return cp.eg ? cp.eg[t] : emax;
  };
  const bool per_cand = cp.eg || (cp.colmode && cp.ecol);
  if (G >= k) {
    if (per_cand) {
      for (int e = lane; e < G; e += 32)
        gu[e] = __double2float_ru(ub2_key_e(cp, b, (double)gk[e], ej_of(gid[e])));
      __syncwarp();
      const float ubk = ord2f(kth_from_above(gu, G, k, lane));
      if (ubk < CUDART_INF_F) UB = (double)ubk;
    } else {
      const float kappa = ord2f(kth_from_above(gk, G, k, lane));
      if (kappa < CUDART_INF_F) UB = ub2_key_e(cp, b, (double)kappa, emax);
    }
  }
  __syncwarp();  // gu reads done (visc may alias it)
  const bool fin = UB < CUDART_INF;
  const double Ts = fin ? cut_scaled(cp, UB) : 0.0;
  const float kcut = fin ? key_cut_e(cp, b, Ts, emax) : CUDART_INF_F;
  nvg = 0;
  nvc = 0;
  for (int e0 = 0; e0 < G; e0 += 32) {
    const int e = e0 + lane;
    bool v = false;
    int t = 0;
    if (e < G) {
      t = gid[e];
      const float cut = (fin && per_cand) ? key_cut_e(cp, b, Ts, ej_of(t)) : kcut;
      v = gk[e] <= cut;
    }
    const bool col = (t & kColFlag) != 0;
    const unsigned vg = __ballot_sync(0xffffffffu, v && !col);
    const unsigned vc = __ballot_sync(0xffffffffu, v && col);
    const unsigned below = (1u << lane) - 1u;
    if (v && !col) {
      const int pos = nvg + __popc(vg & below);
      if (pos < capg) visg[pos] = t;
    }
    if (v && col) {
      const int pos = nvc + __popc(vc & below);
      if (pos < capc) visc[pos * cstride] = t & (kColFlag - 1);
    }
    nvg += __popc(vg);
    nvc += __popc(vc);
  }
  __syncwarp();
}

// 256-bit read-only global load (sm_100: LDG.E.ENL2.256); p must be 32-byte aligned.
__device__ __forceinline__ void ldg8(const float* p, float* v) {
  asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]), "=f"(v[4]), "=f"(v[5]),
                 "=f"(v[6]), "=f"(v[7])
               : "l"(p));
}

// O1 for a compile-time d (multiple of 8): the whole reference row in flight as
// 32-byte loads (full sectors), the query row read as 16-byte pairs of doubles
// (shared-memory broadcast); the sum stays sequential in c, no FMA.
template <int DT>
__device__ __forceinline__ double d64_fixed(const double* __restrict__ xq, const float* xj) {
  constexpr int CH = DT < 64 ? DT : 64;  // dims per chunk held in registers
  double acc = 0.0;
#pragma unroll 1
  for (int cb = 0; cb < DT; cb += CH) {
    float v[CH];
#pragma unroll
    for (int u = 0; u < CH / 8; ++u) ldg8(xj + cb + 8 * u, v + 8 * u);
#pragma unroll
    for (int c = 0; c < CH; c += 2) {
      const double2 q2 = *reinterpret_cast<const double2*>(xq + cb + c);
      double t = __dsub_rn(q2.x, (double)v[c]);
      acc = __dadd_rn(acc, __dmul_rn(t, t));
      t = __dsub_rn(q2.y, (double)v[c + 1]);
      acc = __dadd_rn(acc, __dmul_rn(t, t));
    }
  }
  return acc;
}

// ---- per-column pre-bound (DESIGN.md §5 "Re-rank"): before the exact O1 of a
// visited group's column j, a lower bound on its D64 from the 16-bit operand
// image alone -- R^ = ||xhat_i - xhat_j|| with both rows read from the image the
// tensor core multiplied (half the bytes of the fp32 row), then the residuals
// e_i, e_j, the scale and the oracle's own rounding exactly as in lb2_from_key.
// It drops the group bound's accumulation term E_i and uses the column's own
// distance instead of its group's minimum, so most columns of a visited group
// are excluded without gathering their fp32 rows.  Only a VALID lower bound is
// needed: a column is skipped iff the bound exceeds UB >= the k-th distance.
template <int FMT>
__device__ __forceinline__ float widen_img(uint32_t h) {
  if constexpr (FMT == 2) return __uint_as_float(h << 16);  // bf16: exact
  else return __half2float(__ushort_as_half((unsigned short)h));
}
// The 16-bit value of element c of image row r (swizzled K-major layout, prep.cu).
__device__ __forceinline__ uint32_t img_elem(const CertParams& cp, int64_t r, int c) {
  const int epr = cp.b_rb / 2;
  const uint32_t M = (uint32_t)(cp.b_rb / 16 - 1);
  const uint64_t o = (uint64_t)r * cp.b_rb + (uint64_t)(c % epr) * 2u;
  const uint64_t phys = o ^ (((o >> 7) & M) << 4);
  return *reinterpret_cast<const uint16_t*>(cp.bimg + (size_t)(c / epr) * cp.b_region + phys);
}
// The fp32 sum of (q - y)^2 over one image row, DP (= dpad) a compile-time
// constant: every 16-byte chunk load in flight at once, four independent partial
// sums (the bound below holds for any summation order of nonnegative terms).
template <int FMT, int DP>
__device__ __forceinline__ float img_dist2(const CertParams& cp, const float* qh, int64_t j) {
  constexpr int RB = DP * 2 < 128 ? DP * 2 : 128;
  constexpr int NREG = DP * 2 / RB;
  constexpr int CPR = RB / 16;
  const uint32_t x = (uint32_t)(((uint64_t)j * RB >> 7) & (uint64_t)(CPR - 1));
  uint4 v[NREG * CPR];
#pragma unroll
  for (int kb = 0; kb < NREG; ++kb) {
    const uint4* row = reinterpret_cast<const uint4*>(cp.bimg + (size_t)kb * cp.b_region +
                                                      (size_t)j * RB);
#pragma unroll
    for (int k = 0; k < CPR; ++k) v[kb * CPR + k] = __ldg(row + (k ^ x));
  }
  float a[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
  for (int k = 0; k < NREG * CPR; ++k) {
    const uint32_t w4[4] = {v[k].x, v[k].y, v[k].z, v[k].w};
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      const float d0 = qh[8 * k + 2 * t] - widen_img<FMT>(w4[t] & 0xFFFFu);
      const float d1 = qh[8 * k + 2 * t + 1] - widen_img<FMT>(w4[t] >> 16);
      a[t] = fmaf(d0, d0, a[t]);
      a[t] = fmaf(d1, d1, a[t]);
    }
  }
  return (a[0] + a[1]) + (a[2] + a[3]);
}

// Lower bound on D64(i, j) in original units (<= 0: none).  qh = xhat_i in fp32
// (shared), ei = e_i.  fp32 sum of dpad terms fl(fl(q - y)^2 + acc), all >= 0:
// acc <= Rhat^2 (1 + u)^2 (1 + gamma_dpad) <= Rhat^2 (1 + gamma_{dpad+3}) (+ underflow).
template <int FMT, int DP = 0>
__device__ __forceinline__ double lb2_col(const CertParams& cp, const float* qh, int64_t j,
                                          double ei) {
  const double u53 = 1.1102230246251565e-16;
  if constexpr (DP > 0) {
    const float acc = img_dist2<FMT, DP>(cp, qh, j);
    const double D = (double)acc / (1.0 + gamma_up(DP + 3, 5.9604644775390625e-08)) -
                     (DP + 3) * 1.1754943508222875e-38 /*2^-126*/;
    if (!(D > 0.0)) return -1.0;
    const double R = sqrt(D) * (1.0 - 2.0 * u53);
    const double LB = (R - ei - cp.ecol[j]) * (1.0 - 8.0 * u53);
    if (!(LB > 0.0)) return -1.0;
    const double lbo = LB / cp.g->s;  // s = 2^e: exact
    return lbo * lbo * (1.0 - 8.0 * u53) * (1.0 - gamma_up(cp.d + 2, u53));
  }
  const int nreg = cp.dpad * 2 / cp.b_rb;
  const int cpr = cp.b_rb / 16;  // 16-byte chunks per row per region
  const uint32_t x = (uint32_t)(((uint64_t)j * cp.b_rb >> 7) & (uint64_t)(cpr - 1));
  float acc = 0.f;
  for (int kb = 0; kb < nreg; ++kb) {
    const uint4* row = reinterpret_cast<const uint4*>(cp.bimg + (size_t)kb * cp.b_region +
                                                      (size_t)j * cp.b_rb);
    const float* q = qh + kb * (cp.b_rb / 2);
    for (int k = 0; k < cpr; ++k) {
      const uint4 v = __ldg(row + (k ^ x));
      const uint32_t w4[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const float d0 = q[8 * k + 2 * t] - widen_img<FMT>(w4[t] & 0xFFFFu);
        const float d1 = q[8 * k + 2 * t + 1] - widen_img<FMT>(w4[t] >> 16);
        acc = fmaf(d0, d0, acc);
        acc = fmaf(d1, d1, acc);
      }
    }
  }
  const double D = (double)acc / (1.0 + gamma_up(cp.dpad + 3, 5.9604644775390625e-08)) -
                   (cp.dpad + 3) * 1.1754943508222875e-38 /*2^-126*/;
  if (!(D > 0.0)) return -1.0;
  const double R = sqrt(D) * (1.0 - 2.0 * u53);
  const double LB = (R - ei - cp.ecol[j]) * (1.0 - 8.0 * u53);
  if (!(LB > 0.0)) return -1.0;
  const double lbo = LB / cp.g->s;  // s = 2^e: exact
  return lbo * lbo * (1.0 - 8.0 * u53) * (1.0 - gamma_up(cp.d + 2, u53));
}

// Per-warp telemetry (one global atomic per warp at exit, not per row).
struct RowTel {
  unsigned long long G = 0, nv = 0, nc = 0, pre = 0;  // pre: columns the pre-bound excluded
  double maxerr = 0.0;
};

template <int DT>
__device__ __forceinline__ void rerank_groups_row(
    const float* __restrict__ Q, int64_t q_begin, int64_t q_count, const float* __restrict__ X,
    int64_t n, int d, int k, int self_join, const int32_t* __restrict__ cand_idx,
    const float* __restrict__ cand_key, const float* __restrict__ cand_v, int kp, int lists,
    const uint2* __restrict__ mbuf, const int* __restrict__ mcnt, int mcap, int mparts,
    const CertParams& cp,
    const KnnOutDev& out, int32_t* __restrict__ fail_rows, double* __restrict__ fail_ub,
    int32_t* __restrict__ fail_count, int64_t r, RowTel& tel) {
  __shared__ float s_gk[kGrpWarps][kSelMax];      // staged group keys
  __shared__ int s_gi[kGrpWarps][kSelMax];        // staged group indices
  __shared__ float s_gu[kGrpWarps][kSelMax];      // per-group upper bounds (scratch)
  __shared__ double s_ck[kGrpWarps][kColMax];     // surviving columns: D64
  __shared__ int s_ci[kGrpWarps][kColMax];        //                    index
  __shared__ double s_tk[kGrpWarps][kMaxK];       // selected top-k
  __shared__ int s_ti[kGrpWarps][kMaxK];
  __shared__ float s_qh[kGrpWarps][256];          // query row xhat (pre-bound; dpad <= 256)
  extern __shared__ double s_xq[];                // [warps][d] query row in fp64
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t gi = q_begin + r;
  const float* xi = self_join ? X + gi * d : Q + r * d;
  double* xq = s_xq + (size_t)w * d;
  for (int c = lane; c < d; c += 32) xq[c] = (double)xi[c];
  const bool pre = cp.bimg != nullptr && self_join && cp.dpad <= 256;
  float* qh = s_qh[w];
  if (pre)
    for (int c = lane; c < cp.dpad; c += 32)
      qh[c] = cp.fmt == 2 ? widen_img<2>(img_elem(cp, gi, c)) : widen_img<1>(img_elem(cp, gi, c));

  float* gk = s_gk[w];
  int* gid = s_gi[w];
  // ---- stage every kept group (compacted with ballots)
  int G = 0;
  bool overflow = false;
  const int L = lists * kp;
  float vmin = CUDART_INF_F;  // the row's certificate threshold
  for (int c = 0; c < lists; ++c) vmin = fminf(vmin, cand_v[r * lists + c]);
  for (int e0 = 0; e0 < L; e0 += 32) {
    const int e = e0 + lane;
    const int g = e < L ? cand_idx[r * L + e] : -1;
    const unsigned live = __ballot_sync(0xffffffffu, g >= 0);
    const int pos = G + __popc(live & ((1u << lane) - 1u));
    if (g >= 0 && pos < kSelMax) {
      gk[pos] = cand_key[r * L + e];
      gid[pos] = g;
    }
    G += __popc(live);
  }
  if (mbuf) {
    // all part counts first, then every entry load of the row in flight at once
    int cnt[4] = {0, 0, 0, 0}, off[5];
#pragma unroll
    for (int h = 0; h < 4; ++h)
      if (h < mparts) cnt[h] = mcnt[r * mparts + h];
    off[0] = 0;
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      overflow |= cnt[h] > mcap;
      off[h + 1] = off[h] + min(cnt[h], mcap);
    }
    const int M = off[4];
    const int colflag = cp.colmode ? kColFlag : 0;  // main-pass appends are columns
    // appends at or above the row's certificate threshold vmin are dropped: they
    // bound nothing a certified row needs (its top-k lies strictly below
    // LB(vmin)), and UB stays valid over the rest (three-stage: the sample-tile
    // appends between tau and tau0)
    for (int e0 = 0; e0 < M; e0 += 128) {
      uint2 kv[4];
      bool keep[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int e = e0 + u * 32 + lane;
        keep[u] = false;
        if (e < M) {
          int h = 0;
#pragma unroll
          for (int q = 1; q < 4; ++q) h += e >= off[q];
          kv[u] = __ldcg(mbuf + (r * mparts + h) * (int64_t)mcap + (e - off[h]));
          keep[u] = __uint_as_float(kv[u].x) < vmin;
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const unsigned bm = __ballot_sync(0xffffffffu, keep[u]);
        const int pos = G + __popc(bm & ((1u << lane) - 1u));
        if (keep[u] && pos < kSelMax) {
          gk[pos] = __uint_as_float(kv[u].x);
          gid[pos] = (int)kv[u].y | colflag;
        }
        G += __popc(bm);
      }
    }
  }
  overflow |= G > kSelMax;
  if (G > kSelMax) G = kSelMax;
  __syncwarp();
  // ---- 1-2. UB and the candidates that can hold a top-k column: groups compacted
  // in place into gid[0, nvg), columns into the (then free) ub scratch; groups
  // expand 4 per step (4 x 8 columns), then columns 32 per step
  double UB;
  int nvg, nvc;
  int* visc = reinterpret_cast<int*>(s_gu[w]);
  plan_row(cp, r, k, gk, gid, s_gu[w], G, gid, kSelMax, visc, kSelMax, 1, UB, nvg, nvc, lane);
  const int nv = nvg + nvc;
  double* ck = s_ck[w];
  int* ci = s_ci[w];
  int nc = 0;
  const int gsteps = (nvg + 3) / 4;
  for (int st = 0; st < gsteps + (nvc + 31) / 32; ++st) {
    int64_t j;
    int g;
    if (st < gsteps) {
      const int gs = 4 * st + (lane >> 3);
      g = gs < nvg ? gid[gs] : -1;
      j = (int64_t)g * 8 + (lane & 7);
    } else {
      const int cs = 32 * (st - gsteps) + lane;
      g = cs < nvc ? visc[cs] : -1;
      j = g;
    }
    double key = CUDART_INF;
    bool live = g >= 0 && j < n && !(self_join && j == gi);
    if (pre && st < gsteps) {
      bool skip = false;
      if (live) {
        // d = dpad in {16, 32, 64} (DT > 0): the unrolled image read
        constexpr int DP = DT <= 64 ? DT : 0;
        const double lbc = cp.fmt == 2 ? lb2_col<2, DP>(cp, qh, j, cp.qe[r])
                                       : lb2_col<1, DP>(cp, qh, j, cp.qe[r]);
        skip = lbc > UB;  // provably not within the k nearest: no fp32 row gather, no O1
      }
      tel.pre += (unsigned long long)__popc(__ballot_sync(0xffffffffu, skip));
      live = live && !skip;
    }
    if (live) {
      const float* xj = X + j * d;
      double acc = 0.0;  // O1, bit-identical to the oracle (no FMA, ascending c)
      if constexpr (DT > 0) {
        acc = d64_fixed<DT>(xq, xj);
      } else if ((d & 15) == 0) {
        // 4 independent 16-byte loads in flight, then the 16 terms in order
        const float4* x4 = reinterpret_cast<const float4*>(xj);
        for (int c16 = 0; c16 < (d >> 4); ++c16) {
          float4 v[4];
#pragma unroll
          for (int u = 0; u < 4; ++u) v[u] = __ldg(x4 + 4 * c16 + u);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const double* xc = xq + 16 * c16 + 4 * u;
            double t = __dsub_rn(xc[0], (double)v[u].x);
            acc = __dadd_rn(acc, __dmul_rn(t, t));
            t = __dsub_rn(xc[1], (double)v[u].y);
            acc = __dadd_rn(acc, __dmul_rn(t, t));
            t = __dsub_rn(xc[2], (double)v[u].z);
            acc = __dadd_rn(acc, __dmul_rn(t, t));
            t = __dsub_rn(xc[3], (double)v[u].w);
            acc = __dadd_rn(acc, __dmul_rn(t, t));
          }
        }
      } else if ((d & 3) == 0) {
        const float4* x4 = reinterpret_cast<const float4*>(xj);
        for (int c4 = 0; c4 < (d >> 2); ++c4) {
          const float4 v = __ldg(x4 + c4);
          double t = __dsub_rn(xq[4 * c4 + 0], (double)v.x);
          acc = __dadd_rn(acc, __dmul_rn(t, t));
          t = __dsub_rn(xq[4 * c4 + 1], (double)v.y);
          acc = __dadd_rn(acc, __dmul_rn(t, t));
          t = __dsub_rn(xq[4 * c4 + 2], (double)v.z);
          acc = __dadd_rn(acc, __dmul_rn(t, t));
          t = __dsub_rn(xq[4 * c4 + 3], (double)v.w);
          acc = __dadd_rn(acc, __dmul_rn(t, t));
        }
      } else {
        for (int c = 0; c < d; ++c) {
          const double t = __dsub_rn(xq[c], (double)__ldg(xj + c));
          acc = __dadd_rn(acc, __dmul_rn(t, t));
        }
      }
      key = acc;
    }
    const bool keep = key <= UB && key < CUDART_INF;
    const unsigned km = __ballot_sync(0xffffffffu, keep);
    const int pos = nc + __popc(km & ((1u << lane) - 1u));
    if (keep && pos < kColMax) {
      ck[pos] = key;
      ci[pos] = (int)j;
    }
    nc += __popc(km);
  }
  overflow |= nc > kColMax;
  if (nc > kColMax) nc = kColMax;
  __syncwarp();
  // ---- 3. the k smallest by (D64, index)
  double* tk = s_tk[w];
  int* ti = s_ti[w];
  if (nc <= 32) {
    double kk1 = lane < nc ? ck[lane] : CUDART_INF;
    int ii1 = lane < nc ? ci[lane] : INT32_MAX;
    warp_sort32(kk1, ii1, lane);
    if (lane < k) {
      tk[lane] = kk1;
      ti[lane] = ii1;
    }
  } else if (nc <= 64) {
    double kk[2];
    int ii[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int p = 2 * lane + e;
      kk[e] = p < nc ? ck[p] : CUDART_INF;
      ii[e] = p < nc ? ci[p] : INT32_MAX;
    }
    warp_sort64(kk, ii, lane);
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int p = 2 * lane + e;
      if (p < k) {
        tk[p] = kk[e];
        ti[p] = ii[e];
      }
    }
  } else {
    // k rounds of warp argmin; each lane caches the minimum of its slice
    auto slice_min = [&](double& mk, int& mi, int& mp) {
      mk = CUDART_INF;
      mi = INT32_MAX;
      mp = -1;
      for (int e = lane; e < nc; e += 32)
        if (key_less(ck[e], ci[e], mk, mi)) {
          mk = ck[e];
          mi = ci[e];
          mp = e;
        }
    };
    double lk;
    int li, lp;
    slice_min(lk, li, lp);
    for (int m = 0; m < k; ++m) {
      double bk = lk;
      int bi = li;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ok = __shfl_xor_sync(0xffffffffu, bk, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (key_less(ok, oi, bk, bi)) {
          bk = ok;
          bi = oi;
        }
      }
      if (lane == 0) {
        tk[m] = bk;
        ti[m] = bi;
      }
      if (lp >= 0 && li == bi && bi != INT32_MAX) {  // owner retires it
        ck[lp] = CUDART_INF;
        ci[lp] = INT32_MAX;
        slice_min(lk, li, lp);
      }
    }
  }
  __syncwarp();
  double err = 0.0;
  const bool have = nc >= k;
  bool cert = !overflow && have && row_certified(cp, r, vmin, tk[k - 1], &err);
  if (cp.force_fail) cert = false;
  tel.maxerr = fmax(tel.maxerr, err);
  tel.G += (unsigned long long)G;
  tel.nv += (unsigned long long)nv;
  tel.nc += (unsigned long long)nc;
  if (cert) {
    write_row(out, r, k, tk, ti, lane, 32);
  } else if (lane == 0) {
    const int slot = atomicAdd(fail_count, 1);
    fail_rows[slot] = (int32_t)r;
    // both UB and the k-th exact distance among kept columns bound the true
    // k-th distance from above (the fallback only collects columns below it)
    fail_ub[slot] = fmin(UB, have ? tk[k - 1] : CUDART_INF);
  }
}

// 4 blocks (16 warps) per SM = 128 registers: measured on B200 (C2, C3) no
// slower than 5 or 6 blocks at 92 / 80 registers, and faster than the 168
// registers the compiler picks unconstrained.
template <int DT>
__global__ void __launch_bounds__(kGrpWarps * 32, 4)
    k_rerank_groups(const float* __restrict__ Q, int64_t q_begin, int64_t q_count,
                    const float* __restrict__ X, int64_t n, int d, int k, int self_join,
                    const int32_t* __restrict__ cand_idx, const float* __restrict__ cand_key,
                    const float* __restrict__ cand_v, int kp, int lists,
                    const uint2* __restrict__ mbuf, const int* __restrict__ mcnt, int mcap,
                    int mparts,
                    CertParams cp, KnnOutDev out, int32_t* __restrict__ fail_rows,
                    double* __restrict__ fail_ub, int32_t* __restrict__ fail_count,
                    unsigned long long* __restrict__ max_err_bits,
                    unsigned long long* __restrict__ counters) {
  // persistent grid-stride over rows: no block barriers, balanced tails
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  RowTel tel;
  for (int64_t r = (int64_t)blockIdx.x * kGrpWarps + w; r < q_count;
       r += (int64_t)gridDim.x * kGrpWarps) {
    __syncwarp();
    rerank_groups_row<DT>(Q, q_begin, q_count, X, n, d, k, self_join, cand_idx, cand_key, cand_v,
                          kp, lists, mbuf, mcnt, mcap, mparts, cp, out, fail_rows, fail_ub,
                          fail_count, r, tel);
  }
  if (lane == 0) {
    if (tel.maxerr > 0.0) atomicMax(max_err_bits, (unsigned long long)__double_as_longlong(tel.maxerr));
    if (tel.G) atomicAdd(counters + 0, tel.G);
    if (tel.nv) atomicAdd(counters + 1, tel.nv);
    if (tel.nc) atomicAdd(counters + 2, tel.nc);
    if (tel.pre) atomicAdd(counters + 3, tel.pre);
  }
}


// ============================================= split re-rank (two-pass mode)
// The per-row warp of k_rerank_groups walks its visited groups in ~6 dependent
// rounds (gather, then a 3*d-step fp64 chain), so the kernel is bound by that
// per-row latency.  The split form keeps the same arithmetic but flattens the
// expansion across the whole GPU:
//   k_rr_plan   (warp per row)  stage the kept groups, kappa, UB, key cut, and
//               the visited group list -> global;
//   scan + k_rr_map             task -> (row, round of 4 groups);
//   k_rr_expand (warp per task) O1 for the round's 32 columns, columns with
//               D64 <= UB appended to the row's list (slots by atomicAdd);
//   k_rr_finish (warp per row)  top-k by (D64, index), certificate, outputs.
// The kept set of a row is the same as in k_rerank_groups (its order differs;
// the selection is a total order), so outputs are identical.
constexpr int kRrVis = kSelMax;  // visited groups per row (more: the row goes to the fallback)

struct RrWs {
  int32_t* nv;     // [q] visited groups (front of gid)
  int32_t* nvc;    // [q] visited column candidates (back of gid, descending)
  int32_t* flags;  // [q] bit 0: overflow (the row cannot be certified)
  int32_t* G;      // [q] staged groups (telemetry)
  int32_t* nc;     // [q] kept-column counter
  float* vmin;     // [q] pass-1 threshold (certificate)
  double* ub;      // [q] UB on the k-th exact distance
  int32_t* gid;    // [q][kRrVis]
  double* ck;      // [q][kColMax] kept columns: D64
  int32_t* ci;     // [q][kColMax]                index
  int64_t* tcnt;   // [q] expansion tasks
  int64_t* toff;   // [q + 1]
  int64_t* map;    // [q * kRrVis / 4]
  void* scan;
};

// carve the workspace at base (base = nullptr: offsets only, for sizing)
__host__ RrWs rr_layout(void* base, int64_t q, size_t* total = nullptr) {
  RrWs w;
  const int64_t q1 = q < 1 ? 1 : q;
  size_t off = 0;
  auto take = [&](size_t bytes) {
    char* r = base ? static_cast<char*>(base) + off : nullptr;
    off += (bytes + 255) / 256 * 256;
    return r;
  };
  w.ub = reinterpret_cast<double*>(take(q1 * 8));
  w.ck = reinterpret_cast<double*>(take((size_t)q1 * kColMax * 8));
  w.tcnt = reinterpret_cast<int64_t*>(take(q1 * 8));
  w.toff = reinterpret_cast<int64_t*>(take((q1 + 1) * 8));
  w.map = reinterpret_cast<int64_t*>(take((size_t)q1 * (kRrVis / 4) * 8));
  w.scan = take(scan_workspace(q1));
  w.nv = reinterpret_cast<int32_t*>(take(q1 * 4));
  w.nvc = reinterpret_cast<int32_t*>(take(q1 * 4));
  w.flags = reinterpret_cast<int32_t*>(take(q1 * 4));
  w.G = reinterpret_cast<int32_t*>(take(q1 * 4));
  w.nc = reinterpret_cast<int32_t*>(take(q1 * 4));
  w.vmin = reinterpret_cast<float*>(take(q1 * 4));
  w.gid = reinterpret_cast<int32_t*>(take((size_t)q1 * kRrVis * 4));
  w.ci = reinterpret_cast<int32_t*>(take((size_t)q1 * kColMax * 4));
  if (total) *total = off;
  return w;
}

__global__ void __launch_bounds__(kGrpWarps * 32, 4)
    k_rr_plan(int64_t q_count, int k, const int32_t* __restrict__ cand_idx,
              const float* __restrict__ cand_key, const float* __restrict__ cand_v, int kp, int lists,
              const uint2* __restrict__ mbuf, const int* __restrict__ mcnt, int mcap, int mparts,
              CertParams cp, RrWs rw) {
  __shared__ float s_gk[kGrpWarps][kSelMax];
  __shared__ int s_gi[kGrpWarps][kSelMax];
  __shared__ float s_gu[kGrpWarps][kSelMax];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* gk = s_gk[w];
  int* gid = s_gi[w];
  for (int64_t r = (int64_t)blockIdx.x * kGrpWarps + w; r < q_count;
       r += (int64_t)gridDim.x * kGrpWarps) {
    __syncwarp();
    int G = 0;
    bool overflow = false;
    const int L = lists * kp;
    float vmin = CUDART_INF_F;  // the row's certificate threshold
    for (int c = 0; c < lists; ++c) vmin = fminf(vmin, cand_v[r * lists + c]);
    for (int e0 = 0; e0 < L; e0 += 32) {
      const int e = e0 + lane;
      const int g = e < L ? cand_idx[r * L + e] : -1;
      const unsigned live = __ballot_sync(0xffffffffu, g >= 0);
      const int pos = G + __popc(live & ((1u << lane) - 1u));
      if (g >= 0 && pos < kSelMax) {
        gk[pos] = cand_key[r * L + e];
        gid[pos] = g;
      }
      G += __popc(live);
    }
    if (mbuf) {
      int cnt[4] = {0, 0, 0, 0}, off[5];
#pragma unroll
      for (int h = 0; h < 4; ++h)
        if (h < mparts) cnt[h] = mcnt[r * mparts + h];
      off[0] = 0;
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        overflow |= cnt[h] > mcap;
        off[h + 1] = off[h] + min(cnt[h], mcap);
      }
      const int M = off[4];
      const int colflag = cp.colmode ? kColFlag : 0;  // main-pass appends are columns
      // appends at or above the row's certificate threshold vmin are dropped: they
      // bound nothing a certified row needs (its top-k lies strictly below
      // LB(vmin)), and UB stays valid over the rest (three-stage: the sample-tile
      // appends between tau and tau0)
      for (int e0 = 0; e0 < M; e0 += 128) {
        uint2 kv[4];
        bool keep[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int e = e0 + u * 32 + lane;
          keep[u] = false;
          if (e < M) {
            int h = 0;
#pragma unroll
            for (int q = 1; q < 4; ++q) h += e >= off[q];
            kv[u] = __ldcg(mbuf + (r * mparts + h) * (int64_t)mcap + (e - off[h]));
            keep[u] = __uint_as_float(kv[u].x) < vmin;
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const unsigned bm = __ballot_sync(0xffffffffu, keep[u]);
          const int pos = G + __popc(bm & ((1u << lane) - 1u));
          if (keep[u] && pos < kSelMax) {
            gk[pos] = __uint_as_float(kv[u].x);
            gid[pos] = (int)kv[u].y | colflag;
          }
          G += __popc(bm);
        }
      }
    }
    overflow |= G > kSelMax;
    if (G > kSelMax) G = kSelMax;
    __syncwarp();
    // UB and the visited groups, as in rerank_groups_row, straight to the row's global list
    double UB;
    int nvg, nvc;
    plan_row(cp, r, k, gk, gid, s_gu[w], G, rw.gid + r * kRrVis, kRrVis,
             rw.gid + r * kRrVis + (kRrVis - 1), kRrVis, -1, UB, nvg, nvc, lane);
    int nv = nvg + nvc;  // groups from the front of the row's list, columns from its back
    if (nv > kRrVis) {
      overflow = true;
      nvg = nvc = 0;
      nv = 0;
    }
    if (lane == 0) {
      rw.nv[r] = nvg;
      rw.nvc[r] = nvc;
      rw.flags[r] = overflow ? 1 : 0;
      rw.G[r] = G;
      rw.nc[r] = 0;
      rw.vmin[r] = vmin;
      rw.ub[r] = UB;
      rw.tcnt[r] = (nvg + 3) / 4 + (nvc + 31) / 32;
    }
  }
}

__global__ void k_rr_map(int64_t q_count, RrWs rw) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= q_count) return;
  const int64_t t0 = rw.toff[r];
  const int nt = (int)(rw.toff[r + 1] - t0);
  for (int c = 0; c < nt; ++c) rw.map[t0 + c] = (r << 8) | c;
}

template <int DT>
__global__ void __launch_bounds__(kGrpWarps * 32)
    k_rr_expand(const float* __restrict__ Q, int64_t q_begin, const float* __restrict__ X,
                int64_t n, int d, int self_join, RrWs rw, const int64_t* __restrict__ ntasks) {
  extern __shared__ double s_xq[];  // [warps][d]
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* xq = s_xq + (size_t)w * d;
  const int64_t T = *ntasks;
  for (int64_t task = (int64_t)blockIdx.x * kGrpWarps + w; task < T;
       task += (int64_t)gridDim.x * kGrpWarps) {
    const int64_t code = rw.map[task];
    const int64_t r = code >> 8;
    const int c = (int)(code & 0xFF);
    const int64_t gi = q_begin + r;
    const float* xi = self_join ? X + gi * d : Q + r * d;
    __syncwarp();
    for (int e = lane; e < d; e += 32) xq[e] = (double)xi[e];
    __syncwarp();
    const int nv = rw.nv[r];
    const double UB = rw.ub[r];
    int g;
    int64_t j;
    const int gtasks = (nv + 3) / 4;
    if (c < gtasks) {  // 4 groups x 8 columns per task
      const int gs = 4 * c + (lane >> 3);
      g = gs < nv ? rw.gid[r * kRrVis + gs] : -1;
      j = (int64_t)g * 8 + (lane & 7);
    } else {           // 32 column candidates per task (stored from the back)
      const int cs = 32 * (c - gtasks) + lane;
      g = cs < rw.nvc[r] ? rw.gid[r * kRrVis + (kRrVis - 1 - cs)] : -1;
      j = g;
    }
    double key = CUDART_INF;
    if (g >= 0 && j < n && !(self_join && j == gi)) {
      const float* xj = X + j * d;
      if constexpr (DT > 0) {
        key = d64_fixed<DT>(xq, xj);
      } else {
        double acc = 0.0;  // O1: ascending c, no FMA
        for (int cc = 0; cc < d; ++cc) {
          const double t = __dsub_rn(xq[cc], (double)__ldg(xj + cc));
          acc = __dadd_rn(acc, __dmul_rn(t, t));
        }
        key = acc;
      }
    }
    const bool keep = key <= UB && key < CUDART_INF;
    const unsigned km = __ballot_sync(0xffffffffu, keep);
    if (km == 0u) continue;
    int base = 0;
    if (lane == 0) base = atomicAdd(rw.nc + r, __popc(km));
    base = __shfl_sync(0xffffffffu, base, 0);
    const int pos = base + __popc(km & ((1u << lane) - 1u));
    if (keep && pos < kColMax) {
      rw.ck[r * kColMax + pos] = key;
      rw.ci[r * kColMax + pos] = (int)j;
    }
  }
}

__global__ void __launch_bounds__(kGrpWarps * 32)
    k_rr_finish(int64_t q_count, int k, CertParams cp, RrWs rw, KnnOutDev out,
                int32_t* __restrict__ fail_rows, double* __restrict__ fail_ub,
                int32_t* __restrict__ fail_count, unsigned long long* __restrict__ max_err_bits,
                unsigned long long* __restrict__ counters) {
  __shared__ double s_ck[kGrpWarps][kColMax];
  __shared__ int s_ci[kGrpWarps][kColMax];
  __shared__ double s_tk[kGrpWarps][kMaxK];
  __shared__ int s_ti[kGrpWarps][kMaxK];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  RowTel tel;
  for (int64_t r = (int64_t)blockIdx.x * kGrpWarps + w; r < q_count;
       r += (int64_t)gridDim.x * kGrpWarps) {
    __syncwarp();
    const int ncr = rw.nc[r];
    bool overflow = rw.flags[r] != 0 || ncr > kColMax;
    const int nc = ncr < kColMax ? ncr : kColMax;
    double* ck = s_ck[w];
    int* ci = s_ci[w];
    double* tk = s_tk[w];
    int* ti = s_ti[w];
    if (nc > 64) {
      for (int e = lane; e < nc; e += 32) {
        ck[e] = rw.ck[r * kColMax + e];
        ci[e] = rw.ci[r * kColMax + e];
      }
    }
    __syncwarp();
    if (nc <= 32) {
      double kk1 = lane < nc ? rw.ck[r * kColMax + lane] : CUDART_INF;
      int ii1 = lane < nc ? rw.ci[r * kColMax + lane] : INT32_MAX;
      warp_sort32(kk1, ii1, lane);
      if (lane < k) {
        tk[lane] = kk1;
        ti[lane] = ii1;
      }
    } else if (nc <= 64) {
      double kk[2];
      int ii[2];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int p = 2 * lane + e;
        kk[e] = p < nc ? rw.ck[r * kColMax + p] : CUDART_INF;
        ii[e] = p < nc ? rw.ci[r * kColMax + p] : INT32_MAX;
      }
      warp_sort64(kk, ii, lane);
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int p = 2 * lane + e;
        if (p < k) {
          tk[p] = kk[e];
          ti[p] = ii[e];
        }
      }
    } else {
      auto slice_min = [&](double& mk, int& mi, int& mp) {
        mk = CUDART_INF;
        mi = INT32_MAX;
        mp = -1;
        for (int e = lane; e < nc; e += 32)
          if (key_less(ck[e], ci[e], mk, mi)) {
            mk = ck[e];
            mi = ci[e];
            mp = e;
          }
      };
      double lk;
      int li, lp;
      slice_min(lk, li, lp);
      for (int m = 0; m < k; ++m) {
        double bk = lk;
        int bi = li;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ok = __shfl_xor_sync(0xffffffffu, bk, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (key_less(ok, oi, bk, bi)) {
            bk = ok;
            bi = oi;
          }
        }
        if (lane == 0) {
          tk[m] = bk;
          ti[m] = bi;
        }
        if (lp >= 0 && li == bi && bi != INT32_MAX) {
          ck[lp] = CUDART_INF;
          ci[lp] = INT32_MAX;
          slice_min(lk, li, lp);
        }
      }
    }
    __syncwarp();
    double err = 0.0;
    const bool have = nc >= k;
    bool cert = !overflow && have && row_certified(cp, r, rw.vmin[r], tk[k - 1], &err);
    if (cp.force_fail) cert = false;
    tel.maxerr = fmax(tel.maxerr, err);
    tel.G += (unsigned long long)rw.G[r];
    tel.nv += (unsigned long long)(rw.nv[r] + rw.nvc[r]);
    tel.nc += (unsigned long long)nc;
    if (cert) {
      write_row(out, r, k, tk, ti, lane, 32);
    } else if (lane == 0) {
      const int slot = atomicAdd(fail_count, 1);
      fail_rows[slot] = (int32_t)r;
      fail_ub[slot] = fmin(rw.ub[r], have ? tk[k - 1] : CUDART_INF);
    }
  }
  if (lane == 0) {
    if (tel.maxerr > 0.0) atomicMax(max_err_bits, (unsigned long long)__double_as_longlong(tel.maxerr));
    if (tel.G) atomicAdd(counters + 0, tel.G);
    if (tel.nv) atomicAdd(counters + 1, tel.nv);
    if (tel.nc) atomicAdd(counters + 2, tel.nc);
  }
}

// ============================================ second tier for bf16 first passes
// Rows a bf16 pass could not certify are re-answered by an fp16 pass (a finer
// quantization of the same method, SURVEY 8(a) a4 tier 1): their rows are
// gathered as queries, the library runs them against all of X with k+1
// neighbours and no exclusion (k for query-mode calls), and the scatter drops
// the row's own index (or, if it is not among the k+1 -- k+1 exact duplicates
// with smaller indices -- the last entry), writing the outputs as write_row does.
__global__ void k_gather_rows(const float* __restrict__ src, int64_t base,
                              const int32_t* __restrict__ rows, int nr, int d,
                              float* __restrict__ dst) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (int64_t)nr * d) return;
  const int64_t r = i / d, c = i - r * d;
  dst[i] = src[(base + rows[r]) * d + c];
}

__global__ void k_mark_rows(const int32_t* __restrict__ rows, int nr, int32_t value,
                            int32_t* __restrict__ dst) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < nr) dst[rows[i]] = value;
}

__global__ void k_tier2_scatter(const int32_t* __restrict__ rows, int nr, int64_t q_begin,
                                int self_join, int k, int k2, const int64_t* __restrict__ idx2,
                                const double* __restrict__ dd2, KnnOutDev out) {
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (w >= nr) return;
  const int64_t r = rows[w];
  const int64_t self = self_join ? q_begin + r : -1;
  // position of the self entry among the k2 (k2 - 1 = drop the last when absent)
  int drop = k2 > k ? k2 - 1 : k2;
  for (int m0 = 0; m0 < k2; m0 += 32) {
    const int m = m0 + lane;
    const unsigned hit = __ballot_sync(0xffffffffu, m < k2 && idx2[(int64_t)w * k2 + m] == self);
    if (hit && drop == k2 - 1 && k2 > k) drop = m0 + __ffs(hit) - 1;
  }
  double acc = 0.0;
  for (int m0 = 0; m0 < k; m0 += 32) {
    const int m = m0 + lane;
    double dd = 0.0;
    if (m < k) {
      const int src = m < drop ? m : m + 1;
      dd = dd2[(int64_t)w * k2 + src];
      const int64_t j = idx2[(int64_t)w * k2 + src];
      if (out.idx) out.idx[r * k + m] = j;
      if (out.dist64) out.dist64[r * k + m] = dd;
      if (out.dist) out.dist[r * k + m] = __double2float_rn(dd);
      if (m == k - 1) {
        if (out.kdist64) out.kdist64[r] = dd;
        if (out.score_kth) out.score_kth[r] = __double2float_rn(dd);
      }
    }
    if (out.score_mean) {
      const int cnt = k - m0 < 32 ? k - m0 : 32;
      for (int t = 0; t < cnt; ++t) acc = __dadd_rn(acc, __shfl_sync(0xffffffffu, dd, t));
    }
  }
  if (lane == 0 && out.score_mean) out.score_mean[r] = __double2float_rn(__ddiv_rn(acc, (double)k));
}

// ===================================================================== NWR
// Neighbours within range (§5.3): {j != i : D_ij <= phi},
// D_ij the squared distance of Eq. (3) evaluated as the oracle's O1.  Provable
// quantization applied as the paper prescribes: the fp16
// tensor-core main pass decides every pair it can, the rest is verified in fp64.
//  * tau_i = key_cut_from_ub(phi): every column with D64 <= phi has its pass-1
//    key w~ <= tau_i (lower-bound inversion, all roundings upward), so the
//    append-only main pass with threshold tau_i keeps a superset of row i's
//    neighbours (a group is kept when its minimum is below tau_i).
//  * verify: the kept groups, sorted by index, expanded and decided with O1
//    (exactly the oracle's comparison), neighbours written ascending by j.
//  * rows whose candidate buffers overflowed are answered by fp64 brute force.

__global__ void k_nwr_tau(int64_t q_count, double phi, CertParams cp, float* __restrict__ tau) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= q_count) return;
  const float cut = key_cut_from_ub(cp, r, phi);
  tau[r] = nextafterf(cut, CUDART_INF_F);  // the filter keeps groups with min < tau
}

constexpr int kNwrWarps = 4;
constexpr int kNwrMaxG = 4096;   // kept groups per row (4 parts x up to 1024)
constexpr int kNwrChunk = 64;    // kept groups per verification task

// Verification is flattened into tasks of <= 64 kept groups, so a dense row
// with thousands of kept groups is spread over many warps instead of holding
// one warp for the whole pass (the per-row warp left the kernel waiting on its
// heaviest rows).
//   k_nwr_tasks: per row, overflow check (-> brute-force list) and task count;
//   scan -> task offsets; k_nwr_map: task -> (row, part, chunk);
//   k_nwr_mask: per task, O1 for every column of its groups; each entry is
//     rewritten in place as (8-bit mask of the columns with D64 <= phi, group)
//     and the row's count accumulated;
//   k_nwr_emit: per row, the entries with a nonzero mask sorted by group, then
//     their columns written ascending at row_ptr[r] (no distance computed twice).
__global__ void k_nwr_tasks(int64_t q_count, const int* __restrict__ mcnt, int mcap, int mparts,
                            int64_t* __restrict__ tcnt, int64_t* __restrict__ counts,
                            int32_t* __restrict__ ovf_rows, int32_t* __restrict__ ovf_count) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= q_count) return;
  bool over = false;
  int64_t nt = 0;
  for (int h = 0; h < mparts; ++h) {
    const int c = mcnt[r * mparts + h];
    over |= c > mcap;
    nt += (min(c, mcap) + kNwrChunk - 1) / kNwrChunk;
  }
  tcnt[r] = over ? 0 : nt;
  counts[r] = over ? -1 : 0;
  if (over) ovf_rows[atomicAdd(ovf_count, 1)] = (int32_t)r;
}

__global__ void k_nwr_map(int64_t q_count, const int* __restrict__ mcnt, int mcap, int mparts,
                          const int64_t* __restrict__ toff, int64_t* __restrict__ map) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= q_count) return;
  int64_t t = toff[r];
  if (toff[r + 1] == t) return;  // overflowed or empty
  for (int h = 0; h < mparts; ++h) {
    const int m = min(mcnt[r * mparts + h], mcap);
    for (int c = 0; c * kNwrChunk < m; ++c) map[t++] = ((r * mparts + h) << 8) | c;
  }
}

template <int DT>
__global__ void __launch_bounds__(kNwrWarps * 32)
    k_nwr_mask(const float* __restrict__ Q, int64_t q_begin, const float* __restrict__ X,
               int64_t n, int d, int self_join, double phi, uint2* __restrict__ mbuf,
               const int* __restrict__ mcnt, int mcap, int mparts,
               const int64_t* __restrict__ map, const int64_t* __restrict__ ntasks,
               int64_t* __restrict__ counts) {
  extern __shared__ double s_xq[];  // [warps][d] query rows in fp64
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double* xq = s_xq + (size_t)w * d;
  const int64_t T = *ntasks;
  for (int64_t task = (int64_t)blockIdx.x * kNwrWarps + w; task < T;
       task += (int64_t)gridDim.x * kNwrWarps) {
    const int64_t code = map[task];
    const int64_t rp = code >> 8;
    const int c = (int)(code & 0xFF);
    const int64_t r = rp / mparts;
    const int64_t gi = q_begin + r;
    const float* xi = self_join ? X + gi * d : Q + r * d;
    __syncwarp();
    for (int e = lane; e < d; e += 32) xq[e] = (double)xi[e];
    __syncwarp();
    uint2* ent = mbuf + rp * (int64_t)mcap;
    const int e1 = min(min(mcnt[rp], mcap), (c + 1) * kNwrChunk);
    int cnt = 0;
    for (int b0 = c * kNwrChunk; b0 < e1; b0 += 4) {
      const int gs = b0 + (lane >> 3);
      const int grp = gs < e1 ? (int)ent[gs].y : -1;
      const int64_t j = (int64_t)grp * 8 + (lane & 7);
      bool keep = false;
      if (grp >= 0 && j < n && !(self_join && j == gi)) {
        const float* xj = X + j * d;
        double acc;
        if constexpr (DT > 0) {
          acc = d64_fixed<DT>(xq, xj);
        } else {
          acc = 0.0;  // O1: ascending c, no FMA
          for (int cc = 0; cc < d; ++cc) {
            const double t = __dsub_rn(xq[cc], (double)__ldg(xj + cc));
            acc = __dadd_rn(acc, __dmul_rn(t, t));
          }
        }
        keep = acc <= phi;
      }
      const unsigned km = __ballot_sync(0xffffffffu, keep);
      if ((lane & 7) == 0 && grp >= 0) ent[gs].x = (km >> (lane & 24)) & 0xFFu;
      cnt += __popc(km);
    }
    if (lane == 0 && cnt) atomicAdd(reinterpret_cast<unsigned long long*>(counts + r),
                                    (unsigned long long)cnt);
  }
}

// Rows with at most kEmitLight nonzero entries are sorted by one warp; the
// rest (dense rows) are queued for k_nwr_emit_heavy, a 512-thread block each.
constexpr int kEmitLight = 256;
constexpr int kEmitWarps = 4;
constexpr int kEmitHeavyThreads = 512;

// the row's entries with a nonzero mask, compacted into (g, mk); returns the count
__device__ __forceinline__ int nwr_compact(const uint2* __restrict__ mbuf, const int* __restrict__ mcnt,
                                           int mcap, int mparts, int64_t r, int lane, int* g,
                                           int* mk, int cap) {
  int nz = 0;
  for (int h = 0; h < mparts; ++h) {
    const int m = min(mcnt[r * mparts + h], mcap);
    const uint2* src = mbuf + (r * mparts + h) * (int64_t)mcap;
    for (int e0 = 0; e0 < m; e0 += 32) {
      const int e = e0 + lane;
      const uint2 v = e < m ? src[e] : make_uint2(0u, 0u);
      const unsigned live = __ballot_sync(0xffffffffu, v.x != 0u);
      const int pos = nz + __popc(live & ((1u << lane) - 1u));
      if (v.x && pos < cap) {
        g[pos] = (int)v.y;
        mk[pos] = (int)v.x;
      }
      nz += __popc(live);
    }
  }
  return nz;
}

__global__ void __launch_bounds__(kEmitWarps * 32)
    k_nwr_emit(int64_t q_count, const uint2* __restrict__ mbuf, const int* __restrict__ mcnt,
               int mcap, int mparts, const int64_t* __restrict__ row_ptr,
               int32_t* __restrict__ cols, int32_t* __restrict__ heavy, int32_t* __restrict__ nheavy) {
  __shared__ int s_g[kEmitWarps][kEmitLight], s_m[kEmitWarps][kEmitLight];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * kEmitWarps + w;
  if (r >= q_count) return;
  int* g = s_g[w];
  int* mk = s_m[w];
  bool over = false;
  for (int h = 0; h < mparts; ++h) over |= mcnt[r * mparts + h] > mcap;
  if (over) return;  // the brute-force tier writes this row
  const int nz = nwr_compact(mbuf, mcnt, mcap, mparts, r, lane, g, mk, kEmitLight);
  if (nz > kEmitLight) {
    if (lane == 0) heavy[atomicAdd(nheavy, 1)] = (int32_t)r;
    return;
  }
  // ascending by group (bitonic over the next power of two; groups are unique)
  int P = 1;
  while (P < nz) P <<= 1;
  for (int e = nz + lane; e < P; e += 32) {
    g[e] = INT32_MAX;
    mk[e] = 0;
  }
  __syncwarp();
  for (int kk = 2; kk <= P; kk <<= 1)
    for (int j = kk >> 1; j > 0; j >>= 1) {
      for (int e = lane; e < P; e += 32) {
        const int l = e ^ j;
        if (l > e) {
          const int a = g[e], b = g[l];
          const bool up = (e & kk) == 0;
          if (up ? a > b : a < b) {
            g[e] = b;
            g[l] = a;
            const int t = mk[e];
            mk[e] = mk[l];
            mk[l] = t;
          }
        }
      }
      __syncwarp();
    }
  int64_t base = row_ptr[r];
  for (int e0 = 0; e0 < nz; e0 += 32) {
    const int e = e0 + lane;
    const unsigned m8 = e < nz ? (unsigned)mk[e] : 0u;
    const int pc = __popc(m8);
    int incl = pc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    int64_t pos = base + incl - pc;
    for (unsigned m = m8; m; m &= m - 1u) cols[pos++] = (int32_t)((unsigned)g[e] * 8u + (unsigned)(__ffs(m) - 1));
    base += __shfl_sync(0xffffffffu, incl, 31);
  }
}

// dense rows: one 512-thread block per row (compaction by warp 0, block-wide
// bitonic sort, block prefix sums for the output positions)
__global__ void __launch_bounds__(kEmitHeavyThreads)
    k_nwr_emit_heavy(const uint2* __restrict__ mbuf, const int* __restrict__ mcnt, int mcap,
                     int mparts, const int64_t* __restrict__ row_ptr, int32_t* __restrict__ cols,
                     const int32_t* __restrict__ heavy, const int32_t* __restrict__ nheavy) {
  extern __shared__ int s_h[];  // [kNwrMaxG] groups, [kNwrMaxG] masks
  __shared__ int s_nz, s_wsum[kEmitHeavyThreads / 32];
  __shared__ int64_t s_base;
  int* g = s_h;
  int* mk = s_h + kNwrMaxG;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int nh = *nheavy;
  for (int hr = blockIdx.x; hr < nh; hr += gridDim.x) {
    const int64_t r = heavy[hr];
    __syncthreads();
    if (w == 0) {
      const int nz = nwr_compact(mbuf, mcnt, mcap, mparts, r, lane, g, mk, kNwrMaxG);
      if (lane == 0) {
        s_nz = nz;
        s_base = row_ptr[r];
      }
    }
    __syncthreads();
    const int nz = s_nz;
    int P = 1;
    while (P < nz) P <<= 1;
    for (int e = nz + t; e < P; e += kEmitHeavyThreads) {
      g[e] = INT32_MAX;
      mk[e] = 0;
    }
    __syncthreads();
    for (int kk = 2; kk <= P; kk <<= 1)
      for (int j = kk >> 1; j > 0; j >>= 1) {
        for (int e = t; e < P; e += kEmitHeavyThreads) {
          const int l = e ^ j;
          if (l > e) {
            const int a = g[e], b = g[l];
            const bool up = (e & kk) == 0;
            if (up ? a > b : a < b) {
              g[e] = b;
              g[l] = a;
              const int x = mk[e];
              mk[e] = mk[l];
              mk[l] = x;
            }
          }
        }
        __syncthreads();
      }
    for (int e0 = 0; e0 < nz; e0 += kEmitHeavyThreads) {
      const int e = e0 + t;
      const unsigned m8 = e < nz ? (unsigned)mk[e] : 0u;
      const int pc = __popc(m8);
      int incl = pc;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      if (lane == 31) s_wsum[w] = incl;
      __syncthreads();
      int before = 0, tot = 0;
      for (int q = 0; q < kEmitHeavyThreads / 32; ++q) {
        before += q < w ? s_wsum[q] : 0;
        tot += s_wsum[q];
      }
      int64_t pos = s_base + before + incl - pc;
      for (unsigned m = m8; m; m &= m - 1u) cols[pos++] = (int32_t)((unsigned)g[e] * 8u + (unsigned)(__ffs(m) - 1));
      __syncthreads();
      if (t == 0) s_base += tot;
      __syncthreads();
    }
  }
}

// fp64 brute force for rows whose candidate buffers overflowed.  Each row is
// split over kNwrSlices blocks of consecutive columns (grid = rows x slices, so
// a handful of heavy rows still fills the GPU); mode 0 stores every slice's
// count in bcnt and k_nwr_brute_sum totals them, mode 1 starts each slice at
// row_ptr[r] + the counts of the slices before it, so the columns come out
// ascending.  O1 per pair (ascending c, no FMA), exactly the oracle's test.
constexpr int kNwrSlices = 64;

__global__ void __launch_bounds__(256)
    k_nwr_brute(const float* __restrict__ Q, int64_t q_begin, const float* __restrict__ X,
                int64_t n, int d, int self_join, double phi, const int32_t* __restrict__ rows,
                int mode, int64_t* __restrict__ bcnt, const int64_t* __restrict__ row_ptr,
                int32_t* __restrict__ cols) {
  __shared__ int s_w[8];
  __shared__ int64_t s_base;
  extern __shared__ double s_xq1[];  // [d] the query row in fp64
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int slot = blockIdx.x, b = blockIdx.y;
  const int64_t r = rows[slot];
  const int64_t gi = q_begin + r;
  const float* xi = self_join ? X + gi * d : Q + r * d;
  for (int c = t; c < d; c += 256) s_xq1[c] = (double)xi[c];
  const int64_t j_begin = n * b / kNwrSlices, j_end = n * (b + 1) / kNwrSlices;
  if (t == 0) {
    int64_t base = 0;
    if (mode == 1) {
      base = row_ptr[r];
      for (int q = 0; q < b; ++q) base += bcnt[(int64_t)slot * kNwrSlices + q];
    }
    s_base = base;
  }
  __syncthreads();
  const bool v4 = (d & 3) == 0 && (reinterpret_cast<uintptr_t>(X) & 15) == 0;
  for (int64_t j0 = j_begin; j0 < j_end; j0 += 256) {
    const int64_t j = j0 + t;
    bool keep = false;
    if (j < j_end && !(self_join && j == gi)) {
      const float* xj = X + j * d;
      double acc = 0.0;
      if (v4) {
        const float4* x4 = reinterpret_cast<const float4*>(xj);
        for (int c4 = 0; c4 < (d >> 2); ++c4) {
          const float4 v = __ldg(x4 + c4);
          double tt = __dsub_rn(s_xq1[4 * c4 + 0], (double)v.x);
          acc = __dadd_rn(acc, __dmul_rn(tt, tt));
          tt = __dsub_rn(s_xq1[4 * c4 + 1], (double)v.y);
          acc = __dadd_rn(acc, __dmul_rn(tt, tt));
          tt = __dsub_rn(s_xq1[4 * c4 + 2], (double)v.z);
          acc = __dadd_rn(acc, __dmul_rn(tt, tt));
          tt = __dsub_rn(s_xq1[4 * c4 + 3], (double)v.w);
          acc = __dadd_rn(acc, __dmul_rn(tt, tt));
        }
      } else {
        for (int c = 0; c < d; ++c) {
          const double tt = __dsub_rn(s_xq1[c], (double)__ldg(xj + c));
          acc = __dadd_rn(acc, __dmul_rn(tt, tt));
        }
      }
      keep = acc <= phi;
    }
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) s_w[w] = __popc(m);
    __syncthreads();
    int before = 0, tot = 0;
    for (int q = 0; q < 8; ++q) {
      before += q < w ? s_w[q] : 0;
      tot += s_w[q];
    }
    if (mode == 1 && keep) cols[s_base + before + __popc(m & ((1u << lane) - 1u))] = (int32_t)j;
    __syncthreads();
    if (t == 0) s_base += tot;
    __syncthreads();
  }
  if (mode == 0 && t == 0) bcnt[(int64_t)slot * kNwrSlices + b] = s_base;
}

__global__ void k_nwr_brute_sum(const int32_t* __restrict__ rows, int nrows,
                                const int64_t* __restrict__ bcnt, int64_t* __restrict__ counts) {
  const int slot = blockIdx.x * blockDim.x + threadIdx.x;
  if (slot >= nrows) return;
  int64_t c = 0;
  for (int q = 0; q < kNwrSlices; ++q) c += bcnt[(int64_t)slot * kNwrSlices + q];
  counts[rows[slot]] = c;
}

// Exclusive scan of q int64 counts into row_ptr[0..q] (3 phases, 1024 per block).
__global__ void k_scan_part(const int64_t* __restrict__ c, int64_t q, int64_t* __restrict__ part) {
  __shared__ int64_t s[32];
  int64_t v = 0;
  for (int64_t i = (int64_t)blockIdx.x * 1024 + threadIdx.x; i < min(q, (int64_t)(blockIdx.x + 1) * 1024);
       i += blockDim.x)
    v += c[i];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s[w];
    part[blockIdx.x] = t;
  }
}
__global__ void k_scan_parts(int64_t* __restrict__ part, int nb, int64_t* __restrict__ total) {
  if (threadIdx.x == 0) {
    int64_t acc = 0;
    for (int b = 0; b < nb; ++b) {
      const int64_t v = part[b];
      part[b] = acc;
      acc += v;
    }
    *total = acc;
  }
}
__global__ void k_scan_final(const int64_t* __restrict__ c, int64_t q, const int64_t* __restrict__ part,
                             const int64_t* __restrict__ total, int64_t* __restrict__ row_ptr) {
  __shared__ int64_t s[1024];
  const int64_t i0 = (int64_t)blockIdx.x * 1024;
  for (int e = threadIdx.x; e < 1024; e += blockDim.x) s[e] = (i0 + e < q) ? c[i0 + e] : 0;
  __syncthreads();
  if (threadIdx.x == 0) {  // 1024 sequential adds per block: cheap next to the passes
    int64_t acc = part[blockIdx.x];
    for (int e = 0; e < 1024; ++e) {
      const int64_t v = s[e];
      s[e] = acc;
      acc += v;
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < 1024; e += blockDim.x)
    if (i0 + e < q) row_ptr[i0 + e] = s[e];
  if (blockIdx.x == 0 && threadIdx.x == 0) row_ptr[q] = *total;
}

// ---------------------------------------------------------------- fallback
// Brute-force fp64 tier for rows the certificate could not prove ("recalculate
// on the subset").  Phase 1: grid (P slices x failing rows); block
// (p, f) scans the reference slice p for row f with the oracle's D64 formula,
// per-thread sorted top-k, block k-way merge -> k partial results.  Phase 2:
// one block per failing row merges the P sorted partial lists.  Spreading a
// row over P SMs makes a handful of failures cost one pass over X, not one
// SM's bandwidth.
constexpr int kFbThreads = 256;
constexpr int kFbCap = 1024;   // collected columns per failing row (threshold tier)
constexpr int kFbQB = 16;      // failing rows per block of the collect kernel

// Threshold tier of the fallback: every column whose D64 (oracle formula O1)
// is <= ub_f -- an upper bound on row f's k-th distance handed over by the
// re-rank -- is collected; the k smallest of them are the row's answer.  Each
// block scans one reference slice for kFbQB failing rows, so X is read once per
// row group; appends are warp-aggregated.
__global__ void __launch_bounds__(kFbThreads)
    k_fb_collect(const float* __restrict__ Q, int64_t q_begin, const float* __restrict__ X,
                 int64_t n, int d, int self_join, const int32_t* __restrict__ fail_rows,
                 const double* __restrict__ fail_ub, int nfail, int P,
                 double* __restrict__ ck, int* __restrict__ ci, int* __restrict__ ccnt) {
  // A cheap fp32 screen first (difference form, one FFMA per term: |D~ - rho^2| <=
  // gamma_{d+2}(2^-24) rho^2, the SIMT pass's bound), then the oracle's fp64 O1
  // only for columns that can be at or below the row's bound -- the exact
  // evaluation decides, the screen only skips columns that provably cannot.
  extern __shared__ float s_q32[];  // [kFbQB][d] query rows (fp32, exact)
  const int t = threadIdx.x, lane = t & 31;
  const int p = blockIdx.y, f0 = blockIdx.x * kFbQB;  // x: row groups (large), y: slices
  const int nq = min(kFbQB, nfail - f0);
  int64_t gq[kFbQB];
  double ub[kFbQB];
  float thr[kFbQB];
  const double g32 = gamma_up(d + 2, 5.9604644775390625e-08);
  const double g64 = gamma_up(d + 2, 1.1102230246251565e-16);
#pragma unroll
  for (int q = 0; q < kFbQB; ++q) {
    const int f = f0 + (q < nq ? q : 0);
    const int64_t r = fail_rows[f];
    gq[q] = q_begin + r;
    ub[q] = q < nq ? fail_ub[f] : -1.0;
    // D64 <= ub  =>  rho^2 <= ub / (1 - g64)  =>  D~ <= ub (1 + g32) / (1 - g64)
    const double th = ub[q] * (1.0 + g32) / (1.0 - g64) * (1.0 + 9.5367431640625e-07) +
                      (d + 2) * 1.1754943508222875e-38;
    thr[q] = q < nq ? __double2float_ru(th) : -1.0f;
    const float* xi = self_join ? X + gq[q] * d : Q + r * d;
    for (int c = t; c < d; c += kFbThreads) s_q32[q * d + c] = xi[c];
  }
  __syncthreads();
  const int64_t j_lo = n * p / P, j_hi = n * (p + 1) / P;
  const bool vec8 = (d & 7) == 0 && (reinterpret_cast<uintptr_t>(X) & 31) == 0;
  for (int64_t jb = j_lo; jb < j_hi; jb += kFbThreads) {
    const int64_t j = jb + t;
    float acc[kFbQB];
#pragma unroll
    for (int q = 0; q < kFbQB; ++q) acc[q] = 0.0f;
    const float* xj = X + (j < j_hi ? j : j_lo) * d;
    if (j < j_hi) {
      if (vec8) {
        for (int c8 = 0; c8 < d; c8 += 8) {
          float v[8];
          ldg8(xj + c8, v);
#pragma unroll
          for (int u = 0; u < 8; ++u)
#pragma unroll
            for (int q = 0; q < kFbQB; ++q) {
              const float tt = s_q32[q * d + c8 + u] - v[u];
              acc[q] = fmaf(tt, tt, acc[q]);
            }
        }
      } else {
        for (int c = 0; c < d; ++c) {
          const float xv = __ldg(xj + c);
#pragma unroll
          for (int q = 0; q < kFbQB; ++q) {
            const float tt = s_q32[q * d + c] - xv;
            acc[q] = fmaf(tt, tt, acc[q]);
          }
        }
      }
    }
#pragma unroll
    for (int q = 0; q < kFbQB; ++q) {
      bool keep = false;
      double dd = 0.0;
      // NaN / inf (fp32 overflow) also go to the exact evaluation
      if (j < j_hi && !(self_join && j == gq[q]) && !(acc[q] > thr[q])) {
        const float* xi = s_q32 + q * d;
        double a64 = 0.0;  // O1: ascending c, no FMA
        for (int c = 0; c < d; ++c) {
          const double tt = __dsub_rn((double)xi[c], (double)__ldg(xj + c));
          a64 = __dadd_rn(a64, __dmul_rn(tt, tt));
        }
        dd = a64;
        keep = a64 <= ub[q];
      }
      const unsigned m = __ballot_sync(0xffffffffu, keep);
      if (m) {
        int base = 0;
        if (lane == 0) base = atomicAdd(ccnt + f0 + q, __popc(m));
        base = __shfl_sync(0xffffffffu, base, 0);
        const int pos = base + __popc(m & ((1u << lane) - 1u));
        if (keep && pos < kFbCap) {
          ck[(int64_t)(f0 + q) * kFbCap + pos] = dd;
          ci[(int64_t)(f0 + q) * kFbCap + pos] = (int)j;
        }
      }
    }
  }
}

// One warp per failing row: the k smallest collected columns by (D64, index).
// Rows whose collection is unusable (fewer than k, or more than kFbCap) are
// left to the block brute-force tier (done = 0).
__global__ void __launch_bounds__(128)
    k_fb_select(int k, const int32_t* __restrict__ fail_rows, int nfail,
                double* __restrict__ ck, int* __restrict__ ci, const int* __restrict__ ccnt,
                int* __restrict__ done, KnnOutDev out) {
  __shared__ double s_tk[4][kMaxK];
  __shared__ int s_ti[4][kMaxK];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int f = blockIdx.x * 4 + w;
  if (f >= nfail) return;
  const int c = ccnt[f];
  if (c < k || c > kFbCap) {
    if (lane == 0) done[f] = 0;
    return;
  }
  double* bk = ck + (int64_t)f * kFbCap;
  int* bi = ci + (int64_t)f * kFbCap;
  double* tk = s_tk[w];
  int* ti = s_ti[w];
  if (c <= 64) {
    double kk[2];
    int ii[2];
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int p = 2 * lane + e;
      kk[e] = p < c ? bk[p] : CUDART_INF;
      ii[e] = p < c ? bi[p] : INT32_MAX;
    }
    warp_sort64(kk, ii, lane);
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int p = 2 * lane + e;
      if (p < k) {
        tk[p] = kk[e];
        ti[p] = ii[e];
      }
    }
  } else {
    auto slice_min = [&](double& mk, int& mi, int& mp) {
      mk = CUDART_INF;
      mi = INT32_MAX;
      mp = -1;
      for (int e = lane; e < c; e += 32)
        if (key_less(bk[e], bi[e], mk, mi)) {
          mk = bk[e];
          mi = bi[e];
          mp = e;
        }
    };
    double lk;
    int li, lp;
    slice_min(lk, li, lp);
    for (int m = 0; m < k; ++m) {
      double b = lk;
      int b2 = li;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ok = __shfl_xor_sync(0xffffffffu, b, o);
        const int oi = __shfl_xor_sync(0xffffffffu, b2, o);
        if (key_less(ok, oi, b, b2)) {
          b = ok;
          b2 = oi;
        }
      }
      if (lane == 0) {
        tk[m] = b;
        ti[m] = b2;
      }
      if (lp >= 0 && li == b2 && b2 != INT32_MAX) {
        bk[lp] = CUDART_INF;
        bi[lp] = INT32_MAX;
        slice_min(lk, li, lp);
      }
    }
  }
  __syncwarp();
  write_row(out, fail_rows[f], k, tk, ti, lane, 32);
  if (lane == 0) done[f] = 1;
}



template <int KMAX>
__global__ void __launch_bounds__(kFbThreads)
    k_fallback_part(const float* __restrict__ Q, int64_t q_begin, const float* __restrict__ X,
                    int64_t n, int d, int k, int self_join, const int32_t* __restrict__ fail_rows,
                    int P, const int* __restrict__ done, double* __restrict__ part_key,
                    int* __restrict__ part_id) {
  if (done[blockIdx.x]) return;  // answered by the threshold tier
  __shared__ double s_hk[kFbThreads / 32];
  __shared__ int s_hi[kFbThreads / 32];
  __shared__ int s_ht[kFbThreads / 32];
  __shared__ int s_win;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int p = blockIdx.y, f = blockIdx.x;  // x: failing rows (large), y: slices
  const int64_t r = fail_rows[f];
  const int64_t gi = q_begin + r;
  const float* xi = self_join ? X + gi * d : Q + r * d;
  const int64_t j_lo = n * p / P, j_hi = n * (p + 1) / P;
  double lk[KMAX];
  int li[KMAX];
  int cnt = 0;
  for (int64_t j = j_lo + t; j < j_hi; j += kFbThreads) {
    if (self_join && j == gi) continue;
    const double key = d64_row(xi, X + j * d, d);
    const int jj = (int)j;
    if (cnt < k || key_less(key, jj, lk[cnt - 1], li[cnt - 1])) {
      int q = cnt < k ? cnt : k - 1;
      while (q > 0 && key_less(key, jj, lk[q - 1], li[q - 1])) {
        lk[q] = lk[q - 1];
        li[q] = li[q - 1];
        --q;
      }
      lk[q] = key;
      li[q] = jj;
      if (cnt < k) ++cnt;
    }
  }
  double* ok_out = part_key + ((int64_t)f * P + p) * k;
  int* oi_out = part_id + ((int64_t)f * P + p) * k;
  // Block k-way merge: k rounds of lexicographic argmin over list heads.
  int head = 0;
  for (int m = 0; m < k; ++m) {
    double hk = head < cnt ? lk[head] : CUDART_INF;
    int hi = head < cnt ? li[head] : INT32_MAX;
    int ht = t;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ok = __shfl_xor_sync(0xffffffffu, hk, o);
      const int oi = __shfl_xor_sync(0xffffffffu, hi, o);
      const int ot = __shfl_xor_sync(0xffffffffu, ht, o);
      if (key_less(ok, oi, hk, hi)) {
        hk = ok;
        hi = oi;
        ht = ot;
      }
    }
    if (lane == 0) {
      s_hk[w] = hk;
      s_hi[w] = hi;
      s_ht[w] = ht;
    }
    __syncthreads();
    if (t == 0) {
      int b = 0;
      for (int q = 1; q < kFbThreads / 32; ++q)
        if (key_less(s_hk[q], s_hi[q], s_hk[b], s_hi[b])) b = q;
      ok_out[m] = s_hk[b];
      oi_out[m] = s_hi[b];
      s_win = s_ht[b];
    }
    __syncthreads();
    if (t == s_win) ++head;
    __syncthreads();
  }
}

constexpr int kFbMaxP = 64;

__global__ void __launch_bounds__(kFbMaxP)
    k_fallback_merge(int k, const int32_t* __restrict__ fail_rows, int P,
                     const int* __restrict__ done, const double* __restrict__ part_key,
                     const int* __restrict__ part_id, KnnOutDev out) {
  if (done[blockIdx.x]) return;
  __shared__ double s_key[kMaxK];
  __shared__ int s_id[kMaxK];
  __shared__ double s_hk[kFbMaxP / 32];
  __shared__ int s_hi[kFbMaxP / 32];
  __shared__ int s_ht[kFbMaxP / 32];
  __shared__ int s_win;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int f = blockIdx.x;
  const double* pk = part_key + ((int64_t)f * P + t) * k;
  const int* pi = part_id + ((int64_t)f * P + t) * k;
  int head = 0;
  for (int m = 0; m < k; ++m) {
    double hk = (t < P && head < k) ? pk[head] : CUDART_INF;
    int hi = (t < P && head < k) ? pi[head] : INT32_MAX;
    int ht = t;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const double ok = __shfl_xor_sync(0xffffffffu, hk, o);
      const int oi = __shfl_xor_sync(0xffffffffu, hi, o);
      const int ot = __shfl_xor_sync(0xffffffffu, ht, o);
      if (key_less(ok, oi, hk, hi)) {
        hk = ok;
        hi = oi;
        ht = ot;
      }
    }
    if (lane == 0) {
      s_hk[w] = hk;
      s_hi[w] = hi;
      s_ht[w] = ht;
    }
    __syncthreads();
    if (t == 0) {
      int b = 0;
      for (int q = 1; q < kFbMaxP / 32; ++q)
        if (key_less(s_hk[q], s_hi[q], s_hk[b], s_hi[b])) b = q;
      s_key[m] = s_hk[b];
      s_id[m] = s_hi[b];
      s_win = s_ht[b];
    }
    __syncthreads();
    if (t == s_win) ++head;
    __syncthreads();
  }
  if (w == 0) write_row(out, fail_rows[f], k, s_key, s_id, lane, 32);
}

}  // namespace

cudaError_t launch_nwr_tau(int64_t q_count, double phi, CertParams cp, float* tau,
                           cudaStream_t st, int* launches) {
  if (q_count <= 0) return cudaSuccess;
  k_nwr_tau<<<(unsigned)((q_count + 255) / 256), 256, 0, st>>>(q_count, phi, cp, tau);
  *launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_nwr_verify(const float* Q, int64_t q_begin, int64_t q_count, const float* X,
                              int64_t n, int d, bool self_join, double phi, const MainPass& mp,
                              int mode, int64_t* counts, const int64_t* row_ptr, int32_t* cols,
                              int32_t* ovf_rows, int32_t* ovf_count, int64_t* tasks_ws,
                              void* scan_ws, int num_sms, cudaStream_t st, int* launches) {
  if (q_count <= 0) return cudaSuccess;
  if (mp.parts * mp.cap > kNwrMaxG || mp.cap / kNwrChunk > 255) return cudaErrorInvalidValue;
  const unsigned rb = (unsigned)((q_count + 255) / 256);
  if (mode == 1) {
    // tasks_ws: reused for the dense-row queue ([0] count, then row ids)
    int32_t* nheavy = reinterpret_cast<int32_t*>(tasks_ws);
    int32_t* heavy = nheavy + 1;
    cudaError_t e = cudaMemsetAsync(nheavy, 0, 4, st);
    if (e != cudaSuccess) return e;
    k_nwr_emit<<<(unsigned)((q_count + kEmitWarps - 1) / kEmitWarps), kEmitWarps * 32, 0, st>>>(
        q_count, mp.buf, mp.cnt, mp.cap, mp.parts, row_ptr, cols, heavy, nheavy);
    const size_t smem = (size_t)2 * kNwrMaxG * 4;
    e = cudaFuncSetAttribute(k_nwr_emit_heavy, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_nwr_emit_heavy<<<(unsigned)(num_sms * 2), kEmitHeavyThreads, smem, st>>>(
        mp.buf, mp.cnt, mp.cap, mp.parts, row_ptr, cols, heavy, nheavy);
    *launches += 2;
    return cudaGetLastError();
  }
  // tasks_ws: [q_count] task counts, [q_count + 1] offsets, then the task map
  int64_t* tcnt = tasks_ws;
  int64_t* toff = tasks_ws + q_count;
  int64_t* map = toff + q_count + 1;
  k_nwr_tasks<<<rb, 256, 0, st>>>(q_count, mp.cnt, mp.cap, mp.parts, tcnt, counts, ovf_rows, ovf_count);
  cudaError_t e = launch_scan(tcnt, q_count, toff, scan_ws, st, launches);
  if (e != cudaSuccess) return e;
  k_nwr_map<<<rb, 256, 0, st>>>(q_count, mp.cnt, mp.cap, mp.parts, toff, map);
  const size_t smem = (size_t)kNwrWarps * d * 8;
  const bool al = ((reinterpret_cast<uintptr_t>(X) & 31) == 0);
  auto kern = (al && d == 16) ? k_nwr_mask<16>
            : (al && d == 32) ? k_nwr_mask<32>
            : (al && d == 64) ? k_nwr_mask<64> : k_nwr_mask<0>;
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  kern<<<(unsigned)(num_sms * 16), kNwrWarps * 32, smem, st>>>(
      Q, q_begin, X, n, d, self_join ? 1 : 0, phi, mp.buf, mp.cnt, mp.cap, mp.parts, map,
      toff + q_count, counts);
  *launches += 3;
  return cudaGetLastError();
}

// int64 words of the mode-0 task workspace
size_t nwr_tasks_ws(int64_t q_count, const MainPass& mp) {
  return (size_t)(2 * q_count + 1) +
         (size_t)q_count * mp.parts * ((mp.cap + kNwrChunk - 1) / kNwrChunk);
}

cudaError_t launch_nwr_brute(const float* Q, int64_t q_begin, const float* X, int64_t n, int d,
                             bool self_join, double phi, const int32_t* rows, int nrows, int mode,
                             int64_t* counts, const int64_t* row_ptr, int32_t* cols, int64_t* bcnt,
                             cudaStream_t st, int* launches) {
  if (nrows <= 0) return cudaSuccess;
  const size_t smem = (size_t)d * 8;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(k_nwr_brute, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  k_nwr_brute<<<dim3((unsigned)nrows, kNwrSlices), 256, smem, st>>>(
      Q, q_begin, X, n, d, self_join ? 1 : 0, phi, rows, mode, bcnt, row_ptr, cols);
  *launches += 1;
  if (mode == 0) {
    k_nwr_brute_sum<<<(unsigned)((nrows + 127) / 128), 128, 0, st>>>(rows, nrows, bcnt, counts);
    *launches += 1;
  }
  return cudaGetLastError();
}

int nwr_brute_slices() { return kNwrSlices; }

cudaError_t launch_gather_rows(const float* src, int64_t base, const int32_t* rows, int nr, int d,
                               float* dst, cudaStream_t st, int* launches) {
  if (nr <= 0) return cudaSuccess;
  const int64_t tot = (int64_t)nr * d;
  k_gather_rows<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(src, base, rows, nr, d, dst);
  *launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_mark_rows(const int32_t* rows, int nr, int32_t value, int32_t* dst,
                             cudaStream_t st, int* launches) {
  if (nr <= 0) return cudaSuccess;
  k_mark_rows<<<(nr + 255) / 256, 256, 0, st>>>(rows, nr, value, dst);
  *launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_tier2_scatter(const int32_t* rows, int nr, int64_t q_begin, bool self_join, int k,
                                 int k2, const int64_t* idx2, const double* dd2, KnnOutDev out,
                                 cudaStream_t st, int* launches) {
  if (nr <= 0) return cudaSuccess;
  k_tier2_scatter<<<(unsigned)((nr + 3) / 4), 128, 0, st>>>(rows, nr, q_begin, self_join ? 1 : 0, k,
                                                           k2, idx2, dd2, out);
  *launches += 1;
  return cudaGetLastError();
}

size_t scan_workspace(int64_t q) { return (size_t)((q + 1023) / 1024 + 2) * 8; }

cudaError_t launch_scan(const int64_t* counts, int64_t q, int64_t* row_ptr, void* ws,
                        cudaStream_t st, int* launches) {
  const int nb = (int)((q + 1023) / 1024);
  int64_t* part = static_cast<int64_t*>(ws);
  int64_t* total = part + nb + 1;
  if (nb == 0) return cudaMemsetAsync(row_ptr, 0, 8, st);
  k_scan_part<<<nb, 256, 0, st>>>(counts, q, part);
  k_scan_parts<<<1, 32, 0, st>>>(part, nb, total);
  k_scan_final<<<nb, 256, 0, st>>>(counts, q, part, total, row_ptr);
  *launches += 3;
  return cudaGetLastError();
}

int rerank_use_split(int d) {
  const char* se = getenv("TOD_RR_SPLIT");  // experiment knob: 0 / 1 forces the choice
  return se ? atoi(se) != 0 : d > 256;
}

size_t rerank_split_ws(int64_t q) {
  size_t total = 0;
  (void)rr_layout(nullptr, q, &total);
  return total;
}

cudaError_t launch_rerank(const float* Q, int64_t q_begin, int64_t q_count, const float* X,
                          int64_t n, int d, int k, bool self_join, Cands c, const MainPass* mp,
                          CertParams cp, KnnOutDev out, int32_t* fail_rows, double* fail_ub,
                          int32_t* fail_count, double* max_err, unsigned long long* counters,
                          void* split_ws, cudaStream_t st, int* launches) {
  if (k > kMaxK) return cudaErrorInvalidValue;
  if (cp.kind == PASS_TC) {  // group (or column) candidates
    if (c.lists * c.kp > kSelMax || !c.key) return cudaErrorInvalidValue;
    cp.colmode = mp ? mp->colmode : 0;
    if (cp.colmode && n >= kColFlag) return cudaErrorInvalidValue;  // tagged column indices
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    // Split form for wide rows only: measured on B200, C5 width (d = 512, k = 50) 83 -> 57 ms
    // at n = 2e5; slower at d <= 256 (C2 0.61 -> 0.79 ms, d = 128 5.7 -> 6.5 ms), where the
    // per-row gathers are short and the extra passes over the row state cost more.
    if (split_ws && rerank_use_split(d)) {
      if (q_count <= 0) return cudaSuccess;
      const RrWs rw = rr_layout(split_ws, q_count);
      const unsigned rb = (unsigned)std::min<int64_t>((q_count + kGrpWarps - 1) / kGrpWarps, (int64_t)sms * 8);
      k_rr_plan<<<rb, kGrpWarps * 32, 0, st>>>(q_count, k, c.idx, c.key, c.v, c.kp, c.lists,
                                              mp ? mp->buf : nullptr, mp ? mp->cnt : nullptr,
                                              mp ? mp->cap : 0, mp ? mp->parts : 0, cp, rw);
      cudaError_t e = launch_scan(rw.tcnt, q_count, rw.toff, rw.scan, st, launches);
      if (e != cudaSuccess) return e;
      k_rr_map<<<(unsigned)((q_count + 255) / 256), 256, 0, st>>>(q_count, rw);
      const size_t smem = (size_t)kGrpWarps * d * 8;
      if (smem > 160 * 1024) return cudaErrorInvalidValue;
      const bool al = ((reinterpret_cast<uintptr_t>(X) & 31) == 0);
      auto kx = (al && d == 16) ? k_rr_expand<16>
              : (al && d == 32) ? k_rr_expand<32>
              : (al && d == 64) ? k_rr_expand<64>
              : (al && d == 128) ? k_rr_expand<128>
              : (al && d == 256) ? k_rr_expand<256>
              : (al && d == 512) ? k_rr_expand<512> : k_rr_expand<0>;
      e = cudaFuncSetAttribute(kx, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      if (e != cudaSuccess) return e;
      kx<<<(unsigned)(sms * 16), kGrpWarps * 32, smem, st>>>(Q, q_begin, X, n, d, self_join ? 1 : 0,
                                                             rw, rw.toff + q_count);
      k_rr_finish<<<rb, kGrpWarps * 32, 0, st>>>(q_count, k, cp, rw, out, fail_rows, fail_ub,
                                                fail_count,
                                                reinterpret_cast<unsigned long long*>(max_err),
                                                counters);
      *launches += 4;
      return cudaGetLastError();
    }
    int mult = 8;
    if (const char* e = getenv("TOD_RR_GRID")) mult = std::max(1, atoi(e));  // experiment knob
    const int64_t gb = std::min<int64_t>((q_count + kGrpWarps - 1) / kGrpWarps, (int64_t)sms * mult);
    if (gb == 0) return cudaSuccess;
    const size_t smem = (size_t)kGrpWarps * d * 8;
    if (smem > 160 * 1024) return cudaErrorInvalidValue;
    // compile-time d for the common widths (32-byte aligned rows), else generic
    const bool al = ((reinterpret_cast<uintptr_t>(X) & 31) == 0);
    auto kern = (al && d == 16) ? k_rerank_groups<16>
              : (al && d == 32) ? k_rerank_groups<32>
              : (al && d == 64) ? k_rerank_groups<64>
              : (al && d == 128) ? k_rerank_groups<128>
              : (al && d == 256) ? k_rerank_groups<256>
              : (al && d == 512) ? k_rerank_groups<512> : k_rerank_groups<0>;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    kern<<<(unsigned)gb, kGrpWarps * 32, smem, st>>>(
        Q, q_begin, q_count, X, n, d, k, self_join ? 1 : 0, c.idx, c.key, c.v, c.kp, c.lists,
        mp ? mp->buf : nullptr, mp ? mp->cnt : nullptr, mp ? mp->cap : 0, mp ? mp->parts : 0, cp,
        out, fail_rows,
        fail_ub, fail_count, reinterpret_cast<unsigned long long*>(max_err), counters);
    *launches += 1;
    return cudaGetLastError();
  }
  if (c.lists * c.kp > kMaxCands) return cudaErrorInvalidValue;
  const int64_t blocks = (q_count + kRerankWarps - 1) / kRerankWarps;
  if (blocks == 0) return cudaSuccess;
  k_rerank<<<(unsigned)blocks, kRerankWarps * 32, 0, st>>>(
      Q, q_begin, q_count, X, n, d, k, self_join ? 1 : 0, c.idx, c.v, c.kp, c.lists, cp, out,
      fail_rows, fail_ub, fail_count, reinterpret_cast<unsigned long long*>(max_err));
  *launches += 1;
  return cudaGetLastError();
}

constexpr int kFbThrMaxRows = 65536;  // larger failure sets skip the threshold tier

size_t fallback_workspace(int nfail, int k, int64_t n, int num_sms) {
  const int P = fallback_slices(nfail, n, num_sms);
  const size_t thr = nfail <= kFbThrMaxRows ? (size_t)nfail * kFbCap * 12 : 0;
  return (size_t)nfail * P * k * (sizeof(double) + sizeof(int)) + thr + (size_t)nfail * 8 + 64;
}

int fallback_slices(int nfail, int64_t n, int num_sms) {
  int P = (4 * num_sms + nfail - 1) / nfail;
  P = P > kFbMaxP ? kFbMaxP : P;
  while (P > 1 && n / P < 2048) --P;
  return P < 1 ? 1 : P;
}

cudaError_t launch_fallback(const float* Q, int64_t q_begin, const float* X, int64_t n, int d,
                            int k, bool self_join, const int32_t* fail_rows,
                            const double* fail_ub, int nfail, KnnOutDev out, void* ws,
                            int num_sms, cudaStream_t st, int* launches) {
  if (nfail <= 0) return cudaSuccess;
  if (k > kMaxK) return cudaErrorInvalidValue;
  const int P = fallback_slices(nfail, n, num_sms);
  const bool thr = nfail <= kFbThrMaxRows && (size_t)kFbQB * d * 4 <= 96 * 1024;
  // workspace: [ck nfail*cap f64][pk nfail*P*k f64][pi nfail*P*k i32][ci nfail*cap i32][done][ccnt]
  double* ck = static_cast<double*>(ws);
  double* pk = ck + (thr ? (size_t)nfail * kFbCap : 0);
  int* pi = reinterpret_cast<int*>(pk + (size_t)nfail * P * k);
  int* ci = pi + (size_t)nfail * P * k;
  int* done = ci + (thr ? (size_t)nfail * kFbCap : 0);
  int* ccnt = done + nfail;
  cudaError_t e = cudaMemsetAsync(done, 0, (size_t)nfail * 8, st);  // done and ccnt
  if (e != cudaSuccess) return e;
  if (thr) {
    const int qb = (nfail + kFbQB - 1) / kFbQB;
    int Pt = (4 * num_sms + qb - 1) / qb;
    while (Pt > 1 && n / Pt < 1024) --Pt;
    if (Pt < 1) Pt = 1;
    const size_t smem = (size_t)kFbQB * d * 4;
    e = cudaFuncSetAttribute(k_fb_collect, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    k_fb_collect<<<dim3(qb, Pt), kFbThreads, smem, st>>>(Q, q_begin, X, n, d, self_join ? 1 : 0,
                                                          fail_rows, fail_ub, nfail, Pt, ck, ci,
                                                          ccnt);
    k_fb_select<<<(nfail + 3) / 4, 128, 0, st>>>(k, fail_rows, nfail, ck, ci, ccnt, done, out);
    *launches += 2;
  }
  const dim3 grid(nfail, P);
  if (k <= 32)
    k_fallback_part<32><<<grid, kFbThreads, 0, st>>>(Q, q_begin, X, n, d, k, self_join ? 1 : 0,
                                                     fail_rows, P, done, pk, pi);
  else if (k <= 64)
    k_fallback_part<64><<<grid, kFbThreads, 0, st>>>(Q, q_begin, X, n, d, k, self_join ? 1 : 0,
                                                     fail_rows, P, done, pk, pi);
  else
    k_fallback_part<kMaxK><<<grid, kFbThreads, 0, st>>>(Q, q_begin, X, n, d, k,
                                                        self_join ? 1 : 0, fail_rows, P, done, pk,
                                                        pi);
  k_fallback_merge<<<nfail, kFbMaxP, 0, st>>>(k, fail_rows, P, done, pk, pi, out);
  *launches += 2;
  return cudaGetLastError();
}

}  // namespace tod
