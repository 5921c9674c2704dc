// rerank.cu — K3 re-rank + certificate (provable quantization step (iii),
// "verification", §5.2) and K4 fallback ("recalculate ...
// only on the subset of X where the verification fails").
//
// K3, one warp per query row: the K' (x S chunks) candidates of pass 1 are
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

#include <cstdint>

#include "internal.h"

namespace tod {

namespace {

constexpr int kRerankWarps = 8;
constexpr int kMaxCands = 256;   // S * K' per row
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

// Writes the k outputs of one row from ascending (key, id) arrays (fp64
// squared distances).  Lane-parallel over m; lane 0 does the sequential sums.
__device__ void write_row(const KnnOutDev& out, int64_t r, int k, const double* keys,
                          const int* ids, int lane, int nlanes) {
  for (int m = lane; m < k; m += nlanes) {
    const double dd = __dsqrt_rn(keys[m]);
    if (out.idx) out.idx[r * k + m] = ids[m];
    if (out.dist64) out.dist64[r * k + m] = dd;
    if (out.dist) out.dist[r * k + m] = __double2float_rn(dd);
  }
  if (lane == 0) {
    const double kth = __dsqrt_rn(keys[k - 1]);
    if (out.kdist64) out.kdist64[r] = kth;
    if (out.score_kth) out.score_kth[r] = __double2float_rn(kth);
    if (out.score_mean) {
      double acc = 0.0;
      for (int m = 0; m < k; ++m) acc = __dadd_rn(acc, __dsqrt_rn(keys[m]));
      out.score_mean[r] = __double2float_rn(__ddiv_rn(acc, (double)k));
    }
  }
}

__global__ void __launch_bounds__(kRerankWarps * 32)
    k_rerank(const float* __restrict__ Q, int64_t q_begin, int64_t q_count,
             const float* __restrict__ X, int64_t n, int d, int k, int self_join,
             const int32_t* __restrict__ cand_idx, const float* __restrict__ cand_v, int kp, int S,
             CertParams cp, KnnOutDev out, int32_t* __restrict__ fail_rows,
             int32_t* __restrict__ fail_count, unsigned long long* __restrict__ max_err_bits) {
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
  bool cert = false;
  double err = 0.0;
  if (nv_local >= k) {
    const double dk = s_sk[w][k - 1];
    const double u53 = 1.1102230246251565e-16;
    const double vv = (double)vmin;
    if (vmin == CUDART_INF_F) {
      cert = true;  // every reference was offered and kept: nothing outside
    } else if (cp.kind == PASS_TC) {
      // Tensor-core pass (fp16/bf16 operands, fp32 accumulation), DESIGN.md
      // "Certificate": |w~_ij - w_ij| <= E_i for every reference j, with
      // w_ij = ||xhat_j||^2 - 2 xhat_i.xhat_j exact, so non-kept j satisfy
      // ||xhat_i - xhat_j||^2 >= a_i^2 + v - E_i, then the triangle inequality
      // through the residuals e_i, e_j <= emax.
      const double a2i = cp.qa2[r];
      const double ei = cp.qe[r];
      const double amax2 = cp.g->amax2;
      const double emax = cp.g->emax;
      const double ai = sqrt(a2i) * (1.0 + 4 * u53);
      const double am = sqrt(amax2) * (1.0 + 4 * u53);
      const double gam = gamma_up(2.0 * cp.dpad, 2.384185791015625e-07 /*2^-22*/);
      const double E = (1.1920928955078125e-07 /*2^-23*/ * amax2 + 2.0 * gam * ai * am +
                        5.9604644775390625e-08 /*2^-24*/ * (amax2 + 2.0 * ai * am)) *
                           (1.0 + 9.5367431640625e-07 /*2^-20*/) +
                       1e-300;
      const double slack = (cp.d + 8) * 2.0 * u53 * (fabs(a2i) + fabs(vv) + E);
      const double R2 = a2i + vv - E - slack;
      err = E + slack;
      if (R2 > 0.0) {
        const double Rh = sqrt(R2) * (1.0 - 2.0 * u53);
        const double LB = (Rh - ei - emax) * (1.0 - 8.0 * u53);
        if (LB > 0.0) {
          const double lbo = LB / cp.g->s;  // s = 2^e: exact
          const double lb2 = lbo * lbo * (1.0 - 8.0 * u53);
          cert = dk < lb2 * (1.0 - gamma_up(cp.d + 2, u53));
        }
      }
    } else {
      // fp32 difference-form pass: D~ <= D (1 + gamma_{d+2}(2^-24)) + tiny.
      const double g32 = gamma_up(cp.d + 2, 5.9604644775390625e-08);
      const double lb2 =
          (vv - (cp.d + 2) * 1.1754943508222875e-38 /*2^-126*/) / (1.0 + g32) * (1.0 - 8.0 * u53);
      err = vv * g32;
      if (lb2 > 0.0) cert = dk < lb2 * (1.0 - gamma_up(cp.d + 2, u53));
    }
  }
  if (cp.force_fail) cert = false;
  if (lane == 0 && err > 0.0)
    atomicMax(max_err_bits, (unsigned long long)__double_as_longlong(err));
  if (cert) {
    write_row(out, r, k, s_sk[w], s_si[w], lane, 32);
  } else if (lane == 0) {
    const int slot = atomicAdd(fail_count, 1);
    fail_rows[slot] = (int32_t)r;
  }
}

// ---------------------------------------------------------------- fallback
constexpr int kFbThreads = 256;

template <int KMAX>
__global__ void __launch_bounds__(kFbThreads)
    k_fallback(const float* __restrict__ Q, int64_t q_begin, const float* __restrict__ X,
               int64_t n, int d, int k, int self_join, const int32_t* __restrict__ fail_rows,
               KnnOutDev out) {
  __shared__ double s_hk[kFbThreads / 32];
  __shared__ int s_hi[kFbThreads / 32];
  __shared__ int s_ht[kFbThreads / 32];
  __shared__ double s_key[KMAX];
  __shared__ int s_id[KMAX];
  __shared__ int s_win;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int64_t r = fail_rows[blockIdx.x];
  const int64_t gi = q_begin + r;
  const float* xi = self_join ? X + gi * d : Q + r * d;
  double lk[KMAX];
  int li[KMAX];
  int cnt = 0;
  for (int64_t j = t; j < n; j += kFbThreads) {
    if (self_join && j == gi) continue;
    const double key = d64_row(xi, X + j * d, d);
    const int jj = (int)j;
    if (cnt < k || key_less(key, jj, lk[cnt - 1], li[cnt - 1])) {
      int p = cnt < k ? cnt : k - 1;
      while (p > 0 && key_less(key, jj, lk[p - 1], li[p - 1])) {
        lk[p] = lk[p - 1];
        li[p] = li[p - 1];
        --p;
      }
      lk[p] = key;
      li[p] = jj;
      if (cnt < k) ++cnt;
    }
  }
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
      s_key[m] = s_hk[b];
      s_id[m] = s_hi[b];
      s_win = s_ht[b];
    }
    __syncthreads();
    if (t == s_win) ++head;
    __syncthreads();
  }
  if (w == 0) write_row(out, r, k, s_key, s_id, lane, 32);
}

}  // namespace

cudaError_t launch_rerank(const float* Q, int64_t q_begin, int64_t q_count, const float* X,
                          int64_t n, int d, int k, bool self_join, Cands c, CertParams cp,
                          KnnOutDev out, int32_t* fail_rows, int32_t* fail_count,
                          double* max_err, cudaStream_t st, int* launches) {
  if (c.S * c.kp > kMaxCands || k > kMaxK) return cudaErrorInvalidValue;
  const int64_t blocks = (q_count + kRerankWarps - 1) / kRerankWarps;
  if (blocks == 0) return cudaSuccess;
  k_rerank<<<(unsigned)blocks, kRerankWarps * 32, 0, st>>>(
      Q, q_begin, q_count, X, n, d, k, self_join ? 1 : 0, c.idx, c.v, c.kp, c.S, cp, out,
      fail_rows, fail_count, reinterpret_cast<unsigned long long*>(max_err));
  *launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_fallback(const float* Q, int64_t q_begin, const float* X, int64_t n, int d,
                            int k, bool self_join, const int32_t* fail_rows, int nfail,
                            KnnOutDev out, cudaStream_t st, int* launches) {
  if (nfail <= 0) return cudaSuccess;
  *launches += 1;
  if (k <= 32)
    k_fallback<32><<<nfail, kFbThreads, 0, st>>>(Q, q_begin, X, n, d, k, self_join ? 1 : 0,
                                                 fail_rows, out);
  else if (k <= 64)
    k_fallback<64><<<nfail, kFbThreads, 0, st>>>(Q, q_begin, X, n, d, k, self_join ? 1 : 0,
                                                 fail_rows, out);
  else if (k <= kMaxK)
    k_fallback<kMaxK><<<nfail, kFbThreads, 0, st>>>(Q, q_begin, X, n, d, k, self_join ? 1 : 0,
                                                    fail_rows, out);
  else
    return cudaErrorInvalidValue;
  return cudaGetLastError();
}

}  // namespace tod
