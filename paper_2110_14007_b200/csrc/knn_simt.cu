// knn_simt.cu — K2s: CUDA-core fp32 tile path for small d (north_star part 1:
// "a CUDA-core fp32 tile path for small d") and for TOD_FMT_FP32.
//
// Distance form: the difference form D~_ij = sum_c (x_ic - x_jc)^2 in fp32
// (recursive, one FFMA per term), NOT Eq. (3)'s norm expansion.  The paper
// picks the expansion for GEMM-friendliness; on CUDA cores the
// difference form costs the same two instructions per term and has a purely
// RELATIVE error |D~ - D| <= gamma_{d+2}(2^-24) D (all summands are >= 0), so
// its certificate (rerank.cu) is far tighter than any expansion bound.
//
// Thread = query row (x_i in registers), block = 128 query rows; reference
// rows are staged in shared memory 64 at a time and read as warp broadcasts;
// the per-row top-K' is the same RowTopK list as the tensor-core kernel.
#include <math_constants.h>

#include "internal.h"
#include "topk_list.cuh"

namespace tod {

namespace {

constexpr int kRowsQ = 128;   // query rows per block (= threads)
constexpr int kRowsR = 64;    // reference rows per smem tile

template <int DMAX>
__global__ void __launch_bounds__(kRowsQ)
    k_knn_simt(const float* __restrict__ Q, int64_t q_begin, int64_t q_count,
               const float* __restrict__ X, int64_t n, int d, int self_join, int S, int kp,
               int32_t* __restrict__ cand_idx, float* __restrict__ cand_v) {
  extern __shared__ float smem_f[];
  float* sR = smem_f;                                       // [kRowsR][DMAX]
  uint2* sL = reinterpret_cast<uint2*>(sR + kRowsR * DMAX);  // [(kp+P)][128] (key, index)
  const int t = threadIdx.x;
  const int64_t qtile = blockIdx.x / S;
  const int c = blockIdx.x % S;
  const int64_t r = qtile * kRowsQ + t;           // local query row
  const bool live = r < q_count;
  const int64_t gi = q_begin + r;                 // global row (self-join) / Q row index
  float xq[DMAX];
  const float* qrow = self_join ? X + gi * d : Q + r * d;
#pragma unroll
  for (int cc = 0; cc < DMAX; ++cc) xq[cc] = (live && cc < d) ? qrow[cc] : 0.f;
  const int self = self_join ? (int)gi : -1;

  RowTopK<kRowsQ> L;
  L.init(sL, t, kp);
  const int64_t j_lo = n * c / S, j_hi = n * (c + 1) / S;
  for (int64_t j0 = j_lo; j0 < j_hi; j0 += kRowsR) {
    const int rows = (int)(j_hi - j0 < kRowsR ? j_hi - j0 : kRowsR);
    __syncthreads();
    for (int e = t; e < kRowsR * DMAX; e += kRowsQ) {
      const int rr = e / DMAX, cc = e % DMAX;
      sR[e] = (rr < rows && cc < d) ? X[(j0 + rr) * d + cc] : 0.f;
    }
    __syncthreads();
    for (int jb = 0; jb < kRowsR; jb += 8) {
      float w[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float4* y = reinterpret_cast<const float4*>(sR + (jb + e) * DMAX);
        float acc = 0.f;
#pragma unroll
        for (int cc = 0; cc < DMAX / 4; ++cc) {
          const float4 yv = y[cc];
          float df = xq[4 * cc + 0] - yv.x;
          acc = fmaf(df, df, acc);
          df = xq[4 * cc + 1] - yv.y;
          acc = fmaf(df, df, acc);
          df = xq[4 * cc + 2] - yv.z;
          acc = fmaf(df, df, acc);
          df = xq[4 * cc + 3] - yv.w;
          acc = fmaf(df, df, acc);
        }
        w[e] = (jb + e < rows) ? acc : CUDART_INF_F;
      }
      const float m = fminf(fminf(fminf(w[0], w[1]), fminf(w[2], w[3])),
                            fminf(fminf(w[4], w[5]), fminf(w[6], w[7])));
      if (__any_sync(0xffffffffu, m < L.thr)) {
        L.reserve_group();
        L.offer_group(w, (int)(j0 + jb), self);
      }
    }
  }
  const float v = L.finish(cand_idx + (live ? (r * S + c) * kp : 0), live);
  if (live) cand_v[r * S + c] = v;
}

template <int DMAX>
cudaError_t launch_s(const float* Q, int64_t q_begin, int64_t q_count, const float* X, int64_t n,
                     int d, bool self_join, Cands c, cudaStream_t st) {
  const size_t smem = (size_t)kRowsR * DMAX * 4 + (size_t)(c.kp + RowTopK<kRowsQ>::kPend) * kRowsQ * 8;
  auto kern = k_knn_simt<DMAX>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  const int64_t qtiles = (q_count + kRowsQ - 1) / kRowsQ;
  const int64_t grid = qtiles * c.S;
  if (grid <= 0) return cudaSuccess;
  kern<<<(unsigned)grid, kRowsQ, smem, st>>>(Q, q_begin, q_count, X, n, d, self_join ? 1 : 0, c.S,
                                             c.kp, c.idx, c.v);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_knn_simt(const float* Q, int64_t q_begin, int64_t q_count, const float* X,
                            int64_t n, int d, bool self_join, Cands c, cudaStream_t st,
                            int* launches) {
  *launches += 1;
  if (d <= 16) return launch_s<16>(Q, q_begin, q_count, X, n, d, self_join, c, st);
  if (d <= 32) return launch_s<32>(Q, q_begin, q_count, X, n, d, self_join, c, st);
  if (d <= 64) return launch_s<64>(Q, q_begin, q_count, X, n, d, self_join, c, st);
  return cudaErrorInvalidValue;
}

}  // namespace tod
