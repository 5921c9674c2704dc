// consumers.cu — detectors built on the kNN functional operator's output
// (§4.2 Fig. 3(a): "kNN FO ... then cosine similarity FO";
// Appendix B: kNN classifier = cdist -> topk -> vote).
//
// ABOD (Kriegel 2008, cited P:182; reading A20): for query row i
// with neighbours o_1..o_k (ascending (D64, index), the exact kNN of tod_knn),
// v_m = x_{o_m} - x_i in fp64, q_m = sum_c v_mc^2 sequential, and for each
// neighbour pair (a < b) with nonzero vectors w_ab = (sum_c v_ac v_bc) / (q_a q_b)
// (the distance-weighted angle factor); score = -(population variance of the
// w_ab), two-pass in pair order,
// every operation explicit RN fp64 (no FMA): the oracle's O6 op for op, so
// the fp32 scores are bit-identical.  One warp per row: lanes compute pairs,
// lane 0 folds the sums in pair order.
//
// kNN classifier (reading A21): majority label over the k neighbours, ties to
// the tied class whose first neighbour is nearest.
#include <cstdint>
#include <math_constants.h>

#include "internal.h"

namespace tod {

namespace {

constexpr int kAbodWarps = 4;
constexpr int kAbodMaxK = 48;

__global__ void __launch_bounds__(kAbodWarps * 32)
    k_abod(const float* __restrict__ X, int64_t q_begin, int64_t q_count, int d, int k,
           const int64_t* __restrict__ idx, float* __restrict__ score) {
  extern __shared__ double s_dyn[];  // [warps][k][d] neighbour vectors
  __shared__ double s_nrm[kAbodWarps][kAbodMaxK];
  __shared__ double s_cos[kAbodWarps][kAbodMaxK * (kAbodMaxK - 1) / 2];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * kAbodWarps + w;
  if (r >= q_count) return;
  double* V = s_dyn + (size_t)w * k * d;
  const float* xi = X + (q_begin + r) * d;
  for (int e = lane; e < k * d; e += 32) {
    const int m = e / d, c = e - m * d;
    const int64_t o = idx[r * k + m];
    V[e] = __dsub_rn((double)X[o * d + c], (double)xi[c]);
  }
  __syncwarp();
  for (int m = lane; m < k; m += 32) {
    double acc = 0.0;
    for (int c = 0; c < d; ++c) acc = __dadd_rn(acc, __dmul_rn(V[m * d + c], V[m * d + c]));
    s_nrm[w][m] = acc;  // squared norm
  }
  __syncwarp();
  const int npairs = k * (k - 1) / 2;
  // pair p <-> (a, b) lexicographic
  for (int p = lane; p < npairs; p += 32) {
    int a = 0, rem = p;
    while (rem >= k - 1 - a) {
      rem -= k - 1 - a;
      ++a;
    }
    const int b = a + 1 + rem;
    const double na = s_nrm[w][a], nb = s_nrm[w][b];
    double c = CUDART_NAN;  // NaN marks a skipped pair (coincident neighbour)
    // na, nb: squared norms q_a, q_b
    if (na > 0.0 && nb > 0.0) {
      double dot = 0.0;
      for (int t = 0; t < d; ++t) dot = __dadd_rn(dot, __dmul_rn(V[a * d + t], V[b * d + t]));
      c = __ddiv_rn(dot, __dmul_rn(na, nb));
    }
    s_cos[w][p] = c;
  }
  __syncwarp();
  if (lane == 0) {
    double s = 0.0;
    int P = 0;
    for (int p = 0; p < npairs; ++p) {
      const double c = s_cos[w][p];
      if (c == c) {
        s = __dadd_rn(s, c);
        ++P;
      }
    }
    float out = 0.f;
    if (P > 0) {
      const double mean = __ddiv_rn(s, (double)P);
      double s2 = 0.0;
      for (int p = 0; p < npairs; ++p) {
        const double c = s_cos[w][p];
        if (c == c) {
          const double t = __dsub_rn(c, mean);
          s2 = __dadd_rn(s2, __dmul_rn(t, t));
        }
      }
      out = __double2float_rn(-__ddiv_rn(s2, (double)P));
    }
    score[r] = out;
  }
}

__global__ void k_knn_classify(int64_t nq, int k, const int64_t* __restrict__ idx,
                               const int32_t* __restrict__ labels, int32_t* __restrict__ pred) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= nq) return;
  // k <= 128: count each neighbour's label among all k (O(k^2), tiny)
  int best = -1, bestc = 0;
  for (int m = 0; m < k; ++m) {
    const int l = labels[idx[r * k + m]];
    int c = 0;
    for (int t = 0; t < k; ++t) c += labels[idx[r * k + t]] == l;
    if (c > bestc) {  // strict: the earliest (nearest) class wins ties
      bestc = c;
      best = l;
    }
  }
  pred[r] = best;
}

}  // namespace

cudaError_t launch_abod(const float* X, int64_t q_begin, int64_t q_count, int d, int k,
                        const int64_t* idx, float* score, cudaStream_t st, int* launches) {
  if (q_count <= 0) return cudaSuccess;
  if (k < 1 || k > kAbodMaxK) return cudaErrorInvalidValue;
  const size_t smem = (size_t)kAbodWarps * k * d * 8;
  if (smem > 160 * 1024) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(k_abod, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  k_abod<<<(unsigned)((q_count + kAbodWarps - 1) / kAbodWarps), kAbodWarps * 32, smem, st>>>(
      X, q_begin, q_count, d, k, idx, score);
  *launches += 1;
  return cudaGetLastError();
}

int abod_max_k() { return kAbodMaxK; }

cudaError_t launch_knn_classify(int64_t nq, int k, const int64_t* idx, const int32_t* labels,
                                int32_t* pred, cudaStream_t st, int* launches) {
  if (nq <= 0) return cudaSuccess;
  k_knn_classify<<<(unsigned)((nq + 255) / 256), 256, 0, st>>>(nq, k, idx, labels, pred);
  *launches += 1;
  return cudaGetLastError();
}

}  // namespace tod
