// lof.cu — K5: the LOF stage on top of the exact kNN table (Table 1 P:158,
// P:184, Breunig et al. 2000; O4, readings A5/A6).  fp64 with the
// oracle's operation order (sequential sums over the k neighbours, explicit
// _rn intrinsics: no FMA), so results are bit-identical to oracle/.
// Memory-bound gathers; one thread per row.
#include <math_constants.h>

#include "internal.h"

namespace tod {

namespace {

__global__ void k_lof_lrd(int64_t q_count, int k, const int64_t* __restrict__ idx,
                          const double* __restrict__ dist64, const double* __restrict__ kdist_all,
                          double* __restrict__ lrd_out) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= q_count) return;
  double s = 0.0;
  for (int m = 0; m < k; ++m) {
    const double reach = fmax(kdist_all[idx[r * k + m]], dist64[r * k + m]);
    s = __dadd_rn(s, reach);
  }
  lrd_out[r] = s > 0.0 ? __ddiv_rn((double)k, s) : CUDART_INF;
}

__global__ void k_lof_finish(int64_t q_begin, int64_t q_count, int k,
                             const int64_t* __restrict__ idx, const double* __restrict__ lrd_all,
                             float* __restrict__ lof_out, float* __restrict__ lrd_out) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= q_count) return;
  const double lp = lrd_all[q_begin + r];
  double ls = 0.0;
  for (int m = 0; m < k; ++m) ls = __dadd_rn(ls, lrd_all[idx[r * k + m]]);
  double lof;
  if (isinf(lp))
    lof = 1.0;  // reading A6: >= k duplicates of p
  else
    lof = __ddiv_rn(ls, __dmul_rn((double)k, lp));
  if (lof_out) lof_out[r] = __double2float_rn(lof);
  if (lrd_out) lrd_out[r] = __double2float_rn(lp);
}

}  // namespace

cudaError_t launch_lof_lrd(int64_t q_count, int k, const int64_t* idx, const double* dist64,
                           const double* kdist64_all, double* lrd64_out, cudaStream_t st,
                           int* launches) {
  if (q_count <= 0) return cudaSuccess;
  k_lof_lrd<<<(unsigned)((q_count + 255) / 256), 256, 0, st>>>(q_count, k, idx, dist64,
                                                               kdist64_all, lrd64_out);
  *launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_lof_finish(int64_t q_begin, int64_t q_count, int k, const int64_t* idx,
                              const double* lrd64_all, float* lof_out, float* lrd_out,
                              cudaStream_t st, int* launches) {
  if (q_count <= 0) return cudaSuccess;
  k_lof_finish<<<(unsigned)((q_count + 255) / 256), 256, 0, st>>>(q_begin, q_count, k, idx,
                                                                  lrd64_all, lof_out, lrd_out);
  *launches += 1;
  return cudaGetLastError();
}

}  // namespace tod
