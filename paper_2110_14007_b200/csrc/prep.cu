// prep.cu — K1: input quantization for the tensor-core pass (provable
// quantization step (i), §5.2), re-derived (DESIGN.md
// "Prep"): global translation mu (column mean, fp64, deterministic order),
// power-of-two scale s, x' = s*(x - mu), xhat = RN16(x'), written straight into
// the swizzled UMMA operand image; per-row fp64 ||xhat||^2, fp32 norm for the
// epilogue, and a rigorous per-row residual bound e_i >= ||xhat_i - x'_i||.
// The paper's per-column min-max scaling to [0,1] is NOT applied: it
// changes Euclidean neighbourhoods (reading A11).  All kernels are HBM-bound.
#include <cuda_fp16.h>
#include <cuda_bf16.h>
#include <math_constants.h>

#include "internal.h"

namespace tod {

namespace {

constexpr int kStatThreads = 256;
constexpr int kRowsPerStatBlock = 128;  // short fp64 add chains, many blocks

__device__ __forceinline__ void atomic_max_nonneg(unsigned long long* addr, double v) {
  // Non-negative doubles order like their bit patterns.
  atomicMax(addr, (unsigned long long)__double_as_longlong(v));
}

// Column partial sums over a fixed row range per block (fixed order => the
// result depends only on (X, n, d), never on timing).  Also the finite check.
__global__ void k_colsum_partial(const float* __restrict__ X, int64_t n, int d,
                                 double* __restrict__ partial, PrepGlobals* g) {
  __shared__ double red[kStatThreads];
  __shared__ int bad;
  if (threadIdx.x == 0) bad = 0;
  __syncthreads();
  const int t = threadIdx.x;
  const int nphase = d <= kStatThreads ? kStatThreads / d : 1;
  const int64_t r0 = (int64_t)blockIdx.x * kRowsPerStatBlock;
  const int64_t r1 = min(n, r0 + kRowsPerStatBlock);
  int mybad = 0;
  for (int cbase = 0; cbase < d; cbase += (d <= kStatThreads ? d : kStatThreads)) {
    const int c = d <= kStatThreads ? (t % d) : (cbase + t);
    const int rp = d <= kStatThreads ? (t / d) : 0;
    double s = 0.0;
    const bool active = (rp < nphase) && (c < d);
    if (active) {
      for (int64_t r = r0 + rp; r < r1; r += nphase) {
        const float v = X[r * d + c];
        mybad |= !isfinite(v);
        s += (double)v;
      }
    }
    red[t] = active ? s : 0.0;
    __syncthreads();
    if (d <= kStatThreads) {
      if (t < d) {
        double acc = 0.0;
        for (int p = 0; p < nphase; ++p) acc += red[p * d + t];
        partial[(int64_t)blockIdx.x * d + t] = acc;
      }
    } else if (c < d) {
      partial[(int64_t)blockIdx.x * d + c] = red[t];
    }
    __syncthreads();
    if (d <= kStatThreads) break;
  }
  if (mybad) bad = 1;
  __syncthreads();
  if (t == 0 && bad) atomicOr(&g->nonfinite, 1);
}

// One block (256 threads) per column: thread t sums partials t, t+256, ... in
// order, then a fixed-shape tree -- deterministic for a given (n, d).
__global__ void k_colmean(const double* __restrict__ partial, int blocks, int64_t n, int d,
                          double* __restrict__ mu) {
  __shared__ double red[256];
  const int c = blockIdx.x;
  double acc = 0.0;
  for (int b = threadIdx.x; b < blocks; b += 256) acc += partial[(int64_t)b * d + c];
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) mu[c] = red[0] / (double)n;
}

__global__ void k_finite(const float* __restrict__ X, int64_t total, PrepGlobals* g) {
  int bad = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x)
    bad |= !isfinite(X[i]);
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(&g->nonfinite, 1);
}

__global__ void k_absmax(const float* __restrict__ X, int64_t n, int d,
                         const double* __restrict__ mu, PrepGlobals* g) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  __shared__ unsigned long long s_m;
  if (threadIdx.x == 0) s_m = 0ull;
  __syncthreads();
  double m = 0.0;
  for (int64_t r = warp; r < n; r += nwarps)
    for (int c = lane; c < d; c += 32) m = fmax(m, fabs((double)X[r * d + c] - mu[c]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) atomic_max_nonneg(&s_m, m);   // block-local first: one global atomic per block
  __syncthreads();
  if (threadIdx.x == 0 && s_m) atomicMax(&g->absmax_bits, s_m);
}

// s = 2^e with max|s*(x-mu)| in [2^(E-1), 2^E), E = floor((30 - log2 dpad)/2),
// so every ||xhat||^2 <= dpad * 2^(2E) <= 2^30: the fp16 norm pieces below stay
// in range (fp16 max 65504) and all fp32 accumulations stay far from overflow.
__global__ void k_scale(PrepGlobals* g, int fmt, int dpad) {
  const double amax = __longlong_as_double((long long)g->absmax_bits);
  int lg = 0;
  while ((1 << lg) < dpad) ++lg;
  const int E = (30 - lg) / 2;
  double s = 1.0;
  if (amax > 0.0) {
    int ex;
    frexp(amax, &ex);  // amax in [2^(ex-1), 2^ex)
    s = ldexp(1.0, E - ex);
  }
  g->s = s;
}

template <int FMT>
__device__ __forceinline__ uint16_t rn16(double t) {
  if (FMT == 1) return __half_as_ushort(__double2half(t));
  return __bfloat16_as_ushort(__double2bfloat16(t));
}
template <int FMT>
__device__ __forceinline__ double widen16(uint16_t h) {
  if (FMT == 1) return (double)__half2float(__ushort_as_half(h));
  return (double)__bfloat162float(__ushort_as_bfloat16(h));
}

// Power-of-two constants c_q of the norm pieces (query side of the extra K
// block).  fp16 (11-bit significand): 3 pieces, 2^15, 2^4, 2^-7; bf16 (8-bit):
// 4 pieces, 2^22, 2^14, 2^6, 2^-2.  sum_q c_q p_jq reproduces ||xhat_j||^2
// <= 2^30 to ~2^-33 (fp16) / 2^-32 (bf16) relative; the exact residual is
// measured per row (repmax) and enters the certificate.
template <int FMT>
struct Pieces {
  static constexpr int NP = FMT == 1 ? 3 : 4;
  __device__ static double c(int q) {
    return FMT == 1 ? ldexp(1.0, 15 - 11 * q) : ldexp(1.0, 22 - 8 * q);
  }
};

// W lanes per row (W = 32, or 16 / 8 when dpad/2 <= 16 / 8 element pairs, so
// narrow rows share a warp; rows [0, n_pad)).  side 0 = reference image B:
// [xhat | norm pieces]; side 1 = query image A: [-2 xhat | constants].
// Padding rows are zero (the epilogue masks padding columns).
template <int FMT, int W>
__device__ __forceinline__ void quant_row(const float* __restrict__ X, int64_t n, int d,
                                          const double* __restrict__ mu, PrepGlobals* g,
                                          const Image& img, int side, int64_t r, int lane,
                                          unsigned long long* s_max) {
  const double s = g->s;
  const int epr = img.rb / 2;  // elements per row per main region
  const unsigned M = img.layout == 2 ? 7u : (img.layout == 4 ? 3u : 1u);
  uint8_t* base = reinterpret_cast<uint8_t*>(img.data);
  double a2 = 0.0, r2 = 0.0, tt = 0.0;
  const bool real = r < n;
  for (int p = lane; p < img.dpad / 2; p += W) {
    const int c0 = 2 * p, c1 = 2 * p + 1;
    double t0 = 0.0, t1 = 0.0;
    if (real && c0 < d) t0 = ((double)X[r * d + c0] - mu[c0]) * s;
    if (real && c1 < d) t1 = ((double)X[r * d + c1] - mu[c1]) * s;
    const uint16_t h0 = rn16<FMT>(t0), h1 = rn16<FMT>(t1);
    const double q0 = widen16<FMT>(h0), q1 = widen16<FMT>(h1);
    a2 += q0 * q0 + q1 * q1;
    r2 += (q0 - t0) * (q0 - t0) + (q1 - t1) * (q1 - t1);
    tt += t0 * t0 + t1 * t1;
    uint16_t w0 = h0, w1 = h1;
    if (side == 1) {  // -2 xhat: exact (power-of-two scaling, no overflow by k_scale)
      w0 = rn16<FMT>(-2.0 * q0);
      w1 = rn16<FMT>(-2.0 * q1);
    }
    const int kb = c0 / epr;
    const uint64_t o = (uint64_t)r * img.rb + (uint64_t)(c0 % epr) * 2u;
    const uint64_t phys = o ^ (((o >> 7) & M) << 4);
    *reinterpret_cast<uint32_t*>(base + (size_t)kb * img.region_bytes() + phys) =
        (uint32_t)w0 | ((uint32_t)w1 << 16);
  }
#pragma unroll
  for (int o = W / 2; o > 0; o >>= 1) {  // within the row's W-lane segment
    a2 += __shfl_xor_sync(0xffffffffu, a2, o);
    r2 += __shfl_xor_sync(0xffffffffu, r2, o);
    tt += __shfl_xor_sync(0xffffffffu, tt, o);
  }
  if (lane != 0) return;
  // extra K block (16 elements, 32-byte rows, SW32 swizzle: bit 4 ^= bit 7)
  uint16_t ex[16];
#pragma unroll
  for (int q = 0; q < 16; ++q) ex[q] = 0;
  double rep = 0.0;
  if (side == 1) {
#pragma unroll
    for (int q = 0; q < Pieces<FMT>::NP; ++q) ex[q] = rn16<FMT>(Pieces<FMT>::c(q));
  } else if (real) {
    double rres = a2;
#pragma unroll
    for (int q = 0; q < Pieces<FMT>::NP; ++q) {
      const double cq = Pieces<FMT>::c(q);
      ex[q] = rn16<FMT>(rres / cq);
      rres = rres - cq * widen16<FMT>(ex[q]);  // exact: cq is a power of two
    }
    // |rres| is the representation error w.r.t. the fp64 a2; a2 itself is
    // within (d+2) 2^-53 a2 of the exact ||xhat||^2.
    rep = fabs(rres) * (1.0 + 1e-6) + (double)(d + 4) * 2.220446049250313e-16 * a2;
  }
  {
    const uint64_t o0 = (uint64_t)r * 32u;
    uint8_t* eb = base + img.extra_offset();
    uint4 lo, hi;
    lo.x = ex[0] | ((uint32_t)ex[1] << 16);
    lo.y = ex[2] | ((uint32_t)ex[3] << 16);
    lo.z = ex[4] | ((uint32_t)ex[5] << 16);
    lo.w = ex[6] | ((uint32_t)ex[7] << 16);
    hi.x = ex[8] | ((uint32_t)ex[9] << 16);
    hi.y = ex[10] | ((uint32_t)ex[11] << 16);
    hi.z = ex[12] | ((uint32_t)ex[13] << 16);
    hi.w = ex[14] | ((uint32_t)ex[15] << 16);
    const uint64_t p0 = o0 ^ (((o0 >> 7) & 1u) << 4);
    const uint64_t p1 = (o0 + 16) ^ ((((o0 + 16) >> 7) & 1u) << 4);
    *reinterpret_cast<uint4*>(eb + p0) = lo;
    *reinterpret_cast<uint4*>(eb + p1) = hi;
  }
  if (!real) return;
  img.a2[r] = a2;
  // e >= ||xhat - t|| + ||t - s(x - mu)||: fp64 rounding of the residual sum
  // (relative <= (d+4) 2^-53, doubled) plus the rounding of fl64(x - mu)
  // (<= 2^-53 |x - mu| per element, doubled), then a final margin.
  const double eps = 1.1102230246251565e-16;  // 2^-53
  const double e = (sqrt(r2) * (1.0 + 2.0 * (d + 4) * eps) + 2.0 * eps * sqrt(tt) * (1.0 + 1e-6)) *
                   (1.0 + 8.0 * eps);
  img.e[r] = e;
  if (side == 0) {
    atomic_max_nonneg(&s_max[0], a2);
    atomic_max_nonneg(&s_max[1], e);
    atomic_max_nonneg(&s_max[2], rep);
  }
}


template <int FMT, int W>
__global__ void k_quant(const float* __restrict__ X, int64_t n, int d,
                        const double* __restrict__ mu, PrepGlobals* g, Image img, int side) {
  // per-block maxima (one global atomic per block and quantity, not per row:
  // same-address atomics from every row serialise in L2)
  __shared__ unsigned long long s_max[3];
  if (threadIdx.x < 3) s_max[threadIdx.x] = 0ull;
  __syncthreads();
  const int lane = threadIdx.x & (W - 1);
  const int64_t r = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / W;
  // (n_pad is a multiple of 256 rows, so every warp's segments are all in range
  // or all out of it: the segment shuffles never mix live and exited lanes)
  if (r < img.n_pad) quant_row<FMT, W>(X, n, d, mu, g, img, side, r, lane, s_max);
  __syncthreads();
  if (side == 0 && threadIdx.x < 3 && s_max[threadIdx.x] != 0ull) {
    unsigned long long* dst = threadIdx.x == 0 ? reinterpret_cast<unsigned long long*>(&g->amax2)
                            : threadIdx.x == 1 ? reinterpret_cast<unsigned long long*>(&g->emax)
                                               : reinterpret_cast<unsigned long long*>(&g->repmax);
    atomicMax(dst, s_max[threadIdx.x]);
  }
}

// Diagnostics (tod_debug_mainpass): the 16-bit operand image decoded to fp32,
// out[r][c], c < dpad from the main regions, c in [dpad, dpad + 16) from the
// extra region -- exactly the values the tensor core multiplies.
template <int FMT>
__global__ void k_image_decode(Image img, int64_t rows, float* __restrict__ out) {
  const int K = img.dpad + 16;
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= rows * K) return;
  const int64_t r = i / K;
  const int c = (int)(i - r * K);
  const uint8_t* base = reinterpret_cast<const uint8_t*>(img.data);
  uint64_t phys;
  const uint8_t* reg;
  if (c < img.dpad) {
    const int epr = img.rb / 2;
    const unsigned M = img.layout == 2 ? 7u : (img.layout == 4 ? 3u : 1u);
    const uint64_t o = (uint64_t)r * img.rb + (uint64_t)(c % epr) * 2u;
    phys = o ^ (((o >> 7) & M) << 4);
    reg = base + (size_t)(c / epr) * img.region_bytes();
  } else {
    const uint64_t o = (uint64_t)r * 32u + (uint64_t)(c - img.dpad) * 2u;
    phys = o ^ (((o >> 7) & 1u) << 4);
    reg = base + img.extra_offset();
  }
  const uint16_t h = *reinterpret_cast<const uint16_t*>(reg + phys);
  out[i] = (float)widen16<FMT>(h);
}

}  // namespace

cudaError_t launch_image_decode(const Image& img, int fmt, int64_t rows, float* out, cudaStream_t st,
                                int* launches) {
  const int64_t tot = rows * (img.dpad + 16);
  if (tot <= 0) return cudaSuccess;
  const unsigned blocks = (unsigned)((tot + 255) / 256);
  if (fmt == 1) k_image_decode<1><<<blocks, 256, 0, st>>>(img, rows, out);
  else k_image_decode<2><<<blocks, 256, 0, st>>>(img, rows, out);
  *launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_prep_stats(const float* X, int64_t n, int d, double* mu, double* partial,
                              int partial_blocks, PrepGlobals* g, cudaStream_t st, int* launches) {
  const int blocks = (int)((n + kRowsPerStatBlock - 1) / kRowsPerStatBlock);
  if (blocks > partial_blocks) return cudaErrorInvalidValue;
  k_colsum_partial<<<blocks, kStatThreads, 0, st>>>(X, n, d, partial, g);
  k_colmean<<<d, 256, 0, st>>>(partial, blocks, n, d, mu);
  *launches += 2;
  return cudaGetLastError();
}

// The two halves of launch_prep_stats, for the sharded path: each rank writes
// the partials of its own 128-row blocks (row_offset % 128 == 0, so its local
// block b is global block row_offset/128 + b); the partials of all ranks,
// gathered in global block order, then give the same mean as one process.
cudaError_t launch_prep_colsum(const float* X, int64_t n, int d, double* partial, PrepGlobals* g,
                               cudaStream_t st, int* launches) {
  const int blocks = (int)((n + kRowsPerStatBlock - 1) / kRowsPerStatBlock);
  if (blocks <= 0) return cudaSuccess;
  k_colsum_partial<<<blocks, kStatThreads, 0, st>>>(X, n, d, partial, g);
  *launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_prep_colmean(const double* partial, int blocks, int64_t n, int d, double* mu,
                                cudaStream_t st, int* launches) {
  k_colmean<<<d, 256, 0, st>>>(partial, blocks, n, d, mu);
  *launches += 1;
  return cudaGetLastError();
}

int prep_stat_rows() { return kRowsPerStatBlock; }

cudaError_t launch_finite_check(const float* X, int64_t n, int d, PrepGlobals* g, cudaStream_t st,
                                int* launches) {
  const int64_t total = n * (int64_t)d;
  const int64_t want = (total + 255) / 256;
  const int blocks = (int)(want < 148 * 8 ? want : 148 * 8);
  k_finite<<<max(blocks, 1), 256, 0, st>>>(X, total, g);
  *launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_prep_absmax(const float* X, int64_t n, int d, const double* mu, PrepGlobals* g,
                               cudaStream_t st, int* launches) {
  const int64_t total = n * (int64_t)d;
  const int64_t want = (total + 255) / 256;
  const int blocks = (int)(want < 148 * 8 ? want : 148 * 8);
  k_absmax<<<max(blocks, 1), 256, 0, st>>>(X, n, d, mu, g);
  *launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_prep_scale(PrepGlobals* g, int fmt, int dpad, cudaStream_t st, int* launches) {
  k_scale<<<1, 1, 0, st>>>(g, fmt, dpad);
  *launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_prep_quant(const float* X, int64_t n, int d, const double* mu, PrepGlobals* g,
                              int fmt, Image img, int side, cudaStream_t st, int* launches) {
  const int W = img.dpad / 2 <= 8 ? 8 : (img.dpad / 2 <= 16 ? 16 : 32);  // lanes per row
  const int64_t threads = img.n_pad * W;
  const int blocks = (int)((threads + 255) / 256);
#define TOD_QUANT(F, WW) k_quant<F, WW><<<blocks, 256, 0, st>>>(X, n, d, mu, g, img, side)
  if (fmt == 1) {
    if (W == 8) TOD_QUANT(1, 8); else if (W == 16) TOD_QUANT(1, 16); else TOD_QUANT(1, 32);
  } else {
    if (W == 8) TOD_QUANT(2, 8); else if (W == 16) TOD_QUANT(2, 16); else TOD_QUANT(2, 32);
  }
#undef TOD_QUANT
  *launches += 1;
  return cudaGetLastError();
}

// Per 8-row group of the reference image: e_g = max residual bound of its rows
// (rows >= n count 0).  The re-rank bounds a group's columns with e_g instead of
// the global e_max (DESIGN.md §5 "Re-rank"): the triangle inequality only needs
// e_j <= e_g for the columns j of the group.
__global__ void k_group_emax(const double* __restrict__ e, int64_t n, int64_t ngroups,
                             double* __restrict__ eg) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= ngroups) return;
  double m = 0.0;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int64_t j = g * 8 + u;
    if (j < n) m = fmax(m, e[j]);
  }
  eg[g] = m;
}

cudaError_t launch_group_emax(const double* e, int64_t n, double* eg, cudaStream_t st, int* launches) {
  const int64_t ng = (n + 7) / 8;
  if (ng <= 0) return cudaSuccess;
  k_group_emax<<<(unsigned)((ng + 255) / 256), 256, 0, st>>>(e, n, ng, eg);
  *launches += 1;
  return cudaGetLastError();
}

}  // namespace tod
