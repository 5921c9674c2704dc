// knn_tc.cu — K2: the hot loop.  Fused tile distance + running per-row top-K'
// on 5th-generation tensor cores (tcgen05, sm_100a).
//
// What it computes: for every query row i of a 128-row
// query tile and every reference column j of the chunk's 256-column tiles,
//     G_ij  = xhat_i . xhat_j                (tcgen05.mma kind::f16, fp32 in TMEM)
//     w_ij  = fl32(n_j - 2 G_ij)             (one FFMA; n_j = fp32 ||xhat_j||^2)
// which is Eq. (3)'s right-hand side ||X_i||^2 + ||X_j||^2 - 2 X_i^T X_j
// (§5.3) minus the row-constant ||X_i||^2 (ranking within
// a row does not need it), and keeps the K' smallest w per row (operator
// fusion of cdist and topk: the n x n matrix is never stored).
// Self is excluded by index (reading A3).
//
// Structure (one CTA per SM, persistent over (query tile, chunk) work items):
//   warp 0     producer: bulk async copies (TMA engine) of the resident query
//              tile A, the reference tiles B (ring of NSTAGE stages) and their
//              norms (ring of 4), completion on mbarriers (complete_tx).
//   warp 1     TMEM allocator + single-thread MMA issuer: DPAD/16 MMAs of
//              128 x BN x 16 per reference tile into one of two TMEM
//              accumulators (double buffered: MMA of tile t+1 overlaps the
//              epilogue of tile t); tcgen05.commit frees smem stages and
//              publishes accumulators.
//   warps 2-5  epilogue: thread = query row (TMEM lane), tcgen05.ld 32 columns
//              at a time, FFMA + running min per 8 columns, warp vote against
//              the per-row threshold; rare hits go to the RowTopK list.
// Operands arrive pre-quantized and pre-swizzled (prep.cu writes the exact
// K-major SWIZZLE_{32,64,128}B smem image), so a plain contiguous bulk copy
// replaces tensor-map TMA.
#include <cuda_fp16.h>
#include <math_constants.h>

#include <algorithm>

#include "internal.h"
#include "ptx.cuh"
#include "topk_list.cuh"

namespace tod {

namespace {

constexpr int kBM = 128;
constexpr int kThreads = 192;
constexpr int kNormSlots = 4;

template <int DPAD>
struct TcCfg {
  static constexpr int RB = DPAD * 2 < 128 ? DPAD * 2 : 128;  // bytes per row per K region
  static constexpr int NKB = DPAD * 2 / RB;                  // K regions
  static constexpr int LAYOUT = RB == 128 ? 2 : (RB == 64 ? 4 : 6);
  static constexpr int SBO = 8 * RB;
  static constexpr int BN = DPAD <= 64 ? 256 : 128;
  static constexpr int KSTEPS = DPAD / 16;
  static constexpr int NSTAGE = DPAD <= 32 ? 4 : (DPAD == 64 ? 3 : 3);
  static constexpr int A_BYTES = kBM * DPAD * 2;
  static constexpr int B_BYTES = BN * DPAD * 2;
  static constexpr int TMEM_COLS = 2 * BN;  // two accumulators
};

__host__ __device__ constexpr int align_up(int x, int a) { return (x + a - 1) / a * a; }

template <int DPAD>
__host__ __device__ constexpr int smem_layout_bytes(int kp, int* off_b, int* off_n, int* off_lv,
                                                    int* off_li, int* off_bar) {
  using C = TcCfg<DPAD>;
  int o = 0;
  o += C::A_BYTES;
  o = align_up(o, 1024);
  *off_b = o;
  o += C::NSTAGE * C::B_BYTES;
  *off_n = o;
  o += kNormSlots * C::BN * 4;
  *off_lv = o;
  o += (kp + kPend) * kBM * 4;
  *off_li = o;
  o += (kp + kPend) * kBM * 4;
  o = align_up(o, 8);
  *off_bar = o;
  o += 8 * (2 * C::NSTAGE + 2 + 2 * kNormSlots + 4) + 16;
  return o + 1024;  // slack for aligning the dynamic smem base to 1024
}

template <int DPAD, int FMT>
__global__ void __launch_bounds__(kThreads, 1)
    k_knn_tc(const uint8_t* __restrict__ a_img, size_t a_region, const uint8_t* __restrict__ b_img,
             size_t b_region, const float* __restrict__ b_nrm, int64_t b_tiles, int64_t qt0,
             int64_t n_qtiles, int64_t q_begin, int64_t q_end, int self_join, int S, int kp,
             int32_t* __restrict__ cand_idx, float* __restrict__ cand_v) {
  using C = TcCfg<DPAD>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  int off_b, off_n, off_lv, off_li, off_bar;
  smem_layout_bytes<DPAD>(kp, &off_b, &off_n, &off_lv, &off_li, &off_bar);
  uint8_t* sA = smem;
  uint8_t* sB = smem + off_b;
  float* sN = reinterpret_cast<float*>(smem + off_n);
  float* sLv = reinterpret_cast<float*>(smem + off_lv);
  int* sLi = reinterpret_cast<int*>(smem + off_li);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + off_bar);
  uint64_t* full = bars;                        // [NSTAGE]
  uint64_t* empty = bars + C::NSTAGE;           // [NSTAGE]
  uint64_t* a_full = bars + 2 * C::NSTAGE;      // [1]
  uint64_t* a_empty = a_full + 1;               // [1]
  uint64_t* n_full = a_empty + 1;               // [kNormSlots]
  uint64_t* n_empty = n_full + kNormSlots;      // [kNormSlots]
  uint64_t* t_full = n_empty + kNormSlots;      // [2]
  uint64_t* t_empty = t_full + 2;               // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(t_empty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < C::NSTAGE; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(a_full, 1);
    mbar_init(a_empty, 1);
    for (int i = 0; i < kNormSlots; ++i) {
      mbar_init(&n_full[i], 1);
      mbar_init(&n_empty[i], 4);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&t_full[i], 1);
      mbar_init(&t_empty[i], 4);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int64_t n_items = n_qtiles * S;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------------------ producer
      int stage = 0;
      uint32_t phase = 0;
      int ns = 0;
      uint32_t nphase = 0;
      uint32_t aphase = 0;
      for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
        const int64_t qt = qt0 + item / S;
        const int c = (int)(item % S);
        const int64_t t_lo = b_tiles * c / S, t_hi = b_tiles * (c + 1) / S;
        mbar_wait(a_empty, aphase ^ 1);
        aphase ^= 1;
        mbar_arrive_expect_tx(a_full, C::A_BYTES);
        for (int kb = 0; kb < C::NKB; ++kb)
          bulk_g2s(sA + kb * kBM * C::RB, a_img + kb * a_region + qt * (int64_t)kBM * C::RB,
                   kBM * C::RB, a_full);
        for (int64_t t = t_lo; t < t_hi; ++t) {
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_arrive_expect_tx(&full[stage], C::B_BYTES);
          uint8_t* dst = sB + stage * C::B_BYTES;
          for (int kb = 0; kb < C::NKB; ++kb)
            bulk_g2s(dst + kb * C::BN * C::RB, b_img + kb * b_region + t * (int64_t)C::BN * C::RB,
                     C::BN * C::RB, &full[stage]);
          if (++stage == C::NSTAGE) {
            stage = 0;
            phase ^= 1;
          }
          mbar_wait(&n_empty[ns], nphase ^ 1);
          mbar_arrive_expect_tx(&n_full[ns], C::BN * 4);
          bulk_g2s(sN + ns * C::BN, b_nrm + t * C::BN, C::BN * 4, &n_full[ns]);
          if (++ns == kNormSlots) {
            ns = 0;
            nphase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------------------------------------------------- MMA issuer
      constexpr uint32_t IDESC = idesc_f16(kBM, C::BN, FMT == 1 ? 0u : 1u);
      const uint32_t a_base = smem_u32(sA);
      const uint32_t b_base = smem_u32(sB);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t aphase_acc = 0;
      uint32_t aphase = 0;
      for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
        const int c = (int)(item % S);
        const int64_t t_lo = b_tiles * c / S, t_hi = b_tiles * (c + 1) / S;
        mbar_wait(a_full, aphase);
        aphase ^= 1;
        tc_fence_after();
        for (int64_t t = t_lo; t < t_hi; ++t) {
          mbar_wait(&t_empty[acc], aphase_acc ^ 1);
          tc_fence_after();
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + acc * C::BN;
          const uint32_t bst = b_base + stage * C::B_BYTES;
#pragma unroll
          for (int ks = 0; ks < C::KSTEPS; ++ks) {
            const int kb = (ks * 32) / C::RB;
            const int koff = (ks * 32) % C::RB;
            const uint64_t ad = smem_desc(a_base + kb * kBM * C::RB + koff, C::SBO, C::LAYOUT);
            const uint64_t bd = smem_desc(bst + kb * C::BN * C::RB + koff, C::SBO, C::LAYOUT);
            tc_mma_f16(d_tmem, ad, bd, IDESC, ks > 0 ? 1u : 0u);
          }
          tc_commit(&empty[stage]);
          tc_commit(&t_full[acc]);
          if (++stage == C::NSTAGE) {
            stage = 0;
            phase ^= 1;
          }
          if (++acc == 2) {
            acc = 0;
            aphase_acc ^= 1;
          }
        }
        tc_commit(a_empty);
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue
    const int q = warp & 3;           // TMEM lane quarter this warp may access
    const int t = q * 32 + lane;      // row within the query tile
    RowTopK<kBM> L;
    L.init(sLv, sLi, t, kp);
    int acc = 0;
    uint32_t aphase_acc = 0;
    int ns = 0;
    uint32_t nphase = 0;
    for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int64_t qt = qt0 + item / S;
      const int c = (int)(item % S);
      const int64_t t_lo = b_tiles * c / S, t_hi = b_tiles * (c + 1) / S;
      const int64_t row = qt * kBM + t;
      const int self = self_join ? (int)row : -1;
      for (int64_t tt = t_lo; tt < t_hi; ++tt) {
        mbar_wait(&t_full[acc], aphase_acc);
        tc_fence_after();
        mbar_wait(&n_full[ns], nphase);
        const float* nrm = sN + ns * C::BN;
        const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + acc * C::BN;
        const int j0 = (int)(tt * C::BN);
#pragma unroll 1
        for (int ch = 0; ch < C::BN / 32; ++ch) {
          float v[32];
          tmem_ld32(taddr + ch * 32, v);
          tmem_ld_wait();
          const float4* n4 = reinterpret_cast<const float4*>(nrm + ch * 32);
#pragma unroll
          for (int g = 0; g < 4; ++g) {
            const float4 na = n4[2 * g], nb = n4[2 * g + 1];
            float w[8];
            w[0] = fmaf(-2.f, v[8 * g + 0], na.x);
            w[1] = fmaf(-2.f, v[8 * g + 1], na.y);
            w[2] = fmaf(-2.f, v[8 * g + 2], na.z);
            w[3] = fmaf(-2.f, v[8 * g + 3], na.w);
            w[4] = fmaf(-2.f, v[8 * g + 4], nb.x);
            w[5] = fmaf(-2.f, v[8 * g + 5], nb.y);
            w[6] = fmaf(-2.f, v[8 * g + 6], nb.z);
            w[7] = fmaf(-2.f, v[8 * g + 7], nb.w);
            const float m = fminf(fminf(fminf(w[0], w[1]), fminf(w[2], w[3])),
                                  fminf(fminf(w[4], w[5]), fminf(w[6], w[7])));
            if (__any_sync(0xffffffffu, m < L.thr)) {
              const int jb = j0 + ch * 32 + 8 * g;
#pragma unroll
              for (int e = 0; e < 8; ++e) L.offer(w[e], jb + e, self);
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&t_empty[acc]);
          mbar_arrive(&n_empty[ns]);
        }
        if (++acc == 2) {
          acc = 0;
          aphase_acc ^= 1;
        }
        if (++ns == kNormSlots) {
          ns = 0;
          nphase ^= 1;
        }
      }
      const bool write = row >= q_begin && row < q_end;
      const int64_t r = row - q_begin;
      const float v = L.finish(cand_idx + (write ? (r * S + c) * kp : 0), write);
      if (write) cand_v[r * S + c] = v;
      L.reset();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, C::TMEM_COLS);
  }
}

template <int DPAD, int FMT>
cudaError_t launch_t(const Image& A, const Image& B, int64_t q_begin, int64_t q_count,
                     bool self_join, Cands c, int num_sms, cudaStream_t st) {
  using C = TcCfg<DPAD>;
  int ob, on, olv, oli, obar;
  const int smem = smem_layout_bytes<DPAD>(c.kp, &ob, &on, &olv, &oli, &obar);
  auto kern = k_knn_tc<DPAD, FMT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const int64_t qt0 = q_begin / kBM;
  const int64_t qt1 = (q_begin + q_count + kBM - 1) / kBM;
  const int64_t n_items = (qt1 - qt0) * c.S;
  const int grid = (int)std::min<int64_t>(num_sms, n_items);
  if (grid <= 0) return cudaSuccess;
  kern<<<grid, kThreads, smem, st>>>(
      reinterpret_cast<const uint8_t*>(A.data), A.region_bytes(),
      reinterpret_cast<const uint8_t*>(B.data), B.region_bytes(), B.nrm32, B.n_pad / C::BN, qt0,
      qt1 - qt0, q_begin, q_begin + q_count, self_join ? 1 : 0, c.S, c.kp, c.idx, c.v);
  return cudaGetLastError();
}

}  // namespace

int tc_smem_bytes(int dpad, int kp) {
  int a, b, c, d, e;
  switch (dpad) {
    case 16: return smem_layout_bytes<16>(kp, &a, &b, &c, &d, &e);
    case 32: return smem_layout_bytes<32>(kp, &a, &b, &c, &d, &e);
    case 64: return smem_layout_bytes<64>(kp, &a, &b, &c, &d, &e);
    case 128: return smem_layout_bytes<128>(kp, &a, &b, &c, &d, &e);
  }
  return -1;
}

int tc_block_n(int dpad) { return dpad <= 64 ? 256 : 128; }

cudaError_t launch_knn_tc(const Image& A, const Image& B, int64_t q_begin, int64_t q_count,
                          bool self_join, int fmt, Cands c, int num_sms, cudaStream_t st,
                          int* launches) {
  *launches += 1;
#define TOD_TC_CASE(D)                                                                      \
  case D:                                                                                  \
    return fmt == 1 ? launch_t<D, 1>(A, B, q_begin, q_count, self_join, c, num_sms, st)    \
                    : launch_t<D, 2>(A, B, q_begin, q_count, self_join, c, num_sms, st);
  switch (A.dpad) {
    TOD_TC_CASE(16)
    TOD_TC_CASE(32)
    TOD_TC_CASE(64)
    TOD_TC_CASE(128)
  }
#undef TOD_TC_CASE
  return cudaErrorInvalidValue;
}

}  // namespace tod
