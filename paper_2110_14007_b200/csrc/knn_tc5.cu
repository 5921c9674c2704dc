// knn_tc5.cu — K2 main pass (two-pass candidate selection, append-only
// threshold filter) with a THREE-deep ring of accumulators,
// dpad <= 64, single SM.
//
// Same arithmetic as knn_tc3.cu (Eq. (3)'s right-hand side on tcgen05, the
// norm folded into the MMA; fused with topk); different
// schedule, for the bound the per-tile trace of knn_tc3 measured at d <= 32
// (tools/trace_main.py): with two 256-column accumulators one is
// always held by the filter warps while they read it, so only ONE tile's MMAs
// are in flight and the tile period is the MMA latency (issue -> commit seen,
// ~775 cycles for K = 48) plus the accumulator hand-off, ~2.5x the MMA
// throughput cost (384 cycles).  Here the 512 TMEM columns hold three
// NB-column accumulators (NB = 160: 480 columns), so two tiles' MMAs run while
// the filter drains the third.  Reference tiles are NB rows (any multiple of 8
// rows is one contiguous block of each swizzled image region; the image carries
// 256 rows of slack past n_pad for the last tile).
//
// Roles (one CTA per SM, persistent; items = query tile x reference chunk,
// chunk-major so all SMs sweep the same L2-resident chunk):
//   warp 0       producer: bulk async copies of the query tile (resident) and a
//                ring of NB-row reference tiles;
//   warp 1       TMEM allocator + MMA issuer: (dpad+16)/16 MMAs 128 x NB x 16 per
//                tile into accumulator (tile % 3);
//   warps 2..17  filter: warp (q, h) owns TMEM lane quarter q (32 query rows)
//                and column part h (NB/4 columns) of every tile.
#include <math_constants.h>

#include <algorithm>

#include "filter.cuh"
#include "internal.h"
#include "ptx.cuh"

namespace tod {

namespace {

constexpr int kBM = 128;
constexpr int kNacc = 3;
constexpr int kFW = 16;        // filter warps: 4 lane quarters x 4 column parts
constexpr int kExtraRB = 32;
constexpr int kSmemMax = 232448;
constexpr int kMaxStage = 8;

__host__ __device__ constexpr int align_up(int x, int a) { return (x + a - 1) / a * a; }

template <int DPAD, int NB>
struct Cfg5 {
  static_assert(NB % 32 == 0 && NB * kNacc <= 512 && NB <= 256, "accumulator ring must fit TMEM");
  static constexpr int RB = DPAD * 2 < 128 ? DPAD * 2 : 128;
  static constexpr int NKB = DPAD * 2 / RB;
  static constexpr int LAYOUT = RB == 128 ? 2 : (RB == 64 ? 4 : 6);
  static constexpr int SBO = 8 * RB;
  static constexpr int KSTEPS = DPAD / 16;
  static constexpr int A_ONE = kBM * (DPAD + 16) * 2;
  static constexpr int A_STRIDE = align_up(A_ONE, 1024);
  static constexpr int A_EXTRA = kBM * NKB * RB;
  static constexpr int B_BYTES = NB * (DPAD + 16) * 2;
  static constexpr int B_STRIDE = align_up(B_BYTES, 1024);
  static constexpr int B_EXTRA = NB * NKB * RB;
  static constexpr int BH = NB / 4;  // columns per filter warp per tile
};

template <int DPAD, int NB>
__host__ __device__ constexpr int smem5(int nstage, int* off_b, int* off_p, int* off_bar) {
  using C = Cfg5<DPAD, NB>;
  int o = C::A_STRIDE;
  *off_b = o;
  o += nstage * C::B_STRIDE;
  *off_p = o;
  o += kFW * kPendRun * 32 * 8;
  *off_bar = o;
  o += 8 * (2 * kMaxStage + 2 + 2 * kNacc) + 16;
  return o + 1024;
}

template <int DPAD, int NB>
int pick_stages5() {
  int a, b, c;
  for (int ns = kMaxStage; ns >= 2; --ns)
    if (smem5<DPAD, NB>(ns, &a, &b, &c) <= kSmemMax) return ns;
  return 0;
}

// TMEM reads of one filter warp's part: BH consecutive columns.
template <int BH>
__device__ __forceinline__ void tmem_ld_part(uint32_t taddr, float* v) {
  static_assert(BH % 8 == 0 && BH <= 64, "part width");
  int c = 0;
  if constexpr (BH >= 32) {
    tmem_ld32(taddr, *reinterpret_cast<float(*)[32]>(v));
    c = 32;
  }
  if constexpr (BH - (BH >= 32 ? 32 : 0) >= 16) {
    tmem_ld16(taddr + c, v + c);
    c += 16;
  }
  if constexpr ((BH % 16) == 8) tmem_ld8(taddr + c, v + c);
}

template <int DPAD, int FMT, int NB, bool COL, bool TRACE>
__global__ void __launch_bounds__(64 + 32 * kFW, 1)
    k_knn_tc5(const uint8_t* __restrict__ a_img, size_t a_region, size_t a_extra,
              const uint8_t* __restrict__ b_img, size_t b_region, size_t b_extra, int64_t b_tiles,
              int64_t n_ref, int64_t qt0, int64_t n_qtiles, int64_t q_begin, int64_t q_end,
              int self_join, int S, int nstage, const float* __restrict__ tau_v, int tau_lists,
              uint2* __restrict__ mbuf, int* __restrict__ mcnt, int cap, int64_t col0, int vote,
              long long* __restrict__ trace) {
  using C = Cfg5<DPAD, NB>;
  constexpr int BH = C::BH;
  constexpr int H = 4;
  constexpr int kTraceTiles = 2048;  // x 16 stamps
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  int off_b, off_p, off_bar;
  smem5<DPAD, NB>(nstage, &off_b, &off_p, &off_bar);
  uint8_t* sA = smem;
  uint8_t* sB = smem + off_b;
  const uint32_t s_pend = smem_u32(smem + off_p);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + off_bar);
  uint64_t* full = bars;
  uint64_t* empty = bars + kMaxStage;
  uint64_t* a_full = bars + 2 * kMaxStage;
  uint64_t* a_empty = a_full + 1;
  uint64_t* t_full = a_empty + 1;      // [kNacc]
  uint64_t* t_empty = t_full + kNacc;  // [kNacc]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(t_empty + kNacc);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const bool tron = TRACE && trace != nullptr && blockIdx.x == 0;

  if (threadIdx.x == 0) {
    for (int i = 0; i < nstage; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(a_full, 1);
    mbar_init(a_empty, 1);
    for (int i = 0; i < kNacc; ++i) {
      mbar_init(&t_full[i], 1);
      mbar_init(&t_empty[i], kFW);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int64_t n_items = n_qtiles * S;

  if (warp == 0) {
    // -------------------------------------------------------------- producer
    int stage = 0;
    uint32_t phase = 0, aphase = 0;
    int ptr = 0;
    for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int64_t qtl = item % n_qtiles;
      const int c = (int)(item / n_qtiles);
      const int t0 = (int)(b_tiles * c / S), t1 = (int)(b_tiles * (c + 1) / S);
      int issued = 0;
      bool a_done = false;
      auto load_a = [&]() {
        mbar_wait_backoff(a_empty, aphase ^ 1);
        aphase ^= 1;
        if (elect_one()) {
          mbar_arrive_expect_tx(a_full, C::A_ONE);
          for (int kb = 0; kb < C::NKB; ++kb)
            bulk_g2s(sA + kb * kBM * C::RB, a_img + kb * a_region + qtl * (int64_t)kBM * C::RB,
                     kBM * C::RB, a_full);
          bulk_g2s(sA + C::A_EXTRA, a_img + a_extra + qtl * (int64_t)kBM * kExtraRB,
                   kBM * kExtraRB, a_full);
        }
        __syncwarp();
        a_done = true;
      };
      for (int t = t0; t < t1; ++t) {
        // the item's first B tiles are fetched while the MMA drains the previous item
        if (!a_done && issued == nstage - 1) load_a();
        mbar_wait_backoff(&empty[stage], phase ^ 1);
        if constexpr (TRACE)
          if (tron && lane == 0 && ptr < kTraceTiles) trace[ptr * 16 + 7] = clock64();
        ++ptr;
        if (elect_one()) {
          mbar_arrive_expect_tx(&full[stage], C::B_BYTES);
          uint8_t* dst = sB + stage * C::B_STRIDE;
          const int64_t row0 = (int64_t)t * NB;
          for (int kb = 0; kb < C::NKB; ++kb)
            bulk_g2s(dst + kb * NB * C::RB, b_img + kb * b_region + row0 * C::RB, NB * C::RB,
                     &full[stage]);
          bulk_g2s(dst + C::B_EXTRA, b_img + b_extra + row0 * kExtraRB, NB * kExtraRB,
                   &full[stage]);
        }
        __syncwarp();
        ++issued;
        if (++stage == nstage) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (!a_done) load_a();
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    constexpr uint32_t IDESC = idesc_f16(kBM, NB, FMT == 1 ? 0u : 1u);
    constexpr int NK = C::KSTEPS + 1;
    const uint32_t a_base = smem_u32(sA);
    const uint32_t b_base = smem_u32(sB);
    uint64_t adesc[NK], bdesc[NK];
#pragma unroll
    for (int ks = 0; ks < C::KSTEPS; ++ks) {
      const int kb = (ks * 32) / C::RB;
      const int koff = (ks * 32) % C::RB;
      adesc[ks] = smem_desc(a_base + kb * kBM * C::RB + koff, C::SBO, C::LAYOUT);
      bdesc[ks] = smem_desc(b_base + kb * NB * C::RB + koff, C::SBO, C::LAYOUT);
    }
    adesc[C::KSTEPS] = smem_desc(a_base + C::A_EXTRA, 8 * kExtraRB, 6);
    bdesc[C::KSTEPS] = smem_desc(b_base + C::B_EXTRA, 8 * kExtraRB, 6);
    const uint32_t s_full = smem_u32(full), s_tempty = smem_u32(t_empty);
    int stage = 0, acc = 0;
    uint32_t phase = 0, acc_phase = 0, aphase = 0;
    int mtr = 0;
    for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int c = (int)(item / n_qtiles);
      const int t0 = (int)(b_tiles * c / S), t1 = (int)(b_tiles * (c + 1) / S);
      mbar_wait(a_full, aphase);
      aphase ^= 1;
      tc_fence_after();
      for (int t = t0; t < t1; ++t) {
        const bool tr = TRACE && tron && lane == 0 && mtr < kTraceTiles;
        if (tr) trace[mtr * 16 + 0] = clock64();
        mbar_wait_u32(s_full + stage * 8, phase);
        if (tr) trace[mtr * 16 + 1] = clock64();
        mbar_wait_u32(s_tempty + acc * 8, acc_phase ^ 1);
        if (tr) trace[mtr * 16 + 2] = clock64();
        ++mtr;
        tc_fence_after();
        const uint64_t bst = (uint64_t)((stage * C::B_STRIDE) >> 4);
        if (elect_one()) {
#pragma unroll
          for (int ks = 0; ks < NK; ++ks)
            tc_mma_f16(tmem_base + acc * NB, adesc[ks], bdesc[ks] + bst, IDESC, ks > 0 ? 1u : 0u);
          tc_commit(&t_full[acc]);
          tc_commit(&empty[stage]);
        }
        __syncwarp();
        if (tr) trace[(mtr - 1) * 16 + 8] = clock64();
        if (++stage == nstage) {
          stage = 0;
          phase ^= 1;
        }
        if (++acc == kNacc) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
      if (elect_one()) tc_commit(a_empty);
      __syncwarp();
    }
  } else {
    // --------------------------------------------------------- filter warps
    const int f = warp - 2;
    const int q = warp & 3;           // TMEM lane quarter (warp id % 4 = its sub-partition)
    const int h = f >> 2;             // column part of every tile
    const int rt = q * 32 + lane;     // row within the query tile
    const uint32_t pbase = s_pend + (f * kPendRun * 32 + lane) * 8;
    uint32_t pa = pbase;
    const uint32_t taddr0 = tmem_base + ((uint32_t)(q * 32) << 16) + h * BH;
    const uint32_t s_tfull = smem_u32(t_full), s_tempty = smem_u32(t_empty);
    int acc = 0;
    uint32_t acc_phase = 0;
    int etr = 0;
    for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int64_t qtl = item % n_qtiles;
      const int c = (int)(item / n_qtiles);
      const int t0 = (int)(b_tiles * c / S), t1 = (int)(b_tiles * (c + 1) / S);
      const int64_t row = (qt0 + qtl) * kBM + rt;
      const bool valid = row >= q_begin && row < q_end;
      const int64_t r = valid ? row - q_begin : 0;
      // the self column (block-relative) and padding columns are never candidates
      const int64_t selfc = self_join ? row - col0 : -1;
      float tau = -CUDART_INF_F;  // rows outside the range append nothing
      if (valid) {
        tau = CUDART_INF_F;
        for (int l = 0; l < tau_lists; ++l) tau = fminf(tau, tau_v[r * tau_lists + l]);
      }
      int* cnt = mcnt + r * H + h;
      uint2* buf = mbuf + (r * H + h) * (int64_t)cap;
      auto flush = [&]() {
        const int n = (int)((pa - pbase) / kPendSlot);
        if (n > 0) {
          const int base = atomicAdd(cnt, n);
          for (int e = 0; e < n; ++e) {
            const float2 kv = lds_kv(pbase + e * kPendSlot);
            if (base + e < cap)
              buf[base + e] = make_uint2(__float_as_uint(kv.x), (unsigned)__float_as_int(kv.y));
          }
        }
        pa = pbase;
      };
      for (int t = t0; t < t1; ++t) {
        const bool tr = TRACE && tron && warp == 2 && lane == 0 && etr < kTraceTiles;
        if (tr) trace[etr * 16 + 3] = clock64();
        mbar_wait_u32(s_tfull + acc * 8, acc_phase);
        if (tr) trace[etr * 16 + 4] = clock64();
        tc_fence_after();
        float v[BH];
        tmem_ld_part<BH>(taddr0 + acc * NB, v);
        tmem_ld_wait();
        if (tr) trace[etr * 16 + 9] = clock64();
        const uint32_t acc_now = acc;
        auto release = [=]() {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_u32(s_tempty + acc_now * 8);
        };
        if (!COL) release();  // column candidates: filter_part releases after its vote
        if (tr) trace[etr * 16 + 5] = clock64();
        if constexpr (TRACE)
          if (tron && warp == 1 + kFW && lane == 0 && etr < kTraceTiles) trace[etr * 16 + 10] = clock64();
        ++etr;
        if (++acc == kNacc) {
          acc = 0;
          acc_phase ^= 1;
        }
        const int64_t j0 = (int64_t)t * NB + h * BH;  // block-relative first column of the part
        const bool need_mask = (uint64_t)(selfc - j0) < (uint64_t)BH || j0 + BH > n_ref;
        if (need_mask) {
#pragma unroll
          for (int e = 0; e < BH; ++e)
            v[e] = (j0 + e == selfc || j0 + e >= n_ref) ? CUDART_INF_F : v[e];
        }
        const uint32_t taddr = taddr0 + acc_now * NB;
        auto reload = [=](int gg, float* c8) {
          tmem_ld8(taddr + 8 * gg, c8);
          tmem_ld_wait();
          if (need_mask) {
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const int64_t jj = j0 + 8 * gg + e;
              if (jj == selfc || jj >= n_ref) c8[e] = CUDART_INF_F;
            }
          }
        };
        filter_part<BH, COL>(v, tau, (int)((col0 + j0) >> 3), pa, pbase, vote != 0, flush, reload,
                             release);
        if (tr) trace[(etr - 1) * 16 + 6] = clock64();
      }
      flush();
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

template <int DPAD, int FMT, int NB, bool COL, bool TRACE = false>
cudaError_t launch5(const Image& A, const Image& B, int64_t q_begin, int64_t q_count,
                    bool self_join, const MainPass& m, int num_sms, cudaStream_t st) {
  const int nstage = pick_stages5<DPAD, NB>();
  if (nstage < 3) return cudaErrorInvalidValue;
  if (m.parts != 4 || m.R != 0) return cudaErrorInvalidValue;
  int a, b, c;
  const int smem = smem5<DPAD, NB>(nstage, &a, &b, &c);
  auto kern = k_knn_tc5<DPAD, FMT, NB, COL, TRACE>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const int64_t qt0 = q_begin / kBM;
  const int64_t qt1 = (q_begin + q_count + kBM - 1) / kBM;
  const int64_t b_tiles = (B.n + NB - 1) / NB;
  const int S = (int)std::min<int64_t>(std::max(m.S, 1), b_tiles);
  const int64_t n_items = (qt1 - qt0) * S;
  const int grid = (int)std::min<int64_t>(num_sms, n_items);
  if (grid <= 0) return cudaSuccess;
  kern<<<grid, 64 + 32 * kFW, smem, st>>>(
      reinterpret_cast<const uint8_t*>(A.data), A.region_bytes(), A.extra_offset(),
      reinterpret_cast<const uint8_t*>(B.data), B.region_bytes(), B.extra_offset(), b_tiles, B.n,
      qt0, qt1 - qt0, q_begin, q_begin + q_count, self_join ? 1 : 0, S, nstage, m.tau_v,
      m.tau_lists, m.buf, m.cnt, m.cap, m.col0, m.vote, m.trace);
  return cudaGetLastError();
}

constexpr int kNB = 160;

}  // namespace

int tc5_fits(int dpad) {
  switch (dpad) {
    case 16: return pick_stages5<16, kNB>() >= 3;
    case 32: return pick_stages5<32, kNB>() >= 3;
    case 64: return pick_stages5<64, kNB>() >= 3;
  }
  return 0;
}

cudaError_t launch_knn_tc5(const Image& A, const Image& B, int64_t q_begin, int64_t q_count,
                           bool self_join, int fmt, const MainPass& m, int num_sms, cudaStream_t st,
                           int* launches) {
  *launches += 1;
#define TOD_TC5_CASE(D)                                                                          \
  case D:                                                                                       \
    if (m.trace)  /* profiling trace build */                                                   \
      return fmt == 1 ? launch5<D, 1, kNB, false, true>(A, B, q_begin, q_count, self_join, m, num_sms, st) \
                      : launch5<D, 2, kNB, false, true>(A, B, q_begin, q_count, self_join, m, num_sms, st); \
    if (m.colmode)                                                                              \
      return fmt == 1 ? launch5<D, 1, kNB, true>(A, B, q_begin, q_count, self_join, m, num_sms, st) \
                      : launch5<D, 2, kNB, true>(A, B, q_begin, q_count, self_join, m, num_sms, st); \
    return fmt == 1 ? launch5<D, 1, kNB, false>(A, B, q_begin, q_count, self_join, m, num_sms, st)   \
                    : launch5<D, 2, kNB, false>(A, B, q_begin, q_count, self_join, m, num_sms, st);
  switch (A.dpad) {
    TOD_TC5_CASE(16)
    TOD_TC5_CASE(32)
    TOD_TC5_CASE(64)
  }
#undef TOD_TC5_CASE
  return cudaErrorInvalidValue;
}

}  // namespace tod
