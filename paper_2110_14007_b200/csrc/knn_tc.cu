// knn_tc.cu — K2: the hot loop.  Fused tile distance + running per-row top-K'
// on 5th-generation tensor cores (tcgen05, sm_100a).
//
// What it computes: for every query row i and every
// reference column j,
//     w_ij = ||xhat_j||^2 - 2 xhat_i . xhat_j          (one fp32 TMEM value)
// i.e. Eq. (3)'s right-hand side ||X_i||^2 + ||X_j||^2 - 2 X_i^T X_j (PAPER.md
// §5.3) minus the row constant ||X_i||^2, which a row's ranking does
// not need.  The whole of w comes out of the tensor core: the operand images
// carry an extra 16-wide K block in which the query side holds power-of-two
// constants c_q and the reference side the 16-bit pieces p_jq of ||xhat_j||^2
// (sum_q c_q p_jq = ||xhat_j||^2 to ~2^-33), and the query side stores
// -2 xhat_i.  The epilogue is then a pure min-tree + vote per 8 columns; it
// keeps the K' smallest w per row (operator fusion of cdist and topk,
// the n x n matrix is never stored).  Self is excluded by index
// (reading A3); padding columns are masked.
//
// Work decomposition ("automatic batching" re-derived): items are
// (query group of QT 128-row tiles) x (reference chunk c of S), in chunk-major
// order so that all CTAs sweep the same L2-resident chunk of the reference
// image at the same time; a row's top-K' state is parked in HBM between its
// chunks (st_list / st_done), so chunking adds no candidates and no re-rank
// work.  The query image A holds only the rows of query tiles [qt0, qt1).
//
// Structure (one CTA per SM, persistent):
//   warp 0     producer: bulk async copies (TMA engine, UBLKCP) of the QT
//              resident query tiles and the reference tiles B (ring of
//              nstage stages), completion on mbarriers (complete_tx).
//   warp 1     TMEM allocator + single-thread MMA issuer: per reference tile,
//              for each of the QT query tiles, (DPAD+16)/16 MMAs 128 x BN x 16
//              into one of two TMEM accumulators (double buffered: the MMA of
//              tile t+1 overlaps the epilogue of tile t).  With QT = 2 each B
//              tile feeds 256 query rows, halving L2->SM traffic per pair.
//   warps 2+   epilogue, 4 per query tile: thread = query row (TMEM lane),
//              tcgen05.ld 32 columns at a time (double-buffered), 3-input min
//              trees, one warp OR-reduction per tile; rare hits -> RowTopK.
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
constexpr int kExtraRB = 32;     // bytes per row of the 16-wide extra K block
constexpr int kSmemMax = 232448; // 227 KB opt-in per block
constexpr int kTraceTiles = 4096;
#ifndef TOD_SMALL_BN
#define TOD_SMALL_BN 256
#endif // TOD_F_DEBUG_TRACE: per-tile timestamps of CTA 0

__host__ __device__ constexpr int align_up(int x, int a) { return (x + a - 1) / a * a; }

// SPLIT = epilogue warps per TMEM lane quarter.  With SPLIT = 2 each tile's
// columns are split in two halves, each with its own warp (2 warps per SM
// sub-partition for latency hiding) and its own per-row top-K'' list; the
// re-rank takes the union of the two lists (v = min of the two thresholds).
template <int DPAD, int SPLIT>
struct TcCfg {
  static constexpr int QT = 1;
  static constexpr int RB = DPAD * 2 < 128 ? DPAD * 2 : 128;  // bytes per row per main K region
  static constexpr int NKB = DPAD * 2 / RB;                  // main K regions
  static constexpr int LAYOUT = RB == 128 ? 2 : (RB == 64 ? 4 : 6);
  static constexpr int SBO = 8 * RB;
  // d <= 32: short MMAs, so use 4 accumulators of 128 columns (deeper MMA/epilogue
  // pipeline); d = 64: 2 accumulators of 256 (fewer, longer MMAs; half the smem reads).
  static constexpr int BN = DPAD == 64 ? 256 : (DPAD == 128 ? 128 : TOD_SMALL_BN);
  static constexpr int BH = BN / SPLIT;                      // columns per epilogue warp
  static constexpr int KSTEPS = DPAD / 16;                   // main K steps (+1 extra)
  static constexpr int MAX_STAGE = 4;
  static constexpr int NROWS = kBM;                          // query rows per CTA item
  static constexpr int NLIST = kBM * SPLIT;                  // lists per CTA item
  static constexpr int PEND = SPLIT == 4 ? 16 : (DPAD <= 32 ? 32 : 24);  // pending slots per list
  static constexpr int EPI_WARPS = 4 * SPLIT;
  static constexpr int THREADS = 64 + 32 * EPI_WARPS;
  static constexpr int A_ONE = kBM * (DPAD + 16) * 2;        // one query tile
  static constexpr int A_STRIDE = align_up(A_ONE, 1024);
  static constexpr int A_EXTRA = kBM * NKB * RB;             // offset of a tile's extra block
  static constexpr int B_BYTES = BN * (DPAD + 16) * 2;
  static constexpr int B_STRIDE = align_up(B_BYTES, 1024);
  static constexpr int B_EXTRA = BN * NKB * RB;
  static constexpr int NACC = 512 / BN;                      // accumulators in TMEM
  static constexpr int TMEM_COLS = NACC * BN;
  static_assert(TMEM_COLS <= 512, "TMEM overflow");
};

template <int DPAD, int SPLIT>
__host__ __device__ constexpr int smem_layout_bytes(int kp, int nstage, int* off_b, int* off_l,
                                                    int* off_bar) {
  using C = TcCfg<DPAD, SPLIT>;
  int o = C::A_STRIDE;
  *off_b = o;
  o += nstage * C::B_STRIDE;
  *off_l = o;
  o += (kp + C::PEND) * C::NLIST * 8;
  o = align_up(o, 8);
  *off_bar = o;
  o += 8 * (2 * C::MAX_STAGE + 2 + 2 * C::NACC) + 16;
  return o + 1024;  // slack for aligning the dynamic smem base to 1024
}

// Deepest B pipeline (<= 4 stages) that fits; 0 if even 2 stages do not fit.
template <int DPAD, int SPLIT>
int pick_stages(int kp) {
  int a, b, c;
  for (int ns = TcCfg<DPAD, SPLIT>::MAX_STAGE; ns >= 2; --ns)
    if (smem_layout_bytes<DPAD, SPLIT>(kp, ns, &a, &b, &c) <= kSmemMax) return ns;
  return 0;
}

// 4-bit mask of the 8-column groups of a 32-column chunk whose minimum < thr.
__device__ __forceinline__ unsigned group_bits(const float (&v)[32], float thr) {
  unsigned gm = 0;
#pragma unroll
  for (int g = 0; g < 4; ++g) {
    const float* vg = v + 8 * g;
    const float m = fminf(fminf(fminf(vg[0], vg[1]), vg[2]),
                          fminf(fminf(vg[3], vg[4]), fminf(fminf(vg[5], vg[6]), vg[7])));
    gm |= (m < thr) ? (1u << g) : 0u;
  }
  return gm;
}

// Self column and padding columns (>= n_ref) become +inf: never kept.
__device__ __noinline__ void mask_cols(float (&v)[32], int jb, int self, int64_t n_ref) {
#pragma unroll
  for (int e = 0; e < 32; ++e) v[e] = (jb + e == self || jb + e >= n_ref) ? CUDART_INF_F : v[e];
}

template <int DPAD, int FMT, int SPLIT>
__global__ void __launch_bounds__(TcCfg<DPAD, SPLIT>::THREADS, 1)
    k_knn_tc(const uint8_t* __restrict__ a_img, size_t a_region, size_t a_extra,
             const uint8_t* __restrict__ b_img, size_t b_region, size_t b_extra, int64_t b_tiles,
             int64_t n_ref, int64_t qt0, int64_t n_qtiles, int64_t q_begin, int64_t q_end,
             int self_join, int S, int R, int kp, int nstage, int dbg, int32_t* __restrict__ cand_idx,
             float* __restrict__ cand_v, float* __restrict__ cand_key, uint2* __restrict__ st_list,
             int* __restrict__ st_done, long long* __restrict__ trace) {
  using C = TcCfg<DPAD, SPLIT>;
  constexpr int QT = C::QT;
  using List = RowTopK<C::NLIST, C::PEND>;
  // Reserve pending room once per tile when a tile's worst case fits in half
  // the pending run; otherwise per 32-column chunk.
  constexpr bool kTileReserve = C::BH / 8 <= C::PEND / 2;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  int off_b, off_l, off_bar;
  smem_layout_bytes<DPAD, SPLIT>(kp, nstage, &off_b, &off_l, &off_bar);
  uint8_t* sA = smem;
  uint8_t* sB = smem + off_b;
  uint2* sL = reinterpret_cast<uint2*>(smem + off_l);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + off_bar);
  uint64_t* full = bars;                        // [nstage]
  uint64_t* empty = bars + C::MAX_STAGE;        // [nstage]
  uint64_t* a_full = bars + 2 * C::MAX_STAGE;   // [1]
  uint64_t* a_empty = a_full + 1;               // [1]
  uint64_t* t_full = a_empty + 1;               // [NACC]
  uint64_t* t_empty = t_full + C::NACC;         // [NACC]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(t_empty + C::NACC);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < nstage; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(a_full, 1);
    mbar_init(a_empty, 1);
    for (int i = 0; i < C::NACC; ++i) {
      mbar_init(&t_full[i], 1);
      mbar_init(&t_empty[i], C::EPI_WARPS);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int64_t n_groups = n_qtiles;  // one query tile per item
  const int64_t n_items = n_groups * S;

  if (warp == 0) {
    // -------------------------------------------------------------- producer
    // The whole warp runs the loop (converged); one elected lane issues.
    int stage = 0;
    uint32_t phase = 0;
    uint32_t aphase = 0;
    for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int64_t qg = item % n_groups;
      const int c = (int)(item / n_groups);
      const int64_t t_lo = b_tiles * c / S, t_hi = b_tiles * (c + 1) / S;
      mbar_wait_backoff(a_empty, aphase ^ 1);
      aphase ^= 1;
      if (elect_one()) {
        mbar_arrive_expect_tx(a_full, QT * C::A_ONE);
        for (int s = 0; s < QT; ++s) {
          const int64_t qtl = qg * QT + s;  // local query tile (A image rows qtl*128..)
          uint8_t* dstA = sA + s * C::A_STRIDE;
          for (int kb = 0; kb < C::NKB; ++kb)
            bulk_g2s(dstA + kb * kBM * C::RB, a_img + kb * a_region + qtl * (int64_t)kBM * C::RB,
                     kBM * C::RB, a_full);
          bulk_g2s(dstA + C::A_EXTRA, a_img + a_extra + qtl * (int64_t)kBM * kExtraRB,
                   kBM * kExtraRB, a_full);
        }
      }
      __syncwarp();
      for (int64_t t = t_lo; t < t_hi; ++t) {
        mbar_wait_backoff(&empty[stage], phase ^ 1);
        if (elect_one()) {
          mbar_arrive_expect_tx(&full[stage], C::B_BYTES);
          uint8_t* dst = sB + stage * C::B_STRIDE;
          for (int kb = 0; kb < C::NKB; ++kb)
            bulk_g2s(dst + kb * C::BN * C::RB, b_img + kb * b_region + t * R * (int64_t)C::BN * C::RB,
                     C::BN * C::RB, &full[stage]);
          bulk_g2s(dst + C::B_EXTRA, b_img + b_extra + t * R * (int64_t)C::BN * kExtraRB,
                   C::BN * kExtraRB, &full[stage]);
        }
        __syncwarp();
        if (++stage == nstage) {
          stage = 0;
          phase ^= 1;
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    // Whole warp converged in the loop; descriptors precomputed (a shared-
    // memory descriptor advances by (bytes >> 4) in its low field); one elected
    // lane issues the MMAs and the commits that track them.
    constexpr uint32_t IDESC = idesc_f16(kBM, C::BN, FMT == 1 ? 0u : 1u);
    constexpr int NK = C::KSTEPS + 1;
    const uint32_t a_base = smem_u32(sA);
    const uint32_t b_base = smem_u32(sB);
    uint64_t adesc[NK], bdesc[NK];
#pragma unroll
    for (int ks = 0; ks < C::KSTEPS; ++ks) {
      const int kb = (ks * 32) / C::RB;
      const int koff = (ks * 32) % C::RB;
      adesc[ks] = smem_desc(a_base + kb * kBM * C::RB + koff, C::SBO, C::LAYOUT);
      bdesc[ks] = smem_desc(b_base + kb * C::BN * C::RB + koff, C::SBO, C::LAYOUT);
    }
    adesc[C::KSTEPS] = smem_desc(a_base + C::A_EXTRA, 8 * kExtraRB, 6);
    bdesc[C::KSTEPS] = smem_desc(b_base + C::B_EXTRA, 8 * kExtraRB, 6);
    int stage = 0;
    uint32_t phase = 0;
    int acc = 0;
    uint32_t acc_phase = 0;
    uint32_t aphase = 0;
    int ntr = 0;
    for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int c = (int)(item / n_groups);
      const int64_t t_lo = b_tiles * c / S, t_hi = b_tiles * (c + 1) / S;
      mbar_wait(a_full, aphase);
      aphase ^= 1;
      tc_fence_after();
      for (int64_t t = t_lo; t < t_hi; ++t) {
        const bool tr = trace && blockIdx.x == 0 && lane == 0 && ntr < kTraceTiles;
        if (tr) trace[ntr * 8 + 0] = clock64();
        mbar_wait(&full[stage], phase);
        tc_fence_after();
        if (tr) trace[ntr * 8 + 1] = clock64();
        const uint64_t bst = (uint64_t)((stage * C::B_STRIDE) >> 4);
#pragma unroll
        for (int s = 0; s < QT; ++s) {
          const int ai = acc * QT + s;
          mbar_wait(&t_empty[ai], acc_phase ^ 1);
          tc_fence_after();
          const uint32_t d_tmem = tmem_base + ai * C::BN;
          const uint64_t ast = (uint64_t)((s * C::A_STRIDE) >> 4);
          if (elect_one()) {
#pragma unroll
            for (int ks = 0; ks < NK; ++ks)
              tc_mma_f16(d_tmem, adesc[ks] + ast, bdesc[ks] + bst, IDESC, ks > 0 ? 1u : 0u);
            tc_commit(&t_full[ai]);
          }
          __syncwarp();
        }
        if (elect_one()) tc_commit(&empty[stage]);
        __syncwarp();
        if (tr) trace[ntr * 8 + 2] = clock64();
        ++ntr;
        if (++stage == nstage) {
          stage = 0;
          phase ^= 1;
        }
        if (++acc == C::NACC) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
      if (elect_one()) tc_commit(a_empty);
      __syncwarp();
    }
  } else {
    // ---------------------------------------------------------------- epilogue
    const int ew = warp - 2;          // epilogue warp index
    const int half = ew / 4;          // column part of each tile (0..SPLIT-1)
    const int q = warp & 3;           // TMEM lane quarter this warp may access
    const int t = q * 32 + lane;      // row within the query tile
    const int li = half * kBM + t;    // list slot (row, half)
    List L;
    L.init(sL, li, kp);
    int acc = 0;
    uint32_t acc_phase = 0;
    int etr = 0;
    constexpr int NCH = C::BH / 32;   // 32-column chunks per warp per tile (even)
    for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int64_t qg = item % n_groups;
      const int c = (int)(item / n_groups);  // reference chunk (chunk-major order)
      const int64_t t_lo = b_tiles * c / S, t_hi = b_tiles * (c + 1) / S;
      const int64_t qtl = qg;                // local query tile
      const int64_t row = (qt0 + qtl) * kBM + t;
      const int self = self_join ? (int)row : -1;
      // state layout: [query tile][half][slot][row]
      const int64_t st_base = ((qtl * SPLIT + half) * (int64_t)kp) * kBM + t;
      if (c > 0) {
        // Resume this (row, half)'s top-K'' after chunk c-1 (state parked in HBM).
        if (threadIdx.x == 64) {
          while (ld_acquire_gpu(st_done + qg) < c) __nanosleep(256);
        }
        named_bar(1, 32 * C::EPI_WARPS);
        int fill = 0;
        for (int e = 0; e < kp; ++e) {
          const uint2 kv = __ldcg(st_list + st_base + e * kBM);
          sts_kv(L.base + e * List::S, __uint_as_float(kv.x), (int)kv.y);
          fill += (int)kv.y >= 0;
        }
        L.fill = fill;
        L.thr = fill == kp ? lds_kv(L.base + (kp - 1) * List::S).x : CUDART_INF_F;
      }
      if (kTileReserve) L.reserve(C::BH / 8);
      for (int64_t tt = t_lo; tt < t_hi; ++tt) {
        const bool tr = trace && blockIdx.x == 0 && warp == 2 && lane == 0 && etr < kTraceTiles;
        if (tr) trace[etr * 8 + 3] = clock64();
        mbar_wait(&t_full[acc], acc_phase);
        tc_fence_after();
        if (tr) trace[etr * 8 + 4] = clock64();
        const uint32_t taddr =
            tmem_base + ((uint32_t)(q * 32) << 16) + acc * C::BN + half * C::BH;
        const int j0 = (int)(tt * R * C::BN) + half * C::BH;  // R > 1: strided sample tiles
        if (!(dbg & 1)) {
          // Masking is needed only on the last (padded) tile and on tiles that
          // contain some lane's own column: warp-uniform decision per tile.
          const bool diag = self_join && (self >= j0) && (self < j0 + C::BH);
          const bool masked = __any_sync(0xffffffffu, diag) || (j0 + C::BH > n_ref);
          // Group-min pass (every tile): for each 8-column group, a 3-input
          // min tree; a group whose minimum is below thr is appended to the
          // row's list as (min, group index) with predicated stores -- no
          // branches on the data.  The re-rank expands a kept group to its
          // 8 columns.
          const int gbase = j0 >> 3;
          auto groups = [&](const float(&v)[32], int ch) {
            float m[4];
#pragma unroll
            for (int g = 0; g < 4; ++g) {
              const float* vg = v + 8 * g;
              m[g] = fminf(fminf(fminf(vg[0], vg[1]), vg[2]),
                           fminf(fminf(vg[3], vg[4]), fminf(fminf(vg[5], vg[6]), vg[7])));
            }
            const float th = L.thr;
            if (!kTileReserve) L.reserve(4);
#pragma unroll
            for (int g = 0; g < 4; ++g) L.append_if(m[g] < th, m[g], gbase + ch * 4 + g);
          };
          if (!masked) {
            // 64 columns per TMEM load, waited on immediately: no register of
            // an in-flight tcgen05.ld may be touched (spilled, saved across a
            // call) before tcgen05.wait::ld, so nothing is kept in flight
            // across other work.  Latency is hidden by the other epilogue warps.
            if constexpr (NCH % 2 == 0) {
#pragma unroll
              for (int ch = 0; ch < NCH; ch += 2) {
                float v[64];
                tmem_ld64(taddr + ch * 32, v);
                tmem_ld_wait();
                groups(*reinterpret_cast<const float(*)[32]>(v), ch);
                groups(*reinterpret_cast<const float(*)[32]>(v + 32), ch + 1);
              }
            } else {
#pragma unroll
              for (int ch = 0; ch < NCH; ++ch) {
                float v[32];
                tmem_ld32(taddr + ch * 32, v);
                tmem_ld_wait();
                groups(v, ch);
              }
            }
          } else {
#pragma unroll 1
            for (int ch = 0; ch < NCH; ++ch) {
              float v[32];
              tmem_ld32(taddr + ch * 32, v);
              tmem_ld_wait();
              mask_cols(v, j0 + ch * 32, self, n_ref);
              groups(v, ch);
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (tr) trace[etr * 8 + 5] = clock64();
        ++etr;
        if (lane == 0) mbar_arrive(&t_empty[acc]);
        if (++acc == C::NACC) {
          acc = 0;
          acc_phase ^= 1;
        }
        // Room for the next tile's appends (at most one per 8-column group).
        // Merging only here, between tiles, keeps no TMEM values live across
        // the call, and all epilogue warps tend to merge at the same tile.
        if (kTileReserve) {
          const long long m0 = tr ? clock64() : 0;
          L.reserve(C::BH / 8);
          if (tr) {
            trace[(etr - 1) * 8 + 6] = clock64() - m0;  // merge (or check) cycles after this tile
            trace[(etr - 1) * 8 + 7] = (long long)(L.pa - (L.base + kp * List::S)) / List::S;
          }
        }
      }
      if (c < S - 1) {
        // Park this list's state for chunk c+1 (coalesced [slot][row] layout).
        if (__any_sync(0xffffffffu, L.pa != L.base + kp * List::S)) L.merge();
        for (int e = 0; e < kp; ++e) {
          const float2 kv = e < L.fill ? lds_kv(L.base + e * List::S)
                                       : make_float2(CUDART_INF_F, __int_as_float(-1));
          st_list[st_base + e * kBM] =
              make_uint2(__float_as_uint(kv.x), (unsigned)__float_as_int(kv.y));
        }
        __threadfence();
        named_bar(1, 32 * C::EPI_WARPS);
        if (threadIdx.x == 64) st_release_gpu(st_done + qg, c + 1);
      } else {
        const bool write = row >= q_begin && row < q_end;
        const int64_t r = row - q_begin;
        const int64_t co = write ? (r * SPLIT + half) * kp : 0;
        const float v = L.finish(cand_idx + co, write, cand_key + co);
        if (write) cand_v[r * SPLIT + half] = v;
      }
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

template <int DPAD, int FMT, int SPLIT>
cudaError_t launch_t(const Image& A, const Image& B, int64_t q_begin, int64_t q_count,
                     bool self_join, Cands c, int num_sms, cudaStream_t st) {
  using C = TcCfg<DPAD, SPLIT>;
  const int nstage = pick_stages<DPAD, SPLIT>(c.kp);
  if (nstage == 0) return cudaErrorInvalidValue;
  int ob, ol, obar;
  const int smem = smem_layout_bytes<DPAD, SPLIT>(c.kp, nstage, &ob, &ol, &obar);
  auto kern = k_knn_tc<DPAD, FMT, SPLIT>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const int64_t qt0 = q_begin / kBM;
  const int64_t qt1 = (q_begin + q_count + kBM - 1) / kBM;
  const int64_t n_items = (qt1 - qt0) * c.S;
  const int grid = (int)std::min<int64_t>(num_sms, n_items);
  if (grid <= 0) return cudaSuccess;
  if (c.S > 1 && (!c.st_list || !c.st_done)) return cudaErrorInvalidValue;
  if (c.lists != SPLIT) return cudaErrorInvalidValue;
  kern<<<grid, C::THREADS, smem, st>>>(
      reinterpret_cast<const uint8_t*>(A.data), A.region_bytes(), A.extra_offset(),
      reinterpret_cast<const uint8_t*>(B.data), B.region_bytes(), B.extra_offset(),
      (B.n_pad / C::BN + c.R - 1) / c.R, B.n, qt0, qt1 - qt0, q_begin, q_begin + q_count,
      self_join ? 1 : 0, c.S, c.R, c.kp, nstage, c.dbg, c.idx, c.v, c.key, c.st_list, c.st_done, c.trace);
  return cudaGetLastError();
}

template <int DPAD, int FMT>
cudaError_t launch_d(const Image& A, const Image& B, int64_t q_begin, int64_t q_count,
                     bool self_join, Cands c, int num_sms, cudaStream_t st) {
  if (c.lists == 4) return launch_t<DPAD, FMT, 4>(A, B, q_begin, q_count, self_join, c, num_sms, st);
  if (c.lists == 2) return launch_t<DPAD, FMT, 2>(A, B, q_begin, q_count, self_join, c, num_sms, st);
  return launch_t<DPAD, FMT, 1>(A, B, q_begin, q_count, self_join, c, num_sms, st);
}

}  // namespace

int tc_split_fits(int dpad, int kp, int split) {
#define TOD_FITS(D)                                                               \
  case D:                                                                         \
    return split == 4 ? pick_stages<D, 4>(kp) > 0                                 \
                      : (split == 2 ? pick_stages<D, 2>(kp) > 0 : pick_stages<D, 1>(kp) > 0);
  switch (dpad) {
    TOD_FITS(16)
    TOD_FITS(32)
    TOD_FITS(64)
    TOD_FITS(128)
  }
#undef TOD_FITS
  return 0;
}

cudaError_t launch_knn_tc(const Image& A, const Image& B, int64_t q_begin, int64_t q_count,
                          bool self_join, int fmt, Cands c, int num_sms, cudaStream_t st,
                          int* launches) {
  *launches += 1;
#define TOD_TC_CASE(D)                                                                      \
  case D:                                                                                  \
    return fmt == 1 ? launch_d<D, 1>(A, B, q_begin, q_count, self_join, c, num_sms, st)    \
                    : launch_d<D, 2>(A, B, q_begin, q_count, self_join, c, num_sms, st);
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
