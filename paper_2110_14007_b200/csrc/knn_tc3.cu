// knn_tc3.cu — K2 main pass and key-only sample pass (dpad <= 512): fused tile
// distance + threshold filter on tcgen05 tensor cores, append-only.
//
// Arithmetic: the tensor core produces, per (query row i,
// reference column j),
//     w_ij = ||xhat_j||^2 - 2 xhat_i . xhat_j
// i.e. Eq. (3)'s right-hand side minus the row constant (the norm
// enters through an extra 16-wide K block).  Each 8-column group's minimum is
// compared with the row's threshold tau_i and, when below, (min, group index)
// is appended to the row's candidate buffer in HBM (operator fusion of cdist
// and topk: the n x n matrix is never stored).
//
// tau_i comes from the SAMPLE pass over every R-th reference tile (this kernel's
// sample mode, keys only, or knn_tc.cu's list-based pass): every group NOT kept
// anywhere has key >= tau_i, which is all the certificate needs (DESIGN.md
// "Two-pass candidate selection").  With tau_i fixed for the whole pass there is
// no per-row set to maintain: the epilogue is a pure stream (min trees, one
// compare, predicated shared-memory append), and chunks of the same row may run
// concurrently (slots are reserved with one atomicAdd per flush).
//
// Structure (one CTA per SM, persistent; items = query tile x reference
// chunk, chunk-major so all SMs sweep the same L2-resident chunk):
//   warp 0     producer: bulk async copies (TMA engine) of the query tile and
//              a ring of 256-column reference tiles (dpad <= 64: A resident;
//              dpad > 64: A and B streamed per 64-wide K chunk), mbarrier
//              complete_tx.
//   warp 1     TMEM allocator + MMA issuer: (dpad+16)/16 MMAs 128x256x16 per
//              tile into one of two 256-column TMEM accumulators.
//   warps 2..  FW filter warps (16, or 8 when fewer operand stages fit): warp
//              (q, h) owns TMEM lane quarter q (32 rows) and column part h
//              (256 / (FW/4) columns) of every tile.
#include <math_constants.h>

#include <algorithm>

#include "internal.h"
#include "ptx.cuh"
#include "filter.cuh"

namespace tod {

namespace {

constexpr int kBM = 128;
constexpr int kBN = 256;
static_assert(kBN == 256, "filter addresses accumulators as acc << 8");
constexpr int kExtraRB = 32;
constexpr int kSmemMax = 232448;
constexpr int kMaxStage = 4;

__host__ __device__ constexpr int align_up(int x, int a) { return (x + a - 1) / a * a; }

template <int DPAD>
struct Cfg3 {
  static constexpr int RB = DPAD * 2 < 128 ? DPAD * 2 : 128;
  static constexpr int NKB = DPAD * 2 / RB;
  static constexpr int LAYOUT = RB == 128 ? 2 : (RB == 64 ? 4 : 6);
  static constexpr int SBO = 8 * RB;
  static constexpr int KSTEPS = DPAD / 16;
  static constexpr int A_ONE = kBM * (DPAD + 16) * 2;
  static constexpr int A_STRIDE = align_up(A_ONE, 1024);
  static constexpr int A_EXTRA = kBM * NKB * RB;
  static constexpr int B_BYTES = kBN * (DPAD + 16) * 2;
  static constexpr int B_STRIDE = align_up(B_BYTES, 1024);
  static constexpr int B_EXTRA = kBN * NKB * RB;
  // K-pipelined mode (dpad > 64): A and B both streamed, one 64-element K
  // region (or the 16-wide extra block) per ring stage.
  static constexpr bool KP = DPAD > 64;
  static constexpr int KS_A = kBM * 128;                 // A slice of a region (SW128)
  static constexpr int KS_BYTES = kBM * 128 + kBN * 128; // 48 KB
  static constexpr int KX_BYTES = kBM * 32 + kBN * 32;   // extra-block stage
};

// FW filter warps: 4 lane quarters x FW/4 column parts of every 256-column tile.
template <int DPAD, int FW>
__host__ __device__ constexpr int smem3(int nstage, int* off_b, int* off_p, int* off_bar) {
  using C = Cfg3<DPAD>;
  int o = C::KP ? 0 : C::A_STRIDE;
  *off_b = o;
  o += nstage * (C::KP ? C::KS_BYTES : C::B_STRIDE);
  *off_p = o;
  o += FW * kPendRun * 32 * 8;
  *off_bar = o;
  o += 8 * (2 * kMaxStage + 2 + 4) + 16;
  return o + 1024;
}

template <int DPAD, int FW>
int pick_stages3() {
  int a, b, c;
  for (int ns = kMaxStage; ns >= 2; --ns)
    if (smem3<DPAD, FW>(ns, &a, &b, &c) <= kSmemMax) return ns;
  return 0;
}

// MODE: 0 = main pass over every tile, 1 = main pass skipping the sample tiles
// (t % R == 0), 2 = main pass over only the sample tiles, 4 / 8 = sample pass
// keeping that many minima per (row, part).
template <int DPAD, int FMT, int DBG, int FW, int MODE, bool COL>
__global__ void __launch_bounds__(64 + 32 * FW, 1)
    k_knn_tc3(const uint8_t* __restrict__ a_img, size_t a_region, size_t a_extra,
              const uint8_t* __restrict__ b_img, size_t b_region, size_t b_extra, int64_t b_tiles,
              int64_t n_ref, int64_t qt0, int64_t n_qtiles, int64_t q_begin, int64_t q_end,
              int self_join, int S, int R, int nstage,
              const float* __restrict__ tau_v, int tau_lists,
              uint2* __restrict__ mbuf, int* __restrict__ mcnt, int cap,
              float* __restrict__ samp, int64_t col0, int samp_acc, int vote,
              long long* __restrict__ trace) {
  // trace (profiling): CTA 0, per tile in sweep order, [8] clock64 stamps:
  // 0 MMA: before the B-tile wait, 1 after it, 2 after the accumulator wait;
  // 3 filter warp 2: before the t_full wait, 4 after it, 5 accumulator released,
  // 6 filter done; 7 producer: B-tile copy issued.
  constexpr int kTraceTiles = 2048;  // x 16 stamps
  constexpr int kFWlast = FW;         // warp 1 + FW = the last filter warp
  constexpr bool TRACE = (DBG & 8) != 0;  // profiling build only (no trace code otherwise)
  const bool tron = TRACE && trace != nullptr && blockIdx.x == 0;
  using C = Cfg3<DPAD>;
  constexpr int SMP = MODE >= 4 ? MODE : 0;
  constexpr int SKIP = MODE == 1 ? 1 : 0;
  // MODE 2: the main pass (appends) over ONLY the sample tiles t % R == 0
  // (stage 2 of the three-stage selection)
  constexpr int WALK = (SMP > 0 || MODE == 2) ? 1 : 0;
  constexpr int H = FW / 4;        // column parts per tile
  constexpr int BH = kBN / H;      // columns per filter warp per tile
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  int off_b, off_p, off_bar;
  smem3<DPAD, FW>(nstage, &off_b, &off_p, &off_bar);
  uint8_t* sA = smem;
  uint8_t* sB = smem + off_b;
  const uint32_t s_pend = smem_u32(smem + off_p);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + off_bar);
  uint64_t* full = bars;
  uint64_t* empty = bars + kMaxStage;
  uint64_t* a_full = bars + 2 * kMaxStage;
  uint64_t* a_empty = a_full + 1;
  uint64_t* t_full = a_empty + 1;   // [2]
  uint64_t* t_empty = t_full + 2;   // [2]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(t_empty + 2);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int i = 0; i < nstage; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(a_full, 1);
    mbar_init(a_empty, 1);
    for (int i = 0; i < 2; ++i) {
      mbar_init(&t_full[i], 1);
      mbar_init(&t_empty[i], FW);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int64_t n_items = n_qtiles * S;

  if (warp == 0 && C::KP) {
    // ---------------------------------------- producer, K-pipelined (dpad > 64)
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int64_t qtl = item % n_qtiles;
      const int c = (int)(item / n_qtiles);
      TileSeq<WALK, SKIP> ts;
      ts.begin(b_tiles, S, R, c);
      for (; ts.more(); ts.next()) {
        const int64_t t = ts.t;
        for (int kb = 0; kb <= C::NKB; ++kb) {
          mbar_wait_backoff(&empty[stage], phase ^ 1);
          if (elect_one()) {
            uint8_t* dst = sB + stage * C::KS_BYTES;
            if (kb < C::NKB) {
              mbar_arrive_expect_tx(&full[stage], C::KS_BYTES);
              bulk_g2s(dst, a_img + kb * a_region + qtl * (int64_t)kBM * 128, kBM * 128, &full[stage]);
              bulk_g2s(dst + C::KS_A, b_img + kb * b_region + t * (int64_t)kBN * 128, kBN * 128,
                       &full[stage]);
            } else {
              mbar_arrive_expect_tx(&full[stage], C::KX_BYTES);
              bulk_g2s(dst, a_img + a_extra + qtl * (int64_t)kBM * kExtraRB, kBM * kExtraRB,
                       &full[stage]);
              bulk_g2s(dst + kBM * kExtraRB, b_img + b_extra + t * (int64_t)kBN * kExtraRB,
                       kBN * kExtraRB, &full[stage]);
            }
          }
          __syncwarp();
          if (++stage == nstage) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1 && C::KP) {
    // ------------------------------------------- MMA issuer, K-pipelined
    constexpr uint32_t IDESC = idesc_f16(kBM, kBN, FMT == 1 ? 0u : 1u);
    const uint32_t s_base = smem_u32(sB);
    int stage = 0, acc = 0;
    uint32_t phase = 0, acc_phase = 0;
    for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int c = (int)(item / n_qtiles);
      TileSeq<WALK, SKIP> ts;
      ts.begin(b_tiles, S, R, c);
      for (; ts.more(); ts.next()) {
        mbar_wait(&t_empty[acc], acc_phase ^ 1);
        for (int kb = 0; kb <= C::NKB; ++kb) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = s_base + stage * C::KS_BYTES;
          if (elect_one()) {
            if (kb < C::NKB) {
#pragma unroll
              for (int ks = 0; ks < 4; ++ks)
                tc_mma_f16(tmem_base + acc * kBN, smem_desc(a0 + ks * 32, 8 * 128, 2),
                           smem_desc(a0 + C::KS_A + ks * 32, 8 * 128, 2), IDESC,
                           (kb > 0 || ks > 0) ? 1u : 0u);
            } else {
              tc_mma_f16(tmem_base + acc * kBN, smem_desc(a0, 8 * kExtraRB, 6),
                         smem_desc(a0 + kBM * kExtraRB, 8 * kExtraRB, 6), IDESC, 1u);
              tc_commit(&t_full[acc]);
            }
            tc_commit(&empty[stage]);
          }
          __syncwarp();
          if (++stage == nstage) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (++acc == 2) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp == 0) {
    // -------------------------------------------------------------- producer
    int stage = 0;
    uint32_t phase = 0, aphase = 0;
    int ptr = 0;
    for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int64_t qtl = item % n_qtiles;
      const int c = (int)(item / n_qtiles);
      TileSeq<WALK, SKIP> ts;
      ts.begin(b_tiles, S, R, c);
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
      for (; ts.more(); ts.next()) {
        // the item's first B tiles are fetched while the MMA drains the previous item
        if (!a_done && issued == nstage - 1) load_a();
        mbar_wait_backoff(&empty[stage], phase ^ 1);
        if constexpr (TRACE)
          if (tron && lane == 0 && ptr < kTraceTiles) trace[ptr * 16 + 7] = clock64();
        ++ptr;
        if (elect_one()) {
          mbar_arrive_expect_tx(&full[stage], C::B_BYTES);
          uint8_t* dst = sB + stage * C::B_STRIDE;
          const int64_t t = ts.t;
          for (int kb = 0; kb < C::NKB; ++kb)
            bulk_g2s(dst + kb * kBN * C::RB, b_img + kb * b_region + t * (int64_t)kBN * C::RB,
                     kBN * C::RB, &full[stage]);
          bulk_g2s(dst + C::B_EXTRA, b_img + b_extra + t * (int64_t)kBN * kExtraRB,
                   kBN * kExtraRB, &full[stage]);
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
    constexpr uint32_t IDESC = idesc_f16(kBM, kBN, FMT == 1 ? 0u : 1u);
    constexpr int NK = C::KSTEPS + 1;
    const uint32_t a_base = smem_u32(sA);
    const uint32_t b_base = smem_u32(sB);
    uint64_t adesc[NK], bdesc[NK];
#pragma unroll
    for (int ks = 0; ks < C::KSTEPS; ++ks) {
      const int kb = (ks * 32) / C::RB;
      const int koff = (ks * 32) % C::RB;
      adesc[ks] = smem_desc(a_base + kb * kBM * C::RB + koff, C::SBO, C::LAYOUT);
      bdesc[ks] = smem_desc(b_base + kb * kBN * C::RB + koff, C::SBO, C::LAYOUT);
    }
    adesc[C::KSTEPS] = smem_desc(a_base + C::A_EXTRA, 8 * kExtraRB, 6);
    bdesc[C::KSTEPS] = smem_desc(b_base + C::B_EXTRA, 8 * kExtraRB, 6);
    int stage = 0, acc = 0;
    uint32_t phase = 0, acc_phase = 0, aphase = 0;
    int mtr = 0;
    for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int c = (int)(item / n_qtiles);
      TileSeq<WALK, SKIP> ts;
      ts.begin(b_tiles, S, R, c);
      mbar_wait(a_full, aphase);
      aphase ^= 1;
      tc_fence_after();
      for (; ts.more(); ts.next()) {
        const bool tr = TRACE && tron && lane == 0 && mtr < kTraceTiles;
        if (tr) trace[mtr * 16 + 0] = clock64();
        mbar_wait(&full[stage], phase);
        if (tr) trace[mtr * 16 + 1] = clock64();
        mbar_wait(&t_empty[acc], acc_phase ^ 1);
        if (tr) trace[mtr * 16 + 2] = clock64();
        ++mtr;
        tc_fence_after();
        const uint64_t bst = (uint64_t)((stage * C::B_STRIDE) >> 4);
        if (elect_one()) {
#pragma unroll
          for (int ks = 0; ks < NK; ++ks)
            tc_mma_f16(tmem_base + acc * kBN, adesc[ks], bdesc[ks] + bst, IDESC, ks > 0 ? 1u : 0u);
          tc_commit(&t_full[acc]);
          tc_commit(&empty[stage]);
        }
        __syncwarp();
        if (tr) trace[(mtr - 1) * 16 + 8] = clock64();
        if (++stage == nstage) {
          stage = 0;
          phase ^= 1;
        }
        if (++acc == 2) {
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
    const int q = warp & 3;           // TMEM lane quarter
    const int h = f >> 2;             // column part of every tile
    const int rt = q * 32 + lane;     // row within the query tile
    constexpr uint32_t SLOT = kPendSlot;
    const uint32_t pbase = s_pend + (f * kPendRun * 32 + lane) * 8;
    uint32_t pa = pbase;
    uint32_t tcount = 0;  // tiles consumed: accumulator = tcount & 1, phase = (tcount >> 1) & 1
    const uint32_t taddr0 = tmem_base + ((uint32_t)(q * 32) << 16) + h * BH;
    const uint32_t s_tfull = smem_u32(t_full), s_tempty = smem_u32(t_empty);
    for (int64_t item = blockIdx.x; item < n_items; item += gridDim.x) {
      const int64_t qtl = item % n_qtiles;
      const int c = (int)(item / n_qtiles);
      const int64_t row = (qt0 + qtl) * kBM + rt;
      const bool valid = row >= q_begin && row < q_end;
      const int64_t r = valid ? row - q_begin : 0;
      const int self = self_join ? (int)row : -1;
      // tiles that may need masking: the one holding this query tile's own
      // columns (self-join; the reference rows are the block [col0, col0 + n_ref)
      // of the global index space) and the last (padded) one
      const int64_t qrow0 = (qt0 + qtl) * kBM;
      const int t_self = (self_join && qrow0 >= col0 && qrow0 < col0 + n_ref)
                             ? (int)((qrow0 - col0) / kBN) : -1;
      const int t_last = (int)((n_ref - 1) / kBN);
      const int scol0 = (int)col0;
      float tau = -CUDART_INF_F;  // rows outside the range append nothing
      if (valid) {
        tau = CUDART_INF_F;
        for (int l = 0; l < tau_lists; ++l) tau = fminf(tau, tau_v[r * tau_lists + l]);
      }
      int* cnt = mcnt + r * H + h;
      uint2* buf = mbuf + (r * H + h) * (int64_t)cap;
      // move this lane's pending run to its HBM buffer (slots reserved atomically)
      auto flush = [&]() {
        const int n = (int)((pa - pbase) / SLOT);
        if (n > 0) {
          const int base = atomicAdd(cnt, n);
          for (int e = 0; e < n; ++e) {
            const float2 kv = lds_kv(pbase + e * SLOT);
            if (base + e < cap)
              buf[base + e] = make_uint2(__float_as_uint(kv.x), (unsigned)__float_as_int(kv.y));
          }
        }
        pa = pbase;
      };
      constexpr int T = SMP > 0 ? SMP : 1;  // sample pass: T smallest minima per (row, part)
      float top[T];
#pragma unroll
      for (int i = 0; i < T; ++i)  // a ring of blocks accumulates over launches
        top[i] = (SMP && samp_acc && valid) ? samp[(r * H + h) * T + i] : CUDART_INF_F;
      TileSeq<WALK, SKIP> ts;
      ts.begin(b_tiles, S, R, c);
      for (; ts.more(); ts.next()) {
        const uint32_t acc = tcount & 1u;
        const int etr = (int)tcount;
        const bool tr = TRACE && tron && warp == 2 && lane == 0 && etr < kTraceTiles;
        if (tr) trace[etr * 16 + 3] = clock64();
        mbar_wait_u32(s_tfull + acc * 8, (tcount >> 1) & 1u);
        if (tr) trace[etr * 16 + 4] = clock64();
        tc_fence_after();
        float v[BH];
        const uint32_t taddr = taddr0 + (acc << 8);  // acc * kBN
        if (!(DBG & 2)) {
#pragma unroll
          for (int u = 0; u < BH / 64; ++u)
            tmem_ld64(taddr + 64 * u, *reinterpret_cast<float(*)[64]>(v + 64 * u));
          tmem_ld_wait();
        }
        if (tr) trace[etr * 16 + 9] = clock64();
        auto release = [=]() {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_u32(s_tempty + acc * 8);
        };
        // column candidates (COL): filter_part releases after its vote
        if (!COL || SMP != 0 || DBG != 0) release();
        if (tr) trace[etr * 16 + 5] = clock64();
        if constexpr (TRACE)
          if (tron && warp == 1 + kFWlast && lane == 0 && etr < kTraceTiles) trace[etr * 16 + 10] = clock64();
        ++tcount;
        if (DBG & 3) continue;  // profiling: pipeline without the filter work
        const int t = ts.t;
        const int j0 = t * kBN + h * BH;
        if constexpr ((DBG & 4) != 0) {
          // diagnostics (tod_debug_mainpass): the raw accumulators w~ of the first
          // query tile, [128 x ld] fp32 in mbuf, ld = cap; no appends
          if (qtl == 0) {
            float* dump = reinterpret_cast<float*>(mbuf);
#pragma unroll
            for (int e = 0; e < BH; ++e)
              if (j0 + e < n_ref) dump[(int64_t)rt * cap + j0 + e] = v[e];
          }
          continue;
        }
        // the self column and padding columns (>= n_ref) are never candidates;
        // only the query tile's own reference tile and the last tile need masks
        const bool need_mask = t == t_self || t == t_last;
        if (need_mask) {
#pragma unroll
          for (int e = 0; e < BH; ++e)
            v[e] = (scol0 + j0 + e == self || j0 + e >= n_ref) ? CUDART_INF_F : v[e];
        }
        if constexpr (SMP) {
          float m[BH / 8];
#pragma unroll
          for (int g = 0; g < BH / 8; ++g) m[g] = min8(v + 8 * g);
          // sample pass: the T smallest group minima of this (row, part), keys
          // only, by a branch-free insertion network (new_i = min(r_i, max(r_i-1, x)))
#pragma unroll
          for (int g = 0; g < BH / 8; ++g) {
            const float x = m[g];
#pragma unroll
            for (int i = T - 1; i > 0; --i) top[i] = fminf(top[i], fmaxf(top[i - 1], x));
            top[0] = fminf(top[0], x);
          }
          continue;
        }
        auto reload = [=](int gg, float* c8) {
          tmem_ld8(taddr + 8 * gg, c8);
          tmem_ld_wait();
          if (need_mask) {
#pragma unroll
            for (int e = 0; e < 8; ++e) {
              const int jj = j0 + 8 * gg + e;
              if (scol0 + jj == self || jj >= n_ref) c8[e] = CUDART_INF_F;
            }
          }
        };
        filter_part<BH, COL>(v, tau, (scol0 + j0) >> 3, pa, pbase, vote != 0, flush, reload,
                             release);  // col0 % 256 == 0
        if (tr) trace[etr * 16 + 6] = clock64();
      }
      if constexpr (SMP) {
        if (valid) {
#pragma unroll
          for (int i = 0; i < T; ++i) samp[(r * H + h) * T + i] = top[i];
        }
      } else {
        flush();
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem_base, 512);
  }
}

template <int DPAD, int FMT, int DBG, int FW, int MODE, bool COL = false>
cudaError_t launch3(const Image& A, const Image& B, int64_t q_begin, int64_t q_count,
                    bool self_join, const MainPass& m, int num_sms, cudaStream_t st) {
  const int nstage = pick_stages3<DPAD, FW>();
  if (nstage == 0) return cudaErrorInvalidValue;
  if (m.parts != FW / 4) return cudaErrorInvalidValue;
  int a, b, c;
  const int smem = smem3<DPAD, FW>(nstage, &a, &b, &c);
  auto kern = k_knn_tc3<DPAD, FMT, DBG, FW, MODE, COL>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const int64_t qt0 = q_begin / kBM;
  const int64_t qt1 = (q_begin + q_count + kBM - 1) / kBM;
  const int64_t n_items = (qt1 - qt0) * m.S;
  const int grid = (int)std::min<int64_t>(num_sms, n_items);
  if (grid <= 0) return cudaSuccess;
  kern<<<grid, 64 + 32 * FW, smem, st>>>(
      reinterpret_cast<const uint8_t*>(A.data), A.region_bytes(), A.extra_offset(),
      reinterpret_cast<const uint8_t*>(B.data), B.region_bytes(), B.extra_offset(),
      (B.n + kBN - 1) / kBN, B.n, qt0, qt1 - qt0, q_begin, q_begin + q_count, self_join ? 1 : 0, m.S,
      m.R, nstage, m.tau_v, m.tau_lists, m.buf, m.cnt, m.cap, m.samp, m.col0, m.samp_acc, m.vote,
      m.trace);
  return cudaGetLastError();
}

// tau_i = the j-th smallest of the row's sample minima (parts x 4 values;
// +inf when fewer than j are finite, i.e. tiny inputs: keep everything).
__global__ void k_tau_combine(int64_t q, int nv, int j, const float* __restrict__ samp,
                              float* __restrict__ tau) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= q) return;
  float v[32];
#pragma unroll
  for (int e = 0; e < 32; ++e) v[e] = e < nv ? samp[r * nv + e] : CUDART_INF_F;
#pragma unroll
  for (int a = 1; a < 32; ++a)
#pragma unroll
    for (int b = a; b > 0; --b) {
      const float lo = fminf(v[b - 1], v[b]), hi = fmaxf(v[b - 1], v[b]);
      v[b - 1] = lo;
      v[b] = hi;
    }
  float t = CUDART_INF_F;
#pragma unroll
  for (int e = 0; e < 32; ++e) t = (e == j - 1) ? v[e] : t;
  tau[r] = t;
}

// Three-stage selection, stage 3: tau_r = min(tau0_r, the j-th smallest key the
// sample-tile sweep appended for row r over its parts) -- every non-appended
// sample column has w~ >= tau0 >= tau_r.  Fewer than j appends: tau0 stays.
__global__ void k_tau_from_appends(int64_t q, int parts, int cap, const int* __restrict__ cnt,
                                   const uint2* __restrict__ buf, int j, float* __restrict__ tau) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= q) return;
  float top[32];
#pragma unroll
  for (int i = 0; i < 32; ++i) top[i] = CUDART_INF_F;
  int total = 0;
  for (int h = 0; h < parts; ++h) {
    const int c = min(cnt[r * parts + h], cap);
    total += c;
    const uint2* b = buf + (r * parts + h) * (int64_t)cap;
    for (int e = 0; e < c; ++e) {
      const float x = __uint_as_float(__ldcg(b + e).x);
#pragma unroll
      for (int i = 31; i > 0; --i) top[i] = fminf(top[i], fmaxf(top[i - 1], x));
      top[0] = fminf(top[0], x);
    }
  }
  if (total >= j) {
    float t = CUDART_INF_F;
#pragma unroll
    for (int i = 0; i < 32; ++i) t = (i == j - 1) ? top[i] : t;
    tau[r] = fminf(tau[r], t);
  }
}

}  // namespace

cudaError_t launch_tau_from_appends(int64_t q, int parts, int cap, const int* cnt, const uint2* buf,
                                    int j, float* tau, cudaStream_t st, int* launches) {
  if (q <= 0) return cudaSuccess;
  j = j < 1 ? 1 : (j > 32 ? 32 : j);  // a smaller j only lowers tau (fewer candidates, still valid)
  k_tau_from_appends<<<(unsigned)((q + 127) / 128), 128, 0, st>>>(q, parts, cap, cnt, buf, j, tau);
  *launches += 1;
  return cudaGetLastError();
}

cudaError_t launch_tau_combine(int64_t q, int nv, int j, const float* samp, float* tau,
                               cudaStream_t st, int* launches) {
  if (q <= 0) return cudaSuccess;
  if (nv > 32 || j < 1 || j > nv) return cudaErrorInvalidValue;
  k_tau_combine<<<(unsigned)((q + 255) / 256), 256, 0, st>>>(q, nv, j, samp, tau);
  *launches += 1;
  return cudaGetLastError();
}

// Filter warps per CTA: 16 (4 per SM sub-partition, 64 columns each) when 3+
// operand stages still fit in shared memory, else 8.
template <int DPAD>
int tc3_fw() {
  return pick_stages3<DPAD, 16>() >= 3 ? 16 : (pick_stages3<DPAD, 8>() > 0 ? 8 : 0);
}

int tc3_parts(int dpad) {
  switch (dpad) {
    case 16: return tc3_fw<16>() / 4;
    case 32: return tc3_fw<32>() / 4;
    case 64: return tc3_fw<64>() / 4;
    case 128: return tc3_fw<128>() / 4;
    case 256: return tc3_fw<256>() / 4;
    case 512: return tc3_fw<512>() / 4;
  }
  return 0;
}

int tc3_fits(int dpad) { return tc3_parts(dpad) > 0; }

cudaError_t launch_knn_tc3(const Image& A, const Image& B, int64_t q_begin, int64_t q_count,
                           bool self_join, int fmt, const MainPass& m, int num_sms, int dbg,
                           cudaStream_t st, int* launches) {
  *launches += 1;
  // dbg (profiling only): 1 = skip the filter work (fp16), 2 = also skip the TMEM loads
#define TOD_TC3_FW(D, FW)                                                                          \
  if (m.samp && m.samp_t == 8)                                                                    \
    return fmt == 1 ? launch3<D, 1, 0, FW, 8>(A, B, q_begin, q_count, self_join, m, num_sms, st)  \
                    : launch3<D, 2, 0, FW, 8>(A, B, q_begin, q_count, self_join, m, num_sms, st); \
  if (m.samp)                                                                                     \
    return fmt == 1 ? launch3<D, 1, 0, FW, 4>(A, B, q_begin, q_count, self_join, m, num_sms, st)  \
                    : launch3<D, 2, 0, FW, 4>(A, B, q_begin, q_count, self_join, m, num_sms, st); \
  if (m.smode) {  /* three-stage, stage 2 (d <= 32 on the single-SM kernel) */                   \
    if constexpr (D <= 32 && FW == 16)                                                           \
      return fmt == 1 ? launch3<D, 1, 0, FW, 2>(A, B, q_begin, q_count, self_join, m, num_sms, st) \
                      : launch3<D, 2, 0, FW, 2>(A, B, q_begin, q_count, self_join, m, num_sms, st); \
    return cudaErrorInvalidValue;                                                                \
  }                                                                                               \
  if (dbg & 4)                                                                                    \
    return fmt == 1 ? launch3<D, 1, 4, FW, 0>(A, B, q_begin, q_count, self_join, m, num_sms, st)  \
                    : launch3<D, 2, 4, FW, 0>(A, B, q_begin, q_count, self_join, m, num_sms, st); \
  if ((dbg & 3) == 1 && fmt == 1)                                                                 \
    return launch3<D, 1, 1, FW, 1>(A, B, q_begin, q_count, self_join, m, num_sms, st);            \
  if (dbg & 3)                                                                                    \
    return fmt == 1 ? launch3<D, 1, 2, FW, 1>(A, B, q_begin, q_count, self_join, m, num_sms, st)  \
                    : launch3<D, 2, 2, FW, 1>(A, B, q_begin, q_count, self_join, m, num_sms, st); \
  if ((dbg & 8) && m.R > 0)  /* profiling trace build */                                       \
    return fmt == 1 ? launch3<D, 1, 8, FW, 1>(A, B, q_begin, q_count, self_join, m, num_sms, st)  \
                    : launch3<D, 2, 8, FW, 1>(A, B, q_begin, q_count, self_join, m, num_sms, st); \
  if (dbg & 8)                                                                                    \
    return fmt == 1 ? launch3<D, 1, 8, FW, 0>(A, B, q_begin, q_count, self_join, m, num_sms, st)  \
                    : launch3<D, 2, 8, FW, 0>(A, B, q_begin, q_count, self_join, m, num_sms, st); \
  if (m.R > 0 && m.colmode)                                                                      \
    return fmt == 1 ? launch3<D, 1, 0, FW, 1, true>(A, B, q_begin, q_count, self_join, m, num_sms, st)  \
                    : launch3<D, 2, 0, FW, 1, true>(A, B, q_begin, q_count, self_join, m, num_sms, st); \
  if (m.R > 0)                                                                                    \
    return fmt == 1 ? launch3<D, 1, 0, FW, 1>(A, B, q_begin, q_count, self_join, m, num_sms, st)  \
                    : launch3<D, 2, 0, FW, 1>(A, B, q_begin, q_count, self_join, m, num_sms, st); \
  if (m.colmode)                                                                                  \
    return fmt == 1 ? launch3<D, 1, 0, FW, 0, true>(A, B, q_begin, q_count, self_join, m, num_sms, st)  \
                    : launch3<D, 2, 0, FW, 0, true>(A, B, q_begin, q_count, self_join, m, num_sms, st); \
  return fmt == 1 ? launch3<D, 1, 0, FW, 0>(A, B, q_begin, q_count, self_join, m, num_sms, st)    \
                  : launch3<D, 2, 0, FW, 0>(A, B, q_begin, q_count, self_join, m, num_sms, st);
#define TOD_TC3_CASE(D)          \
  case D:                        \
    if (tc3_fw<D>() == 16) {     \
      TOD_TC3_FW(D, 16)          \
    } else {                     \
      TOD_TC3_FW(D, 8)           \
    }
  switch (A.dpad) {
    TOD_TC3_CASE(16)
    TOD_TC3_CASE(32)
    TOD_TC3_CASE(64)
    TOD_TC3_CASE(128)
    TOD_TC3_CASE(256)
    TOD_TC3_CASE(512)
  }
#undef TOD_TC3_CASE
#undef TOD_TC3_FW
  return cudaErrorInvalidValue;
}

}  // namespace tod
