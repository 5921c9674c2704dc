// knn_tc4.cu — K2 main pass on CTA PAIRS (tcgen05 cta_group::2); dpad <= 64 with
// the query tile resident, dpad > 64 K-pipelined (A and B slices streamed per K region).
//
// Same computation as knn_tc3.cu (the append-only threshold filter of the
// two-pass candidate selection; arithmetic of Eq. (3)'s right-hand
// side, fused with topk), scheduled for the measured
// bottleneck of the single-SM version: shared-memory bandwidth.  A 128x256
// single-SM MMA step reads its whole A and B tiles from one SM's shared memory
// and the B tile is also written there by the copy engine (~1.9 bytes per
// distance at d = 32 against 128 B/clk).  Here two SMs of a cluster issue one
// M = 256 MMA (leader CTA only): each SM stages its own 128 query rows (A) and
// HALF of every 256-column reference tile (B), and receives its 128 x 256
// slice of the product in its own TMEM.  Per-SM operand traffic per distance
// falls by ~40 % (B is written and read once per pair, not once per SM).
//
// Synchronisation across the pair (barriers live at the same shared offset in
// both CTAs):
//   full[s], a_full     CTA 0: arrival count 2 = its own expect_tx arrival +
//                       a forwarded arrival from CTA 1 once CTA 1's copy landed
//                       (CTA 1's warp 1 forwards; CTA 1's own barriers count 1).
//   empty[s], a_empty,  multicast tcgen05.commit from the leader's MMA thread
//   t_full[acc]         to both CTAs.
//   t_empty[acc]        CTA 0 only: all 32 filter warps of the pair arrive
//                       (CTA 1's remotely) before the accumulator is reused.
//
// Two tile geometries (template NB, NACC): 256-column tiles with two
// accumulators (2 x 256 TMEM columns; the tile grid of the list-based sample
// pass), or 160-column tiles with THREE accumulators (3 x 160): the per-tile
// trace showed the accumulator hand-off on the critical path with two
// (the MMA of tile t+2 waits for the filter warps of both SMs to release t);
// with three, two tiles' MMAs are queued while the filter drains the third.
// A tile is any multiple of 8 rows of the swizzled image (the image keeps 256
// rows of slack past n_pad for the last 160-row tile).  smode 1 sweeps only the
// sample tiles t % R == 0 (the three-stage candidate selection).
#include <math_constants.h>

#include <algorithm>

#include "internal.h"
#include "ptx.cuh"
#include "filter.cuh"

namespace tod {

namespace {

constexpr int kBM = 128;        // query rows per CTA (= TMEM lanes)
constexpr int kMaxAcc = 3;      // accumulators in the TMEM ring (NACC <= 3)
constexpr int kExtraRB = 32;
constexpr int kSmemMax = 232448;
constexpr int kMaxStage = 6;

__host__ __device__ constexpr int align_up(int x, int a) { return (x + a - 1) / a * a; }

template <int DPAD, int NB>
struct Cfg4 {
  static constexpr int NBH = NB / 2;  // reference rows of each tile staged per CTA
  static constexpr int RB = DPAD * 2 < 128 ? DPAD * 2 : 128;
  static constexpr int NKB = DPAD * 2 / RB;
  static constexpr int LAYOUT = RB == 128 ? 2 : (RB == 64 ? 4 : 6);
  static constexpr int SBO = 8 * RB;
  static constexpr int KSTEPS = DPAD / 16;
  static constexpr int A_ONE = kBM * (DPAD + 16) * 2;
  static constexpr int A_STRIDE = align_up(A_ONE, 1024);
  static constexpr int A_EXTRA = kBM * NKB * RB;
  static constexpr int B_BYTES = NBH * (DPAD + 16) * 2;    // this CTA's half tile
  static constexpr int B_STRIDE = align_up(B_BYTES, 1024);
  static constexpr int B_EXTRA = NBH * NKB * RB;
  // K-pipelined mode (dpad > 64): each CTA streams its own A slice and its half
  // of the B slice of one 64-element K region (or of the 16-wide extra block)
  // per ring stage: 32 KB per SM per region against the single-SM kernel's 48 KB
  // (its 128 query rows + all 256 reference rows) -- the L2 -> SM operand traffic
  // that bounds the single-SM K-pipelined pass at d = 512.
  static constexpr bool KP = DPAD > 64;
  static constexpr int KS_A = kBM * 128;
  static constexpr int KS_BYTES = kBM * 128 + NBH * 128;
  static constexpr int KX_BYTES = kBM * kExtraRB + NBH * kExtraRB;
};

template <int DPAD, int FW, int NB>
__host__ __device__ constexpr int smem4(int nstage, int* off_b, int* off_p, int* off_bar) {
  using C = Cfg4<DPAD, NB>;
  int o = C::KP ? 0 : C::A_STRIDE;
  *off_b = o;
  o += nstage * (C::KP ? align_up(C::KS_BYTES, 1024) : C::B_STRIDE);
  *off_p = o;
  o += FW * kPendRun * 32 * 8;
  *off_bar = o;
  o += 8 * (2 * kMaxStage + 2 + 2 * kMaxAcc) + 16;
  return o + 1024;
}

template <int DPAD, int FW, int NB>
int pick_stages4() {
  int a, b, c;
  for (int ns = kMaxStage; ns >= 2; --ns)
    if (smem4<DPAD, FW, NB>(ns, &a, &b, &c) <= kSmemMax) return ns;
  return 0;
}

// TMEM reads of one filter warp's part: BH consecutive columns (64 or 40).
template <int BH>
__device__ __forceinline__ void tmem_ld_cols(uint32_t taddr, float* v) {
  static_assert(BH == 64 || BH == 40, "part width");
  if constexpr (BH == 64) {
    tmem_ld64(taddr, *reinterpret_cast<float(*)[64]>(v));
  } else {
    tmem_ld32(taddr, *reinterpret_cast<float(*)[32]>(v));
    tmem_ld8(taddr + 32, v + 32);
  }
}

// SMP (4 or 8; K-pipelined pairs, dpad > 64): the key-only SAMPLE pass -- no
// appends; each filter lane keeps the SMP smallest group minima of its (row,
// part) over the tiles of the sweep (smode 1: the sample tiles) and writes them
// to samp (knn_tc3.cu's sample mode on CTA pairs).
template <int DPAD, int FMT, int DBG, int FW, bool COL, int NB, int NACC, int SMP = 0>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(64 + 32 * FW, 1)
    k_knn_tc4(const uint8_t* __restrict__ a_img, size_t a_region, size_t a_extra,
              const uint8_t* __restrict__ b_img, size_t b_region, size_t b_extra, int64_t b_tiles,
              int64_t n_ref, int64_t qt0, int64_t n_qpairs, int64_t q_begin, int64_t q_end,
              int self_join, int S, int R, int nstage,
              const float* __restrict__ tau_v, int tau_lists,
              uint2* __restrict__ mbuf, int* __restrict__ mcnt, int cap, int64_t col0, int vote,
              int smode, long long* __restrict__ trace, float* __restrict__ samp) {
  // trace (profiling, TOD_F_DEBUG_TRACE): the leader CTA of cluster 0, per tile,
  // the 16 clock64 stamps of knn_tc3.cu (tools/trace_main.py)
  constexpr int kTraceTiles = 2048;
  using C = Cfg4<DPAD, NB>;
  constexpr int H = FW / 4;
  constexpr int BH = NB / H;
  constexpr int NBH = C::NBH;
  static_assert(NB * NACC <= 512 && NACC <= kMaxAcc, "accumulator ring must fit TMEM");
  extern __shared__ uint8_t smem_raw[];
  // identical layout in both CTAs: every offset below is valid in the peer too
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  int off_b, off_p, off_bar;
  smem4<DPAD, FW, NB>(nstage, &off_b, &off_p, &off_bar);
  uint8_t* sA = smem;
  uint8_t* sB = smem + off_b;
  const uint32_t s_pend = smem_u32(smem + off_p);
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + off_bar);
  uint64_t* full = bars;
  uint64_t* empty = bars + kMaxStage;
  uint64_t* a_full = bars + 2 * kMaxStage;
  uint64_t* a_empty = a_full + 1;
  uint64_t* t_full = a_empty + 1;      // [NACC]
  uint64_t* t_empty = t_full + NACC;   // [NACC]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(t_empty + NACC);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const uint32_t rank = cluster_ctarank();
  const bool leader = rank == 0;

  if (threadIdx.x == 0) {
    for (int i = 0; i < nstage; ++i) {
      mbar_init(&full[i], leader ? 2 : 1);
      mbar_init(&empty[i], 1);
    }
    mbar_init(a_full, leader ? 2 : 1);
    mbar_init(a_empty, 1);
    for (int i = 0; i < NACC; ++i) {
      mbar_init(&t_full[i], 1);
      mbar_init(&t_empty[i], 2 * FW);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc2(tmem_slot, 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  const int64_t n_items = n_qpairs * S;
  const int64_t cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;
  constexpr bool TRACE = (DBG & 8) != 0;  // profiling build only
  const bool tron = TRACE && trace != nullptr && blockIdx.x == 0;

  if (warp == 0 && C::KP) {
    // ------------------------------------------------ producer, K-pipelined
    // (both CTAs: per K region, own query-tile slice + own half of the B slice)
    constexpr int KSB = align_up(C::KS_BYTES, 1024);
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t item = cid; item < n_items; item += ncl) {
      const int64_t qtl = (item % n_qpairs) * 2 + rank;
      const int c = (int)(item / n_qpairs);
      TileSeqRT ts;
      ts.begin(b_tiles, S, R, c, smode);
      for (; ts.more(); ts.next()) {
        const int64_t row0 = (int64_t)ts.t * NB + rank * NBH;
        for (int kb = 0; kb <= C::NKB; ++kb) {
          mbar_wait_cl_backoff(&empty[stage], phase ^ 1);
          if (elect_one()) {
            uint8_t* dst = sB + stage * KSB;
            if (kb < C::NKB) {
              mbar_arrive_expect_tx(&full[stage], C::KS_BYTES);
              bulk_g2s(dst, a_img + kb * a_region + qtl * (int64_t)kBM * 128, kBM * 128, &full[stage]);
              bulk_g2s(dst + C::KS_A, b_img + kb * b_region + row0 * 128, NBH * 128, &full[stage]);
            } else {
              mbar_arrive_expect_tx(&full[stage], C::KX_BYTES);
              bulk_g2s(dst, a_img + a_extra + qtl * (int64_t)kBM * kExtraRB, kBM * kExtraRB,
                       &full[stage]);
              bulk_g2s(dst + kBM * kExtraRB, b_img + b_extra + row0 * kExtraRB, NBH * kExtraRB,
                       &full[stage]);
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
  } else if (warp == 1 && leader && C::KP) {
    // ------------------------------- MMA issuer (leader CTA), K-pipelined
    constexpr uint32_t IDESC = idesc_f16(2 * kBM, NB, FMT == 1 ? 0u : 1u);
    constexpr int KSB = align_up(C::KS_BYTES, 1024);
    const uint32_t s_base = smem_u32(sB);
    int stage = 0, acc = 0;
    uint32_t phase = 0, acc_phase = 0;
    for (int64_t item = cid; item < n_items; item += ncl) {
      const int c = (int)(item / n_qpairs);
      TileSeqRT ts;
      ts.begin(b_tiles, S, R, c, smode);
      for (; ts.more(); ts.next()) {
        mbar_wait_cl(&t_empty[acc], acc_phase ^ 1);
        for (int kb = 0; kb <= C::NKB; ++kb) {
          mbar_wait_cl(&full[stage], phase);
          tc_fence_after();
          const uint32_t a0 = s_base + stage * KSB;
          if (elect_one()) {
            if (kb < C::NKB) {
#pragma unroll
              for (int ks = 0; ks < 4; ++ks)
                tc_mma_f16_2cta(tmem_base + acc * NB, smem_desc(a0 + ks * 32, 8 * 128, 2),
                                smem_desc(a0 + C::KS_A + ks * 32, 8 * 128, 2), IDESC,
                                (kb > 0 || ks > 0) ? 1u : 0u);
            } else {
              tc_mma_f16_2cta(tmem_base + acc * NB, smem_desc(a0, 8 * kExtraRB, 6),
                              smem_desc(a0 + kBM * kExtraRB, 8 * kExtraRB, 6), IDESC, 1u);
              tc_commit_mc(&t_full[acc], 0x3);
            }
            tc_commit_mc(&empty[stage], 0x3);
          }
          __syncwarp();
          if (++stage == nstage) {
            stage = 0;
            phase ^= 1;
          }
        }
        if (++acc == NACC) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
    }
  } else if (warp == 1 && C::KP) {
    // ------------------- forwarder (CTA 1), K-pipelined: every stage landed
    const uint32_t r_full = mapa_shared(smem_u32(full), 0);
    int stage = 0;
    uint32_t phase = 0;
    for (int64_t item = cid; item < n_items; item += ncl) {
      const int c = (int)(item / n_qpairs);
      TileSeqRT ts;
      ts.begin(b_tiles, S, R, c, smode);
      for (; ts.more(); ts.next()) {
        for (int kb = 0; kb <= C::NKB; ++kb) {
          mbar_wait_cl(&full[stage], phase);
          if (lane == 0) mbar_arrive_cluster(r_full + stage * 8);
          __syncwarp();
          if (++stage == nstage) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 0) {
    // -------------------------------------------------------------- producer
    // (both CTAs: own query tile, own half of each reference tile)
    int stage = 0;
    uint32_t phase = 0, aphase = 0;
    int ptr = 0;
    for (int64_t item = cid; item < n_items; item += ncl) {
      const int64_t qtl = (item % n_qpairs) * 2 + rank;
      const int c = (int)(item / n_qpairs);
      TileSeqRT ts;
      ts.begin(b_tiles, S, R, c, smode);
      int issued = 0;
      bool a_done = false;
      auto load_a = [&]() {
        mbar_wait_cl_backoff(a_empty, aphase ^ 1);
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
        if (!a_done && issued == nstage - 1) load_a();
        mbar_wait_cl_backoff(&empty[stage], phase ^ 1);
        if constexpr (TRACE)
          if (tron && lane == 0 && ptr < kTraceTiles) trace[ptr * 16 + 7] = clock64();
        ++ptr;
        if (elect_one()) {
          mbar_arrive_expect_tx(&full[stage], C::B_BYTES);
          uint8_t* dst = sB + stage * C::B_STRIDE;
          const int64_t row0 = (int64_t)ts.t * NB + rank * NBH;
          for (int kb = 0; kb < C::NKB; ++kb)
            bulk_g2s(dst + kb * NBH * C::RB, b_img + kb * b_region + row0 * C::RB,
                     NBH * C::RB, &full[stage]);
          bulk_g2s(dst + C::B_EXTRA, b_img + b_extra + row0 * kExtraRB, NBH * kExtraRB,
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
  } else if (warp == 1 && leader) {
    // --------------------------------------------- MMA issuer (leader CTA)
    constexpr uint32_t IDESC = idesc_f16(2 * kBM, NB, FMT == 1 ? 0u : 1u);
    constexpr int NK = C::KSTEPS + 1;
    const uint32_t a_base = smem_u32(sA);
    const uint32_t b_base = smem_u32(sB);
    uint64_t adesc[NK], bdesc[NK];
#pragma unroll
    for (int ks = 0; ks < C::KSTEPS; ++ks) {
      const int kb = (ks * 32) / C::RB;
      const int koff = (ks * 32) % C::RB;
      adesc[ks] = smem_desc(a_base + kb * kBM * C::RB + koff, C::SBO, C::LAYOUT);
      bdesc[ks] = smem_desc(b_base + kb * NBH * C::RB + koff, C::SBO, C::LAYOUT);
    }
    adesc[C::KSTEPS] = smem_desc(a_base + C::A_EXTRA, 8 * kExtraRB, 6);
    bdesc[C::KSTEPS] = smem_desc(b_base + C::B_EXTRA, 8 * kExtraRB, 6);
    int stage = 0, acc = 0;
    uint32_t phase = 0, acc_phase = 0, aphase = 0;
    int mtr = 0;
    for (int64_t item = cid; item < n_items; item += ncl) {
      const int c = (int)(item / n_qpairs);
      TileSeqRT ts;
      ts.begin(b_tiles, S, R, c, smode);
      mbar_wait_cl(a_full, aphase);
      aphase ^= 1;
      tc_fence_after();
      for (; ts.more(); ts.next()) {
        const bool tr = TRACE && tron && lane == 0 && mtr < kTraceTiles;
        if (tr) trace[mtr * 16 + 0] = clock64();
        mbar_wait_cl(&full[stage], phase);
        if (tr) trace[mtr * 16 + 1] = clock64();
        mbar_wait_cl(&t_empty[acc], acc_phase ^ 1);
        if (tr) trace[mtr * 16 + 2] = clock64();
        tc_fence_after();
        const uint64_t bst = (uint64_t)((stage * C::B_STRIDE) >> 4);
        if (elect_one()) {
#pragma unroll
          for (int ks = 0; ks < NK; ++ks)
            tc_mma_f16_2cta(tmem_base + acc * NB, adesc[ks], bdesc[ks] + bst, IDESC,
                            ks > 0 ? 1u : 0u);
          tc_commit_mc(&t_full[acc], 0x3);
          tc_commit_mc(&empty[stage], 0x3);
        }
        __syncwarp();
        if (tr) trace[mtr * 16 + 8] = clock64();
        ++mtr;
        if (++stage == nstage) {
          stage = 0;
          phase ^= 1;
        }
        if (++acc == NACC) {
          acc = 0;
          acc_phase ^= 1;
        }
      }
      if (elect_one()) tc_commit_mc(a_empty, 0x3);
      __syncwarp();
    }
  } else if (warp == 1) {
    // ---------------------------------- forwarder (CTA 1): copies landed here
    const uint32_t r_full = mapa_shared(smem_u32(full), 0);
    const uint32_t r_afull = mapa_shared(smem_u32(a_full), 0);
    int stage = 0;
    uint32_t phase = 0, aphase = 0;
    for (int64_t item = cid; item < n_items; item += ncl) {
      const int c = (int)(item / n_qpairs);
      TileSeqRT ts;
      ts.begin(b_tiles, S, R, c, smode);
      // the producer may issue up to nstage-1 B tiles before the A tile: the
      // forwarder must not block on A first (the leader needs those B tiles
      // to finish the previous item, which releases A)
      int fwd = 0;
      bool a_fwd = false;
      for (; ts.more(); ts.next()) {
        if (!a_fwd && fwd == nstage - 1) {
          mbar_wait_cl(a_full, aphase);
          aphase ^= 1;
          if (lane == 0) mbar_arrive_cluster(r_afull);
          a_fwd = true;
        }
        mbar_wait_cl(&full[stage], phase);
        if (lane == 0) mbar_arrive_cluster(r_full + stage * 8);
        __syncwarp();
        ++fwd;
        if (++stage == nstage) {
          stage = 0;
          phase ^= 1;
        }
      }
      if (!a_fwd) {
        mbar_wait_cl(a_full, aphase);
        aphase ^= 1;
        if (lane == 0) mbar_arrive_cluster(r_afull);
      }
      __syncwarp();
    }
  } else {
    // --------------------------------------------------------- filter warps
    const int f = warp - 2;
    const int q = warp & 3;
    const int h = f >> 2;
    const int rt = q * 32 + lane;
    constexpr uint32_t SLOT = kPendSlot;
    const uint32_t pbase = s_pend + (f * kPendRun * 32 + lane) * 8;
    uint32_t pa = pbase;
    uint32_t acc = 0, acc_phase = 0;  // accumulator ring position of the next tile
    int etr = 0;
    const uint32_t taddr0 = tmem_base + ((uint32_t)(q * 32) << 16) + h * BH;
    const uint32_t r_tempty = mapa_shared(smem_u32(t_empty), 0);
    const uint32_t s_tfull = smem_u32(t_full), s_tempty = smem_u32(t_empty);
    for (int64_t item = cid; item < n_items; item += ncl) {
      const int64_t qtl = (item % n_qpairs) * 2 + rank;
      const int c = (int)(item / n_qpairs);
      const int64_t row = (qt0 + qtl) * kBM + rt;
      const bool valid = row >= q_begin && row < q_end;
      const int64_t r = valid ? row - q_begin : 0;
      // reference rows = the block [col0, col0 + n_ref) of the global index space;
      // the self column (block-relative) and padding columns are never candidates
      const int64_t selfc = self_join ? row - col0 : -1;
      const int scol0 = (int)col0;
      float tau = -CUDART_INF_F;
      if (valid) {
        tau = CUDART_INF_F;
        for (int l = 0; l < tau_lists; ++l) tau = fminf(tau, tau_v[r * tau_lists + l]);
      }
      int* cnt = mcnt + r * H + h;
      uint2* buf = mbuf + (r * H + h) * (int64_t)cap;
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
      constexpr int T = SMP > 0 ? SMP : 1;
      float top[T];
#pragma unroll
      for (int i = 0; i < T; ++i) top[i] = CUDART_INF_F;
      TileSeqRT ts;
      ts.begin(b_tiles, S, R, c, smode);
      for (; ts.more(); ts.next()) {
        const bool tr = TRACE && tron && warp == 2 && lane == 0 && etr < kTraceTiles;
        if (tr) trace[etr * 16 + 3] = clock64();
        mbar_wait_u32(s_tfull + acc * 8, acc_phase);
        if (tr) trace[etr * 16 + 4] = clock64();
        tc_fence_after();
        float v[BH];
        const uint32_t taddr = taddr0 + acc * NB;
        if (!(DBG & 2)) {
          tmem_ld_cols<BH>(taddr, v);
          tmem_ld_wait();
        }
        if (tr) trace[etr * 16 + 9] = clock64();
        auto release = [=]() {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (leader) mbar_arrive_u32(s_tempty + acc * 8);
            else mbar_arrive_cluster(r_tempty + acc * 8);
          }
        };
        // column candidates (COL): filter_part releases after its vote
        if (!COL || DBG != 0) release();
        if (tr) trace[etr * 16 + 5] = clock64();
        if constexpr (TRACE)
          if (tron && warp == 1 + FW && lane == 0 && etr < kTraceTiles) trace[etr * 16 + 10] = clock64();
        ++etr;
        if (++acc == NACC) {
          acc = 0;
          acc_phase ^= 1;
        }
        if (DBG & 3) continue;
        const int t = ts.t;
        const int j0 = t * NB + h * BH;
        if constexpr ((DBG & 4) != 0) {
          // diagnostics (tod_debug_mainpass): raw w~ of the first query tile (CTA 0)
          if (qtl == 0) {
            float* dump = reinterpret_cast<float*>(mbuf);
#pragma unroll
            for (int e = 0; e < BH; ++e)
              if (j0 + e < n_ref) dump[(int64_t)rt * cap + j0 + e] = v[e];
          }
          continue;
        }
        const bool need_mask = (uint64_t)(selfc - j0) < (uint64_t)BH || j0 + BH > n_ref;
        if (need_mask) {
#pragma unroll
          for (int e = 0; e < BH; ++e)
            v[e] = (j0 + e == selfc || j0 + e >= n_ref) ? CUDART_INF_F : v[e];
        }
        if constexpr (SMP > 0) {
          // branch-free insertion of the part's group minima (new_i = min(r_i, max(r_i-1, x)))
#pragma unroll
          for (int g = 0; g < BH / 8; ++g) {
            const float x = min8(v + 8 * g);
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
              const int64_t jj = j0 + 8 * gg + e;
              if (jj == selfc || jj >= n_ref) c8[e] = CUDART_INF_F;
            }
          }
        };
        filter_part<BH, COL>(v, tau, (scol0 + j0) >> 3, pa, pbase, vote != 0, flush, reload,
                             release);  // col0 % 256 == 0
        if (tr) trace[(etr - 1) * 16 + 6] = clock64();
      }
      if constexpr (SMP > 0) {
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
  cluster_sync();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc2(tmem_base, 512);
  }
}

template <int DPAD, int FMT, int DBG, int FW, bool COL, int NB, int NACC, int SMP = 0>
cudaError_t launch4(const Image& A, const Image& B, int64_t q_begin, int64_t q_count,
                    bool self_join, const MainPass& m, int num_sms, cudaStream_t st) {
  const int nstage = pick_stages4<DPAD, FW, NB>();
  if (nstage < 3) return cudaErrorInvalidValue;
  if (m.parts != FW / 4) return cudaErrorInvalidValue;
  int a, b, c;
  const int smem = smem4<DPAD, FW, NB>(nstage, &a, &b, &c);
  auto kern = k_knn_tc4<DPAD, FMT, DBG, FW, COL, NB, NACC, SMP>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  if (e != cudaSuccess) return e;
  const int64_t qt0 = q_begin / kBM;
  const int64_t qt1 = (q_begin + q_count + kBM - 1) / kBM;
  const int64_t n_qpairs = (qt1 - qt0 + 1) / 2;
  const int64_t n_items = n_qpairs * m.S;
  const int64_t pairs = std::min<int64_t>(num_sms / 2, n_items);
  if (pairs <= 0) return cudaSuccess;
  kern<<<(unsigned)(2 * pairs), 64 + 32 * FW, smem, st>>>(
      reinterpret_cast<const uint8_t*>(A.data), A.region_bytes(), A.extra_offset(),
      reinterpret_cast<const uint8_t*>(B.data), B.region_bytes(), B.extra_offset(),
      (B.n + NB - 1) / NB, B.n, qt0, n_qpairs, q_begin, q_begin + q_count, self_join ? 1 : 0, m.S,
      m.R, nstage, m.tau_v, m.tau_lists, m.buf, m.cnt, m.cap, m.col0, m.vote, m.smode, m.trace,
      m.samp);
  return cudaGetLastError();
}

}  // namespace

// Measured on B200 (C2 d=32 / C3 d=64 shapes): the pair wins where the MMA is
// long enough to cover the cross-SM release latency of the accumulators (d=64:
// pass 1 130 vs 136 ms); at d <= 32 the single-SM kernel is faster (1.05 vs
// 1.18 ms), so the pair is the default for dpad >= 64.
int tc4_fits(int dpad, int parts) {
  if (parts != 4) return 0;
  switch (dpad) {
    case 16: return pick_stages4<16, 16, 256>() >= 3 && pick_stages4<16, 16, 160>() >= 3;
    case 32: return pick_stages4<32, 16, 256>() >= 3 && pick_stages4<32, 16, 160>() >= 3;
    case 64: return pick_stages4<64, 16, 256>() >= 3 && pick_stages4<64, 16, 160>() >= 3;
    case 128: return pick_stages4<128, 16, 256>() >= 3;  // K-pipelined (256-column tiles only)
    case 256: return pick_stages4<256, 16, 256>() >= 3;
    case 512: return pick_stages4<512, 16, 256>() >= 3;
  }
  return 0;
}
// dpad > 64 (K-pipelined, measured at the C5 shape n = 5e5, d = 512, k = 50):
// main kernel 236.8 -> 181.8 ms against the single-SM K-pipelined pass (the
// per-SM operand stream per K region falls from 48 to 32 KB); d = 128 / 256 at
// n = 2e5: 9.8 -> 7.5 / 17.2 -> 13.0 ms.
int tc4_preferred(int dpad) { return dpad >= 64; }

// MainPass.nb = 160: the three-accumulator ring (160-column tiles); else 256.
template <int D, int FMT, int DBG, bool COL>
cudaError_t launch4_nb(const Image& A, const Image& B, int64_t q_begin, int64_t q_count,
                       bool self_join, const MainPass& m, int num_sms, cudaStream_t st) {
  if constexpr (D > 64 && DBG == 0 && !COL) {
    if (m.samp) {  // key-only sample pass (smode 1), K-pipelined pairs
      if (m.samp_acc || m.smode != 1) return cudaErrorInvalidValue;
      return m.samp_t == 8
                 ? launch4<D, FMT, 0, 16, false, 256, 2, 8>(A, B, q_begin, q_count, self_join, m, num_sms, st)
                 : launch4<D, FMT, 0, 16, false, 256, 2, 4>(A, B, q_begin, q_count, self_join, m, num_sms, st);
    }
  }
  if (m.samp) return cudaErrorInvalidValue;
  if constexpr (D <= 64) {
    if (m.nb == 160) return launch4<D, FMT, DBG, 16, COL, 160, 3>(A, B, q_begin, q_count, self_join, m, num_sms, st);
  }
  return launch4<D, FMT, DBG, 16, COL, 256, 2>(A, B, q_begin, q_count, self_join, m, num_sms, st);
}

cudaError_t launch_knn_tc4(const Image& A, const Image& B, int64_t q_begin, int64_t q_count,
                           bool self_join, int fmt, const MainPass& m, int num_sms, int dbg,
                           cudaStream_t st, int* launches) {
  *launches += 1;
#define TOD_TC4_CASE(D)                                                                          \
  case D:                                                                                       \
    if (dbg & 4)                                                                                \
      return fmt == 1 ? launch4_nb<D, 1, 4, false>(A, B, q_begin, q_count, self_join, m, num_sms, st) \
                      : launch4_nb<D, 2, 4, false>(A, B, q_begin, q_count, self_join, m, num_sms, st); \
    if (dbg & 3)                                                                                \
      return fmt == 1 ? launch4_nb<D, 1, 2, false>(A, B, q_begin, q_count, self_join, m, num_sms, st) \
                      : launch4_nb<D, 2, 2, false>(A, B, q_begin, q_count, self_join, m, num_sms, st); \
    if (dbg & 8)  /* profiling trace build */                                                   \
      return fmt == 1 ? launch4_nb<D, 1, 8, false>(A, B, q_begin, q_count, self_join, m, num_sms, st) \
                      : launch4_nb<D, 2, 8, false>(A, B, q_begin, q_count, self_join, m, num_sms, st); \
    if (m.colmode)                                                                              \
      return fmt == 1 ? launch4_nb<D, 1, 0, true>(A, B, q_begin, q_count, self_join, m, num_sms, st) \
                      : launch4_nb<D, 2, 0, true>(A, B, q_begin, q_count, self_join, m, num_sms, st); \
    return fmt == 1 ? launch4_nb<D, 1, 0, false>(A, B, q_begin, q_count, self_join, m, num_sms, st)   \
                    : launch4_nb<D, 2, 0, false>(A, B, q_begin, q_count, self_join, m, num_sms, st);
  switch (A.dpad) {
    TOD_TC4_CASE(16)
    TOD_TC4_CASE(32)
    TOD_TC4_CASE(64)
    TOD_TC4_CASE(128)
    TOD_TC4_CASE(256)
    TOD_TC4_CASE(512)
  }
#undef TOD_TC4_CASE
  return cudaErrorInvalidValue;
}

}  // namespace tod
