// api.cu — the C ABI of include/tod.h: argument validation, planning
// (format, K', chunking), workspace management, host<->device staging, and
// the launch sequence of the hot path:
//   prep (K1) -> fused distance + top-K' (K2 tcgen05 | K2s SIMT) ->
//   fp64 re-rank + certificate (K3) -> fp64 brute-force fallback (K4) ->
//   [LOF stage (K5)].
// Every step runs in this library's CUDA kernels; there is no CPU path.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

#include "../../include/tod.h"
#include "ctx.h"
#include "internal.h"

#ifndef TOD_BUILD_INFO
#define TOD_BUILD_INFO "libtod sm_100a"
#endif

using namespace tod;
using namespace todapi;


namespace todapi {

tod_status fail(tod_ctx* ctx, tod_status s, const char* fmt, ...) {
  if (ctx) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    ctx->msg = buf;
  }
  return s;
}


tod_status ensure_ws(tod_ctx* ctx, Workspace& ws, int id, size_t bytes, void** out) {
  Buf& b = ws.bufs[id];
  if (bytes == 0) bytes = 16;
  if (b.bytes < bytes) {
    if (b.p) cudaFree(b.p);
    b = Buf{};
    cudaError_t e = cudaMalloc(&b.p, bytes);
    if (e != cudaSuccess) {
      cudaGetLastError();
      return fail(ctx, TOD_E_NOMEM, "cudaMalloc(%zu) failed: %s", bytes, cudaGetErrorString(e));
    }
    b.bytes = bytes;
  }
  *out = b.p;
  return TOD_OK;
}


// Is p device memory of this context's device?  Host (pageable/pinned) -> false.
bool is_device_ptr(const void* p, int device) {
  if (!p) return false;
  cudaPointerAttributes a;
  cudaError_t e = cudaPointerGetAttributes(&a, p);
  if (e != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) && a.device == device;
}

tod_status make_plan(tod_ctx* ctx, int64_t n_ref, int64_t q_count, int d, int k, Plan* p) {
  int fmt = ctx->cfg.format;
  if (fmt < 0 || fmt > 3) return fail(ctx, TOD_E_ARG, "bad format %d", fmt);
  if (fmt == TOD_FMT_AUTO) fmt = d < 16 ? TOD_FMT_FP32 : TOD_FMT_FP16;
  p->fmt = fmt;
  p->kind = fmt == TOD_FMT_FP32 ? PASS_SIMT : PASS_TC;
  if (p->kind == PASS_TC) {
    if (d > 512)
      return fail(ctx, TOD_E_UNSUPPORTED, "tensor-core pass supports d <= 512 in this build (d=%d)", d);
    p->dpad = d <= 16 ? 16 : d <= 32 ? 32 : d <= 64 ? 64 : d <= 128 ? 128 : d <= 256 ? 256 : 512;
  } else {
    if (d > 64) return fail(ctx, TOD_E_UNSUPPORTED, "fp32 SIMT pass supports d <= 64 (d=%d)", d);
    p->dpad = d;
  }
  int kp = ctx->cfg.kprime;
  const int kmax_list = p->kind == PASS_TC ? 64 : 128;
  int kp_policy = kp;  // uncapped (the two-pass main pass has no list capacity)
  if (kp <= 0) {
    // fp16: k + 24 (C2: 99.999 % certified); wide rows carry more quantization
    // error per key, so more candidates (measured at d = 512, k = 50: K' 80 -> 96
    // cuts the uncertified rows 134 -> 5 of 2e5 and the fallback 6.7 -> 0.4 ms)
    if (fmt == TOD_FMT_FP16) kp = d > 128 ? roundup(3 * k / 2 + 16, 8) : roundup(k + 24, 8);
    else if (fmt == TOD_FMT_BF16) kp = roundup(std::max(6 * k, k + 40), 16);
    else kp = roundup(std::max(k + 8, 16), 8);
    kp_policy = kp;
    kp = std::min(kp, kmax_list);
  }
  if (kp < k) kp = k;  // never fewer candidates than outputs
  if (kp_policy < kp) kp_policy = kp;
  // an explicit K' above the list capacity is only honoured by the two-pass
  // selection (its main pass has no list): checked once the pass is chosen
  const int kp_req = kp;
  if (kp > kmax_list) kp = kmax_list;
  p->kp = kp;
  int S = ctx->cfg.chunks;
  p->two = 0;
  p->R = 1;
  p->main_S = 0;
  p->cap = 0;
  const int64_t bt256 = (n_ref + 255) / 256;
  int64_t bt_v1 = 0;  // reference tiles seen by the v1 kernel (the sample pass: every R-th)
  if (p->kind == PASS_TC && !(ctx->cfg.flags & TOD_F_PASS1_V1) && tc3_fits(p->dpad) &&
      (bt256 >= 32 || p->dpad > 128)) {
    // Two-pass candidate selection: the sample pass keeps kps
    // groups per row over every R-th tile; its threshold filters the main pass,
    // which appends ~R*kps groups per row.  K' is the target count of kept
    // groups; kps = 2K'/R leaves a wide margin for the sample's variance.
    p->two = 1;
    p->kp_target = std::max(kp, kp_policy);
    p->R = 8;
    if (const char* e = getenv("TOD_SAMPLE_R")) {  // experiment knob (power of two >= 2)
      const int v = atoi(e);
      if (v >= 2 && v <= 64 && (v & (v - 1)) == 0) p->R = v;
    }
    const int kps = std::min(64, std::max(8, roundup((2 * p->kp_target + p->R - 1) / p->R, 4)));
    const double img_bytes = (double)bt256 * 256 * (p->dpad + 16) * 2;
    double chunk_mb = 48.0;  // reference chunk of the main pass (L2 locality)
    if (const char* e = getenv("TOD_MAIN_CHUNK_MB")) chunk_mb = std::max(4.0, atof(e));  // experiment knob
    p->main_S = std::max(1, (int)std::ceil(img_bytes / (chunk_mb * 1024 * 1024)));
    {
      // few query tiles (a second tier, small query calls): split the references
      // so the (query tile x chunk) items still cover every SM
      const int64_t units = (q_count + 255) / 256 + 1;  // CTA-pair tile pairs (or ~half the tiles)
      const int64_t want = (ctx->num_sms + units - 1) / units;
      if (want > p->main_S) p->main_S = (int)std::min<int64_t>(want, std::max<int64_t>(1, bt256 / 4));
    }
    {
      // fill the last wave of the persistent grid: items = query tiles x S are
      // dealt round-robin, so the makespan is ceil(items / grid) items of bt/S
      // tiles; take the S in [S, S + 7] (>= 4 tiles per item) minimising
      // ceil(Q S / G) / S.  C2 (782 query tiles on 148 SMs, last wave 42/148 at
      // S = 1): S = 7, main kernel 1.180 -> 1.025 ms (tools/r02_s7.sh).
      const int64_t Q = (q_count + 127) / 128, G = std::max(1, ctx->num_sms);
      const int s0 = p->main_S;
      double best = 1e300;
      for (int s = s0; s <= s0 + 7 && (s == s0 || s <= bt256 / 4); ++s) {
        const double v = (double)((Q * s + G - 1) / G) / s;
        if (v < best - 1e-9) {
          best = v;
          p->main_S = s;
        }
      }
    }
    if (const char* e = getenv("TOD_MAIN_S")) p->main_S = std::max(1, atoi(e));  // experiment knob
    p->cap = roundup(std::max(64, 2 * (p->R - 1) * kps), 32);
    bt_v1 = (bt256 + p->R - 1) / p->R;
  }
  if (p->kind == PASS_TC && !p->two && p->dpad > 128)
    return fail(ctx, TOD_E_UNSUPPORTED, "d=%d needs the two-pass tensor-core path", d);
  if (!p->two && kp_req > kmax_list)
    return fail(ctx, TOD_E_UNSUPPORTED, "K'=%d exceeds this pass's list capacity %d (k=%d)",
                kp_req, kmax_list, k);
  if (p->kind == PASS_TC && !p->two && p->dpad <= 64) bt_v1 = bt256;
  if (p->kind == PASS_TC) {
    // Reference chunks: each chunk's operand image should stay L2-resident
    // while all CTAs sweep it (chunk-major work order), and the (query tile x
    // chunk) items should fill the last wave of the persistent grid.
    // Epilogue split: 1, 2 or 4 warps per TMEM lane quarter, each with its own
    // per-row list over its part of every tile (K'' = K' for 1 part,
    // K'/2 + 8 for 2, K'/4 + 4 for 4; the re-rank takes the union).
    // Two-pass: the sample pass keeps ~2K'/R groups per row in total, split over
    // the lists (its threshold is the minimum of the lists' thresholds).
    auto khalf = [&](int sp) {
      if (p->two) {
        // per-list size from the reference stride 8 (TOD_SAMPLE_KR overrides, experiment knob)
        int kr = 8;
        if (const char* e = getenv("TOD_SAMPLE_KR")) kr = std::max(1, atoi(e));
        return std::max(4, roundup((2 * kp + kr * sp - 1) / (kr * sp), 4));
      }
      return sp == 1 ? kp : (sp == 2 ? roundup(kp / 2 + 8, 4) : roundup(kp / 4 + 4, 4));
    };
    int sp = ctx->cfg.epilogue_split;
    if (p->two && sp == 4) sp = 2;  // measured: 4 lists of K''=4 certify < 98 %
    if (sp != 1 && sp != 2 && sp != 4) {
      sp = 1;
      for (int cand : {4, 2}) {
        if (p->two && cand == 4) continue;
        if (tc_split_fits(p->dpad, khalf(cand), cand)) {
          sp = cand;
          break;
        }
      }
    }
    if (sp != 1 && !tc_split_fits(p->dpad, khalf(sp), sp)) sp = 1;
    p->lists = sp;
    p->kp = khalf(sp);
    const int64_t qtiles = (q_count + 127) / 128 + 1;
    const int64_t btiles = bt_v1 > 0 ? bt_v1 : (n_ref + 255) / 256;
    const double img_bytes = (double)btiles * 256 * (p->dpad + 16) * 2;
    const int s_min = std::max(1, (int)std::ceil(img_bytes / (48.0 * 1024 * 1024)));
    if (S <= 0) {
      double best = 1e30;
      S = s_min;
      for (int s = s_min; s <= s_min + 8; ++s) {
        if (btiles / s < 8) break;
        const double items = (double)(qtiles * s);
        const double waves = std::ceil(items / ctx->num_sms);
        const double cost = waves / items * (1.0 + 0.003 * (s - s_min));
        if (cost < best - 1e-12) {
          best = cost;
          S = s;
        }
      }
    }
    if (S < 1 || S > btiles) return fail(ctx, TOD_E_ARG, "bad chunk count S=%d", S);
  } else {
    p->lists = 0;  // set below
    if (S <= 0) {
      const int64_t qtiles = (q_count + 127) / 128;
      S = 1;
      while (qtiles * S < 2 * ctx->num_sms && (S + 1) * kp <= 256 && n_ref / (S + 1) >= 256) ++S;
    }
    if (S < 1 || S * kp > 256) return fail(ctx, TOD_E_ARG, "bad chunk count S=%d (K'=%d)", S, kp);
    p->lists = S;
  }
  p->S = S;
  return TOD_OK;
}




// Main-pass filter: test each part's minimum with a warp vote first when appends
// are rare.  A row appends ~2K' groups over 4 n/256 (row, part) cells; below
// n ~ 3e5 most warps hold a candidate in most parts and the vote only adds work
// (measured: C2 main kernel 1.13 -> 1.21 ms with the vote, C3 no slower).
// TOD_VOTE (experiment knob) forces it on (1) or off (0).
int main_vote(int64_t n_ref) {
  if (const char* e = getenv("TOD_VOTE")) return atoi(e) != 0;
  return n_ref >= 300000;
}
// The single-SM main pass with a three-deep accumulator ring (knn_tc5.cu):
// opt-in only (TOD_MAIN_RING3=1, experiment knob; dpad <= 64, main pass over
// every tile, no profiling mode) -- measured slower than knn_tc3 at C2
// (1.41 vs 1.08 ms main kernel, profiles/r02).
int main_ring3(int dpad, const MainPass& mp, int dbg) {
  if (mp.R != 0 || mp.parts != 4 || (dbg & 7) != 0 || !tc5_fits(dpad)) return 0;
  if (const char* e = getenv("TOD_MAIN_RING3")) return atoi(e) != 0;
  return 0;
}

// Column candidates (filter.cuh COL): with rare appends (the vote), the main
// pass appends each column below tau of a passing group, and the re-rank
// evaluates only those columns instead of all 8 columns of every visited group
// (a list-based sample's candidates stay groups: the re-rank takes both).  The
// filter then holds the accumulator until its vote (it re-reads passing groups'
// columns from TMEM), which costs a two-deep ring: default only where the tile's
// MMA is long (dpad > 64; C5: re-rank 198 -> 71 ms at n = 5e5), not at d = 64
// (C3: re-rank -10 ms, main pass +61 ms).  TOD_COLMODE (experiment knob) 1 / 0.
int main_colmode(const MainPass& mp, int dpad) {
  if (const char* e = getenv("TOD_COLMODE")) return atoi(e) != 0;
  return mp.vote && dpad > 64;
}

// CTA-pair main pass tile geometry: 160-column tiles with three accumulators
// when no list-based sample tiles (256-column grid) must be skipped;
// TOD_MAIN_NB (experiment knob) 160 / 256.
int main_nb(const MainPass& mp) {
  int nb = 256;
  if (const char* e = getenv("TOD_MAIN_NB")) nb = atoi(e) == 160 ? 160 : 256;
  return mp.R != 0 ? 256 : nb;  // sample tiles are skipped on the 256-column grid
}


// Input quantization (a1) for the tensor-core passes: column mean, power-of-two
// scale, reference image B over all n rows (skipped when ref->ready) and query
// image A over the 128-row query tiles covering [q_begin, q_begin+q_count)
// (self-join) or over Q.
tod_status prep_tc(tod_ctx* ctx, const float* dX, int64_t n, const float* dQ, int64_t q_begin,
                   int64_t q_count, int d, int fmt, int dpad, PrepGlobals* g, Image* Aout,
                   Image* Bout, CertParams* cp, RefPrep* ref, int* launches) {
  cudaStream_t st = ctx->stream;
  const bool self = dQ == nullptr;
  void* p;
  const int64_t n_pad = (n + 255) / 256 * 256;
  // query image rows: the 128-row query tiles covering [q_begin, q_begin+q_count)
  const int64_t a_row0 = self ? (q_begin / 128) * 128 : 0;
  const int64_t a_rows = self ? std::min<int64_t>(n, (q_begin + q_count + 127) / 128 * 128) - a_row0
                              : q_count;
  const int64_t a_pad = (a_rows + 255) / 256 * 256;
  const int rb = std::min(128, dpad * 2);
  auto make_img = [&](int id_img, int id_a2, int id_e, int64_t rows, int64_t rows_pad,
                      Image* img) -> tod_status {
    void* q;
    img->n = rows;
    img->n_pad = rows_pad;
    img->dpad = dpad;
    img->rb = rb;
    img->nkb = dpad * 2 / rb;
    img->layout = rb == 128 ? 2 : (rb == 64 ? 4 : 6);
    TOD_TRY(ensure(ctx, id_img, img->total_bytes(), &q));
    img->data = static_cast<uint16_t*>(q);
    TOD_TRY(ensure(ctx, id_a2, (size_t)std::max<int64_t>(rows, 1) * 8, &q));
    img->a2 = static_cast<double*>(q);
    TOD_TRY(ensure(ctx, id_e, (size_t)std::max<int64_t>(rows, 1) * 8, &q));
    img->e = static_cast<double*>(q);
    return TOD_OK;
  };
  Image& B = *Bout;
  Image& A = *Aout;
  TOD_TRY(make_img(B_IMG_B, B_A2_B, B_E_B, n, n_pad, &B));
  TOD_TRY(make_img(B_IMG_A, B_A2_A, B_E_A, a_rows, a_pad, &A));
  TOD_TRY(ensure(ctx, B_MU, (size_t)d * 8, &p));
  double* mu = static_cast<double*>(p);
  if (!ref->ready) {
    const int stat_blocks = (int)((n + 127) / 128);  // prep.cu kRowsPerStatBlock
    TOD_TRY(ensure(ctx, B_PART, (size_t)stat_blocks * d * 8, &p));
    double* part = static_cast<double*>(p);
    TOD_CUDA(launch_prep_stats(dX, n, d, mu, part, stat_blocks, g, st, launches));
    TOD_CUDA(launch_prep_absmax(dX, n, d, mu, g, st, launches));
    if (!self) {
      const float* qa = ref->dQall ? ref->dQall : dQ;
      const int64_t nqa = ref->dQall ? ref->nq_all : q_count;
      TOD_CUDA(launch_finite_check(qa, nqa, d, g, st, launches));
      TOD_CUDA(launch_prep_absmax(qa, nqa, d, mu, g, st, launches));
    }
    TOD_CUDA(launch_prep_scale(g, fmt, dpad, st, launches));
    TOD_CUDA(launch_prep_quant(dX, n, d, mu, g, fmt, B, 0, st, launches));
    TOD_TRY(ensure(ctx, B_EG, (size_t)std::max<int64_t>((n + 7) / 8, 1) * 8, &p));
    TOD_CUDA(launch_group_emax(B.e, n, static_cast<double*>(p), st, launches));
    ref->ready = true;
  }
  TOD_TRY(ensure(ctx, B_EG, (size_t)std::max<int64_t>((n + 7) / 8, 1) * 8, &p));
  // Per-group residual bounds in the re-rank's UB and visit cut pay where the
  // quantization residuals are large (bf16: C3 re-rank 28.7 -> 18.8 ms); with
  // fp16's 8x smaller residuals they visit barely fewer groups and the per-
  // candidate bound evaluation costs more than it saves (C2: 0.62 -> 0.75 ms).
  // TOD_GROUP_EMAX (experiment knob) 1 / 0 forces them on / off.
  bool use_eg = fmt == 2;
  if (const char* e = getenv("TOD_GROUP_EMAX")) use_eg = atoi(e) != 0;
  cp->eg = use_eg ? static_cast<const double*>(p) : nullptr;
  cp->ecol = B.e;
  // per-column pre-bound of the re-rank from the operand image (self-join):
  // opt-in (TOD_RR_PREBOUND=1, experiment knob) -- it excludes 88-89 % of the
  // visited groups' columns before their fp32 rows are gathered (C2: 169 of 192
  // per row, C3: 267 of 299) but the extra dependent image read lengthens the
  // latency-bound per-row chain: C2 re-rank 0.71 -> 1.00 ms, C3 20.9 -> 28.2 ms.
  bool prebound = false;
  if (const char* e = getenv("TOD_RR_PREBOUND")) prebound = self && atoi(e) != 0;
  cp->bimg = prebound ? reinterpret_cast<const uint8_t*>(B.data) : nullptr;
  cp->b_region = B.region_bytes();
  cp->b_rb = B.rb;
  cp->fmt = fmt;
  const float* qsrc = self ? dX + a_row0 * d : dQ;
  TOD_CUDA(launch_prep_quant(qsrc, a_rows, d, mu, g, fmt, A, 1, st, launches));
  cp->qa2 = A.a2 + (self ? q_begin - a_row0 : 0);
  cp->qe = A.e + (self ? q_begin - a_row0 : 0);
  return TOD_OK;
}

// Core: all pointers device.  Q == nullptr => self-join over X, rows
// [q_begin, q_begin+q_count).  Else queries Q[0..q_count) against X.
tod_status run_knn(tod_ctx* ctx, const float* dX, int64_t n, const float* dQ, int64_t q_begin,
                   int64_t q_count, int d, int k, KnnOutDev out, tod_stats* stats, Timer& tm,
                   int* launches, RefPrep* ref) {
  const bool self = dQ == nullptr;
  bool main_timed = false;
  int main_kernel = 0;
  int sample_pass = 0;
  Plan plan;
  TOD_TRY(make_plan(ctx, n, q_count, d, k, &plan));
  cudaStream_t st = ctx->stream;

  void* p;
  TOD_TRY(ensure(ctx, B_SMALL, sizeof(SmallDev), &p));
  SmallDev* small = static_cast<SmallDev*>(p);
  if (plan.kind == PASS_TC && ref->ready) {  // keep the reference-side globals
    const size_t off = offsetof(SmallDev, fail_count);
    TOD_CUDA(cudaMemsetAsync(reinterpret_cast<char*>(small) + off, 0, sizeof(SmallDev) - off, st));
  } else {
    TOD_CUDA(cudaMemsetAsync(small, 0, sizeof(SmallDev), st));
  }
  PrepGlobals* g = &small->g;

  Cands cands;
  MainPass mp;
  cands.kp = plan.kp;
  cands.S = plan.S;
  cands.lists = plan.lists;
  cands.R = plan.R;
  cands.dbg = (int)((ctx->cfg.flags >> 8) & 0xFF);
  if (cands.dbg & 8) {
    TOD_TRY(ensure(ctx, B_TRACE, 4096 * 8 * sizeof(long long), &p));
    cands.trace = static_cast<long long*>(p);
    TOD_CUDA(cudaMemsetAsync(p, 0, 4096 * 8 * sizeof(long long), st));
  }
  TOD_TRY(ensure(ctx, B_CIDX, (size_t)std::max<int64_t>(q_count, 1) * cands.lists * plan.kp * 4, &p));
  cands.idx = static_cast<int32_t*>(p);
  TOD_TRY(ensure(ctx, B_CV, (size_t)std::max<int64_t>(q_count, 1) * cands.lists * 4, &p));
  cands.v = static_cast<float*>(p);
  if (plan.kind == PASS_TC) {
    TOD_TRY(ensure(ctx, B_CKEY, (size_t)std::max<int64_t>(q_count, 1) * cands.lists * plan.kp * 4, &p));
    cands.key = static_cast<float*>(p);
  }
  if (plan.kind == PASS_TC && plan.S > 1) {
    const int64_t nqt = (q_begin + q_count + 127) / 128 - q_begin / 128;
    TOD_TRY(ensure(ctx, B_STLIST, (size_t)nqt * plan.lists * plan.kp * 128 * 8, &p));
    cands.st_list = static_cast<uint2*>(p);
    TOD_TRY(ensure(ctx, B_STDONE, (size_t)nqt * 4, &p));   // >= query groups
    cands.st_done = static_cast<int*>(p);
    TOD_CUDA(cudaMemsetAsync(cands.st_done, 0, (size_t)nqt * 4, st));
  }
  CertParams cp{};
  cp.kind = plan.kind;
  cp.d = d;
  cp.dpad = plan.dpad;
  cp.s = 1.0;
  cp.g = g;
  cp.force_fail = (ctx->cfg.flags & TOD_F_NO_CERTIFY) ? 1 : 0;

  tm.mark();  // 1: prep start
  if (plan.kind == PASS_TC) {
    Image B, A;
    TOD_TRY(prep_tc(ctx, dX, n, dQ, q_begin, q_count, d, plan.fmt, plan.dpad, g, &A, &B, &cp,
                    ref, launches));
    tm.mark();  // 2: main start
    // Candidate selection (DESIGN.md §5 "Two-pass" and "Three-stage"):
    //  * key-only sample (d <= 32, d >= 128): knn_tc3 sample mode keeps the 4 (or 8)
    //    smallest group minima per (row, part) over every R-th tile; tau = the j-th
    //    smallest of those; the main pass covers every tile.
    //  * three-stage (d = 64 on CTA pairs): a key-only pre-sample over every
    //    (8R)-th tile gives an over-estimate tau0; the main-pass kernel sweeps the
    //    sample tiles (t % R == 0) appending everything below tau0; tau = the j-th
    //    smallest of those appends (<= tau0); the main pass sweeps the other tiles
    //    below tau.  Every non-kept candidate is >= tau either way.
    //  * list-based sample (TOD_SAMPLE3=0 at d = 64; TOD_SAMPLE_V1=1): knn_tc.cu's
    //    running top-K'' lists over the sample tiles, the main pass skips them.
    const char* pe = getenv("TOD_MAIN_PAIR");  // experiment knob: 1 = force pairs, 0 = never
    const bool pair = pe ? atoi(pe) != 0 : tc4_preferred(plan.dpad) != 0;
    const bool use4 = plan.two && pair && !(ctx->cfg.flags & TOD_F_MAIN_1SM) &&
                      tc4_fits(plan.dpad, tc3_parts(plan.dpad));
    const char* sv = getenv("TOD_SAMPLE_V1");
    const char* s3 = getenv("TOD_SAMPLE3");
    // three-stage: d = 64 on CTA pairs; d <= 32 on the single-SM kernel from
    // n = 3e5 (measured n = 1e6, d = 32: pass 1 103.0 -> 93.3 ms; at C2, n = 1e5,
    // neutral: 1.355 vs 1.359 ms)
    // dpad > 64 (K-pipelined pairs) also from n = 3e5 (C5 shape n = 5e5: pass 1
    // 204 -> 187 ms; at n = 2000 the 1/64 pre-sample is too sparse: 71 % certified)
    const bool three = plan.two && (cands.dbg & 7) == 0 && !sv &&
                       ((use4 && (s3 ? atoi(s3) != 0
                                     : (plan.dpad == 64 || (plan.dpad > 64 && n >= 300000)))) ||
                        (!use4 && plan.dpad <= 32 && tc3_parts(plan.dpad) == 4 &&
                         (s3 ? atoi(s3) != 0 : n >= 300000)));
    const bool samp_v1 = plan.two && !three && plan.dpad <= 128 &&
                         (sv ? atoi(sv) != 0 : plan.dpad == 64);
    if (plan.two) sample_pass = samp_v1 ? 1 : (three ? 3 : 2);
    // tau = the j-th smallest sample key, j ~ 2K'/R
    const int jw = std::max(4, (2 * plan.kp_target + plan.R - 1) / plan.R);
    if (plan.two && !samp_v1) {
      MainPass sm;
      sm.S = 1;
      sm.R = three ? 8 * plan.R : plan.R;
      sm.parts = tc3_parts(plan.dpad);
      // 8 minima per (row, part) when 4 per part cannot supply j (large k); the
      // three-stage pre-sample takes the 8th of 16 (an over-estimate of the
      // stage-2 tau: the (8 x 8R)-th group over all tiles in expectation)
      const int ja = three ? 8 : jw;
      sm.samp_t = ja > 3 * sm.parts ? 8 : 4;
      const int nv = sm.parts * sm.samp_t;
      TOD_TRY(ensure(ctx, B_SAMP, (size_t)std::max<int64_t>(q_count, 1) * nv * 4, &p));
      sm.samp = static_cast<float*>(p);
      sm.tau_lists = 0;  // no thresholds in the sample pass
      // dpad > 64 on CTA pairs: the K-pipelined pair kernel's key-only sample mode
      // sweeps the same sample tiles (smode 1); else knn_tc3's sample mode
      const char* sp = getenv("TOD_SAMPLE_PAIR");  // experiment knob 1 / 0
      const bool samp4 = use4 && plan.dpad > 64 && (cands.dbg & 7) == 0 &&
                         (sp ? atoi(sp) != 0 : true);
      if (samp4) {
        sm.smode = 1;
        sm.nb = 256;
        TOD_CUDA(launch_knn_tc4(A, B, self ? q_begin : 0, q_count, self, plan.fmt, sm,
                                ctx->num_sms, 0, st, launches));
      } else {
        TOD_CUDA(launch_knn_tc3(A, B, self ? q_begin : 0, q_count, self, plan.fmt, sm,
                                ctx->num_sms, 0, st, launches));
      }
      TOD_CUDA(launch_tau_combine(q_count, nv, std::min(nv, ja), sm.samp, cands.v, st, launches));
      cands.lists = 1;
      cands.kp = 0;
    } else {
      TOD_CUDA(launch_knn_tc(A, B, self ? q_begin : 0, q_count, self, plan.fmt, cands,
                             ctx->num_sms, st, launches));
    }
    if (plan.two) {
      mp.S = plan.main_S;
      mp.R = (samp_v1 || three) ? plan.R : 0;
      mp.tau_v = cands.v;
      mp.tau_lists = cands.lists;
      mp.parts = tc3_parts(plan.dpad);
      mp.cap = plan.cap * 2 / mp.parts;  // plan.cap is per column half
      mp.vote = main_vote(n);
      mp.trace = cands.trace;
      mp.smode = three ? 1 : 0;
      mp.colmode = cands.dbg ? 0 : main_colmode(mp, plan.dpad);  // profiling builds: groups
      mp.nb = main_nb(mp);
      TOD_TRY(ensure(ctx, B_MBUF, (size_t)std::max<int64_t>(q_count, 1) * mp.parts * mp.cap * 8, &p));
      mp.buf = static_cast<uint2*>(p);
      TOD_TRY(ensure(ctx, B_MCNT, (size_t)std::max<int64_t>(q_count, 1) * mp.parts * 4, &p));
      mp.cnt = static_cast<int*>(p);
      TOD_CUDA(cudaMemsetAsync(mp.cnt, 0, (size_t)std::max<int64_t>(q_count, 1) * mp.parts * 4, st));
      if (three) {
        // stage 2: the sample tiles below tau0, appended; tau = their j-th smallest key
        MainPass mb = mp;
        mb.trace = nullptr;  // the profiling trace records the main sweep (stage 4)
        if (use4)
          TOD_CUDA(launch_knn_tc4(A, B, self ? q_begin : 0, q_count, self, plan.fmt, mb,
                                  ctx->num_sms, 0, st, launches));
        else
          TOD_CUDA(launch_knn_tc3(A, B, self ? q_begin : 0, q_count, self, plan.fmt, mb,
                                  ctx->num_sms, 0, st, launches));
        TOD_CUDA(launch_tau_from_appends(q_count, mp.parts, mp.cap, mp.cnt, mp.buf, jw, cands.v,
                                         st, launches));
        mp.smode = 0;
      }
      if (tm.on) cudaEventRecord(ctx->evk[0], st);
      main_timed = tm.on;
      const bool use5 = !use4 && main_ring3(plan.dpad, mp, cands.dbg);
      if (use4)
        TOD_CUDA(launch_knn_tc4(A, B, self ? q_begin : 0, q_count, self, plan.fmt, mp,
                                ctx->num_sms, cands.dbg, st, launches));
      else if (use5)
        TOD_CUDA(launch_knn_tc5(A, B, self ? q_begin : 0, q_count, self, plan.fmt, mp,
                                ctx->num_sms, st, launches));
      else
        TOD_CUDA(launch_knn_tc3(A, B, self ? q_begin : 0, q_count, self, plan.fmt, mp,
                                ctx->num_sms, cands.dbg, st, launches));
      main_kernel = use4 ? 4 : (use5 ? 5 : 3);
      if (tm.on) cudaEventRecord(ctx->evk[1], st);
    }
  } else {
    TOD_CUDA(launch_finite_check(dX, n, d, g, st, launches));
    if (!self) TOD_CUDA(launch_finite_check(dQ, q_count, d, g, st, launches));
    tm.mark();  // 2
    TOD_CUDA(launch_knn_simt(dQ, q_begin, q_count, dX, n, d, self, cands, st, launches));
  }
  tm.mark();  // 3: certify start
  if (cands.trace) {  // profiling aid: dump CTA 0's per-tile timestamps
    static long long host_trace[4096 * 8];
    TOD_CUDA(cudaMemcpyAsync(host_trace, cands.trace, sizeof host_trace, cudaMemcpyDeviceToHost, st));
    TOD_CUDA(cudaStreamSynchronize(st));
    const char* path = getenv("TOD_TRACE_FILE");
    if (path) {
      FILE* f = fopen(path, "wb");
      if (f) {
        fwrite(host_trace, sizeof host_trace, 1, f);
        fclose(f);
      }
    }
  }
  if (cands.dbg & ~8) {  // profiling aid: pass 1 only, outputs invalid
    TOD_CUDA(cudaStreamSynchronize(st));
    tm.mark();
    tm.mark();
    if (stats) {
      stats->rows = q_count;
      stats->kprime = plan.kp;
      stats->format = plan.fmt;
      stats->chunks = plan.S;
      stats->dpad = plan.dpad;
    }
    return TOD_OK;
  }
  PassInfo pi;
  pi.main_kernel = main_kernel;
  pi.sample_pass = sample_pass;
  pi.main_timed = main_timed;
  return finish_rows(ctx, dX, n, dQ, q_begin, q_count, d, k, plan, cands, plan.two ? &mp : nullptr,
                     cp, small, out, stats, tm, launches, ref, pi);
}

tod_status finish_rows(tod_ctx* ctx, const float* dX, int64_t n, const float* dQ, int64_t q_begin,
                       int64_t q_count, int d, int k, const Plan& plan, Cands cands,
                       const MainPass* mp, CertParams cp, SmallDev* small, KnnOutDev out,
                       tod_stats* stats, Timer& tm, int* launches, RefPrep* ref,
                       const PassInfo& pi) {
  const bool self = dQ == nullptr;
  cudaStream_t st = ctx->stream;
  int32_t* row_tier = out.tier;
  void* p;
  TOD_TRY(ensure(ctx, B_FAIL, (size_t)std::max<int64_t>(q_count, 1) * 4, &p));
  int32_t* fail_rows = static_cast<int32_t*>(p);
  TOD_TRY(ensure(ctx, B_FAILUB, (size_t)std::max<int64_t>(q_count, 1) * 8, &p));
  double* fail_ub = static_cast<double*>(p);
  void* rr_ws = nullptr;
  if (plan.kind == PASS_TC && rerank_use_split(d)) {
    TOD_TRY(ensure(ctx, B_RRWS, rerank_split_ws(q_count), &p));
    rr_ws = p;
  }
  TOD_CUDA(launch_rerank(dQ, q_begin, q_count, dX, n, d, k, self, cands, mp,
                         cp, out, fail_rows, fail_ub,
                         &small->fail_count, &small->max_err, small->counters, rr_ws, st, launches));
  tm.mark();  // 4: fallback start
  SmallDev h{};
  TOD_CUDA(cudaMemcpyAsync(&h, small, sizeof(SmallDev), cudaMemcpyDeviceToHost, st));
  TOD_CUDA(cudaStreamSynchronize(st));
  if (h.g.nonfinite) return fail(ctx, TOD_E_NONFINITE, "X (or Q) contains NaN or Inf");
  const int nf = h.fail_count;
  // TOD_TIER2 (testing knob): 0 = off, 1 = default (not under TOD_F_NO_CERTIFY, which
  // exercises the brute-force tier), 2 = forced (also under TOD_F_NO_CERTIFY, and
  // an fp16 pass's re-run regardless of its cost estimate)
  const char* t2e = getenv("TOD_TIER2");
  const int t2 = t2e ? atoi(t2e) : 1;
  // Second tier (SURVEY 8(a) a4 tier 1): the rows pass 1 could not certify are
  // re-answered as queries by the fp16 two-pass path on just those rows -- for a
  // bf16 pass at the fp16 default K' (finer quantization), for an fp16 pass with
  // twice its K' on the references already prepared (a wider candidate set:
  // C5 2,484 failing rows of 2e6, 371 ms as fp64 threshold passes over X).  Only
  // when the fp16 plan can serve k2 = k (+1 for the dropped self) neighbours, and
  // never nested; otherwise, or if it fails, the fp64 tiers answer.
  // (the fp16 re-run costs about one main pass of ceil(nf/128) query tiles over
  // all references; the fp64 threshold tier one fp64 pass over X per 4 rows:
  // the re-run wins once nf * n * d is large -- C4, C5 -- not for C2's 1 row)
  const bool t2_fp16 = plan.fmt == TOD_FMT_FP16 && plan.two && (t2 == 2 || (double)nf * n * d >= 2e10);
  const int kp2 = t2_fp16 ? std::min(2 * plan.kp_target, 256) : 0;
  bool tier2 = nf > 0 && (plan.fmt == TOD_FMT_BF16 || t2_fp16) && t2 != 0 &&
               ctx->tier_depth == 0 && (t2 == 2 || !(ctx->cfg.flags & TOD_F_NO_CERTIFY)) &&
               (int64_t)k + (self ? 1 : 0) <= n && k + (self ? 1 : 0) <= TOD_MAX_K;
  if (tier2) {
    const int fmt_saved = ctx->cfg.format, kp_saved = ctx->cfg.kprime;
    ctx->cfg.format = TOD_FMT_FP16;
    ctx->cfg.kprime = kp2;
    Plan p2;
    const std::string msg_saved = ctx->msg;
    tier2 = make_plan(ctx, n, nf, d, k + (self ? 1 : 0), &p2) == TOD_OK && (!t2_fp16 || p2.two);
    ctx->cfg.format = fmt_saved;
    ctx->cfg.kprime = kp_saved;
    ctx->msg = msg_saved;
  }
  bool tier2_done = false;
  const int32_t* rows_t2 = nullptr;
  if (row_tier) TOD_CUDA(cudaMemsetAsync(row_tier, 0, (size_t)q_count * 4, st));
  if (tier2) {
    // bf16 rows not certified: the fp16 pass on just those rows (its own
    // fallback answers whatever it cannot certify), then scattered back
    TOD_TRY(ensure(ctx, B_T2ROWS, (size_t)nf * 4, &p));
    int32_t* rows = static_cast<int32_t*>(p);
    rows_t2 = rows;
    TOD_CUDA(cudaMemcpyAsync(rows, fail_rows, (size_t)nf * 4, cudaMemcpyDeviceToDevice, st));
    TOD_TRY(ensure(ctx, B_T2Q, (size_t)nf * d * 4, &p));
    float* qf = static_cast<float*>(p);
    TOD_CUDA(launch_gather_rows(self ? dX : dQ, self ? q_begin : 0, rows, nf, d, qf, st, launches));
    const int k2 = self ? k + 1 : k;
    KnnOutDev o2{};
    TOD_TRY(ensure(ctx, B_T2IDX, (size_t)nf * k2 * 8, &p));
    o2.idx = static_cast<int64_t*>(p);
    TOD_TRY(ensure(ctx, B_T2D64, (size_t)nf * k2 * 8, &p));
    o2.dist64 = static_cast<double*>(p);
    const int fmt_saved = ctx->cfg.format, kp_saved = ctx->cfg.kprime;
    ctx->cfg.format = TOD_FMT_FP16;
    ctx->cfg.kprime = kp2;
    Timer off{ctx, false};
    // a bf16 pass: the fp16 tier re-quantizes the references in its own format;
    // an fp16 pass: its reference image (and scale, bounds) serve as they are
    RefPrep ref2;
    RefPrep* rp = ref;
    if (!t2_fp16) {
      ref->ready = false;
      rp = &ref2;
    }
    ++ctx->tier_depth;
    const tod_status s2 = run_knn(ctx, dX, n, qf, 0, nf, d, k2, o2, nullptr, off, launches, rp);
    --ctx->tier_depth;
    ctx->cfg.format = fmt_saved;
    ctx->cfg.kprime = kp_saved;
    if (s2 == TOD_OK) {
      TOD_CUDA(launch_tier2_scatter(rows, nf, q_begin, self, k, k2, o2.idx, o2.dist64, out, st,
                                    launches));
      tier2_done = true;
    } else if (s2 != TOD_E_UNSUPPORTED && s2 != TOD_E_NOMEM) {
      return s2;
    } else {  // the fp64 tiers answer instead: the failing rows are still in fail_rows
      // (the inner call may have reused fail_rows / fail_ub: restore the rows and
      // drop the upper bounds -- 0x7F7F... is a valid, huge bound)
      ctx->msg.clear();
      TOD_CUDA(cudaMemcpyAsync(fail_rows, rows, (size_t)nf * 4, cudaMemcpyDeviceToDevice, st));
      TOD_CUDA(cudaMemsetAsync(fail_ub, 0x7F, (size_t)nf * 8, st));
    }
  }
  if (row_tier && nf > 0)  // diagnostics: 1 = bf16 -> fp16 second tier, 2 = fp64 tiers
    TOD_CUDA(launch_mark_rows(tier2_done ? rows_t2 : fail_rows, nf, tier2_done ? 1 : 2, row_tier, st,
                              launches));
  if (nf > 0 && !tier2_done) {
    TOD_TRY(ensure(ctx, B_FBPART, fallback_workspace(h.fail_count, k, n, ctx->num_sms), &p));
    TOD_CUDA(launch_fallback(dQ, q_begin, dX, n, d, k, self, fail_rows, fail_ub, h.fail_count, out, p,
                             ctx->num_sms, st, launches));
  }
  tm.mark();  // 5: end of kNN
  if (stats) {
    stats->rows = q_count;
    stats->certified = q_count - h.fail_count;
    stats->fallback_rows = h.fail_count;
    stats->kprime = plan.two ? plan.kp_target : plan.kp;
    stats->format = plan.fmt;
    stats->chunks = plan.two ? plan.main_S : plan.S;
    stats->dpad = plan.dpad;
    stats->scale = plan.kind == PASS_TC ? h.g.s : 1.0;
    stats->max_abs_err = h.max_err;
    stats->main_kernel = pi.main_kernel;
    stats->sample_pass = pi.sample_pass;
    stats->ms_main_kernel = 0.f;
    if (pi.main_timed) cudaEventElapsedTime(&stats->ms_main_kernel, ctx->evk[0], ctx->evk[1]);
    stats->cand_groups = (int64_t)h.counters[0];
    stats->visited_groups = (int64_t)h.counters[1];
    stats->cand_columns = (int64_t)h.counters[2];
    stats->prebound_skipped = (int64_t)h.counters[3];
  }
  return TOD_OK;
}

// NWR core (all pointers device): counts, then (cols != nullptr) the CSR
// neighbour lists.  Returns the total pair count in *total.
tod_status run_nwr(tod_ctx* ctx, const float* dX, int64_t n, int d, double phi, int64_t q_begin,
                   int64_t q_count, int64_t* dcounts, int64_t* drow_ptr, int32_t* dcols,
                   int64_t capacity, int64_t* total, tod_stats* stats, Timer& tm,
                   int* launches) {
  cudaStream_t st = ctx->stream;
  int fmt = ctx->cfg.format;
  if (fmt == TOD_FMT_AUTO) fmt = TOD_FMT_FP16;
  if (fmt != TOD_FMT_FP16 && fmt != TOD_FMT_BF16)
    return fail(ctx, TOD_E_UNSUPPORTED, "NWR runs on the tensor-core pass (fp16/bf16 format)");
  if (d > 64) return fail(ctx, TOD_E_UNSUPPORTED, "NWR supports d <= 64 in this build (d=%d)", d);
  const int dpad = d <= 16 ? 16 : d <= 32 ? 32 : 64;
  void* p;
  TOD_TRY(ensure(ctx, B_SMALL, sizeof(SmallDev), &p));
  SmallDev* small = static_cast<SmallDev*>(p);
  TOD_CUDA(cudaMemsetAsync(small, 0, sizeof(SmallDev), st));
  CertParams cp{};
  cp.kind = PASS_TC;
  cp.d = d;
  cp.dpad = dpad;
  cp.s = 1.0;
  cp.g = &small->g;
  tm.mark();  // 1: prep
  Image A, B;
  RefPrep ref;
  TOD_TRY(prep_tc(ctx, dX, n, nullptr, q_begin, q_count, d, fmt, dpad, &small->g, &A, &B, &cp,
                  &ref, launches));
  TOD_TRY(ensure(ctx, B_NWRTAU, (size_t)std::max<int64_t>(q_count, 1) * 4, &p));
  float* tau = static_cast<float*>(p);
  TOD_CUDA(launch_nwr_tau(q_count, phi, cp, tau, st, launches));
  tm.mark();  // 2: main pass
  MainPass mp;
  const double img_bytes = (double)B.n_pad * (dpad + 16) * 2;
  mp.S = std::max(1, (int)std::ceil(img_bytes / (48.0 * 1024 * 1024)));
  mp.R = 0;
  mp.tau_v = tau;
  mp.tau_lists = 1;
  mp.parts = tc3_parts(dpad);
  // candidate slots per (row, part): as many as a 4 GB budget allows, 128..1024
  // (rows beyond it are answered by the fp64 brute-force tier)
  mp.cap = 1024;
  while (mp.cap > 128 && (double)q_count * mp.parts * mp.cap * 8 > 4.0e9) mp.cap >>= 1;
  TOD_TRY(ensure(ctx, B_MBUF, (size_t)std::max<int64_t>(q_count, 1) * mp.parts * mp.cap * 8, &p));
  mp.buf = static_cast<uint2*>(p);
  TOD_TRY(ensure(ctx, B_MCNT, (size_t)std::max<int64_t>(q_count, 1) * mp.parts * 4, &p));
  mp.cnt = static_cast<int*>(p);
  TOD_CUDA(cudaMemsetAsync(mp.cnt, 0, (size_t)std::max<int64_t>(q_count, 1) * mp.parts * 4, st));
  const bool pair = tc4_preferred(dpad) && !(ctx->cfg.flags & TOD_F_MAIN_1SM) &&
                    tc4_fits(dpad, mp.parts);
  if (tm.on) cudaEventRecord(ctx->evk[0], st);
  if (pair)
    TOD_CUDA(launch_knn_tc4(A, B, q_begin, q_count, true, fmt, mp, ctx->num_sms, 0, st, launches));
  else
    TOD_CUDA(launch_knn_tc3(A, B, q_begin, q_count, true, fmt, mp, ctx->num_sms, 0, st, launches));
  if (tm.on) cudaEventRecord(ctx->evk[1], st);
  tm.mark();  // 3: verification
  TOD_TRY(ensure(ctx, B_FAIL, (size_t)std::max<int64_t>(q_count, 1) * 4, &p));
  int32_t* ovf_rows = static_cast<int32_t*>(p);
  TOD_TRY(ensure(ctx, B_NWRTASK, nwr_tasks_ws(q_count, mp) * 8, &p));
  int64_t* tasks_ws = static_cast<int64_t*>(p);
  TOD_TRY(ensure(ctx, B_SCAN, scan_workspace(q_count), &p));
  void* scan_ws = p;
  TOD_CUDA(launch_nwr_verify(nullptr, q_begin, q_count, dX, n, d, true, phi, mp, 0, dcounts,
                             nullptr, nullptr, ovf_rows, &small->fail_count, tasks_ws, scan_ws,
                             ctx->num_sms, st, launches));
  SmallDev h{};
  TOD_CUDA(cudaMemcpyAsync(&h, small, sizeof(SmallDev), cudaMemcpyDeviceToHost, st));
  TOD_CUDA(cudaStreamSynchronize(st));
  if (h.g.nonfinite) return fail(ctx, TOD_E_NONFINITE, "X contains NaN or Inf");
  const int novf = h.fail_count;
  TOD_TRY(ensure(ctx, B_NWRBLK, (size_t)std::max(novf, 1) * nwr_brute_slices() * 8, &p));
  int64_t* bcnt = static_cast<int64_t*>(p);
  TOD_CUDA(launch_nwr_brute(nullptr, q_begin, dX, n, d, true, phi, ovf_rows, novf, 0, dcounts,
                            nullptr, nullptr, bcnt, st, launches));
  TOD_TRY(ensure(ctx, B_SCAN, scan_workspace(q_count), &p));
  int64_t* part = static_cast<int64_t*>(p);
  TOD_CUDA(launch_scan(dcounts, q_count, drow_ptr, part, st, launches));
  TOD_CUDA(cudaMemcpyAsync(total, drow_ptr + q_count, 8, cudaMemcpyDeviceToHost, st));
  TOD_CUDA(cudaStreamSynchronize(st));
  tm.mark();  // 4: lists
  if (dcols && *total <= capacity) {
    TOD_CUDA(launch_nwr_verify(nullptr, q_begin, q_count, dX, n, d, true, phi, mp, 1, dcounts,
                               drow_ptr, dcols, ovf_rows, &small->fail_count, tasks_ws, nullptr,
                               ctx->num_sms, st, launches));
    TOD_CUDA(launch_nwr_brute(nullptr, q_begin, dX, n, d, true, phi, ovf_rows, novf, 1, dcounts,
                              drow_ptr, dcols, bcnt, st, launches));
  }
  tm.mark();  // 5
  if (stats) {
    stats->rows = q_count;
    stats->certified = q_count - novf;
    stats->fallback_rows = novf;
    stats->format = fmt;
    stats->dpad = dpad;
    stats->scale = h.g.s;
    stats->main_kernel = pair ? 4 : 3;
    stats->chunks = mp.S;
    if (tm.on) cudaEventElapsedTime(&stats->ms_main_kernel, ctx->evk[0], ctx->evk[1]);
  }
  return TOD_OK;
}


tod_status validate_common(tod_ctx* ctx, int64_t n, int32_t d, int32_t k) {
  if (!ctx) return TOD_E_ARG;
  if (n < 1 || n > INT32_MAX) return fail(ctx, TOD_E_RANGE, "n=%lld outside [1, 2^31-1]", (long long)n);
  if (d < 1 || d > 4096) return fail(ctx, TOD_E_RANGE, "d=%d outside [1, 4096]", d);
  if (k < 1) return fail(ctx, TOD_E_RANGE, "k=%d < 1", k);
  if (k > TOD_MAX_K)
    return fail(ctx, TOD_E_UNSUPPORTED, "k=%d exceeds this build's limit TOD_MAX_K=%d", k, TOD_MAX_K);
  return TOD_OK;
}


tod_status stage_outputs(tod_ctx* ctx, const tod_knn_out* o, int64_t q, int k, OutStage* s) {
  tod_knn_out z{};
  if (!o) o = &z;
  const size_t qk = (size_t)q * k;
  TOD_TRY(dev_view(ctx, o->idx, qk, B_IDX, &s->dev.idx, &s->st_idx));
  TOD_TRY(dev_view(ctx, o->dist, qk, B_DIST, &s->dev.dist, &s->st_dist));
  TOD_TRY(dev_view(ctx, o->dist64, qk, B_DIST64, &s->dev.dist64, &s->st_d64));
  TOD_TRY(dev_view(ctx, o->score_kth, (size_t)q, B_KTH, &s->dev.score_kth, &s->st_kth));
  TOD_TRY(dev_view(ctx, o->score_mean, (size_t)q, B_MEAN, &s->dev.score_mean, &s->st_mean));
  TOD_TRY(dev_view(ctx, o->kdist64, (size_t)q, B_KD64, &s->dev.kdist64, &s->st_kd));
  TOD_TRY(dev_view(ctx, o->row_tier, (size_t)q, B_TIER, &s->dev.tier, &s->st_tier));
  return TOD_OK;
}

tod_status unstage_outputs(tod_ctx* ctx, const tod_knn_out* o, int64_t q, int k, const OutStage& s) {
  if (!o) return TOD_OK;
  const size_t qk = (size_t)q * k;
  cudaStream_t st = ctx->stream;
  if (s.st_idx) TOD_CUDA(cudaMemcpyAsync(o->idx, s.dev.idx, qk * 8, cudaMemcpyDeviceToHost, st));
  if (s.st_dist) TOD_CUDA(cudaMemcpyAsync(o->dist, s.dev.dist, qk * 4, cudaMemcpyDeviceToHost, st));
  if (s.st_d64) TOD_CUDA(cudaMemcpyAsync(o->dist64, s.dev.dist64, qk * 8, cudaMemcpyDeviceToHost, st));
  if (s.st_kth) TOD_CUDA(cudaMemcpyAsync(o->score_kth, s.dev.score_kth, q * 4, cudaMemcpyDeviceToHost, st));
  if (s.st_mean) TOD_CUDA(cudaMemcpyAsync(o->score_mean, s.dev.score_mean, q * 4, cudaMemcpyDeviceToHost, st));
  if (s.st_kd) TOD_CUDA(cudaMemcpyAsync(o->kdist64, s.dev.kdist64, q * 8, cudaMemcpyDeviceToHost, st));
  if (s.st_tier) TOD_CUDA(cudaMemcpyAsync(o->row_tier, s.dev.tier, q * 4, cudaMemcpyDeviceToHost, st));
  return TOD_OK;
}

tod_status stage_input(tod_ctx* ctx, const float* user, size_t count, int id, const float** dev) {
  if (!user) return fail(ctx, TOD_E_ARG, "null input pointer");
  if (is_device_ptr(user, ctx->device)) {
    *dev = user;
    return TOD_OK;
  }
  void* p;
  TOD_TRY(ensure(ctx, id, count * 4, &p));
  TOD_CUDA(cudaMemcpyAsync(p, user, count * 4, cudaMemcpyHostToDevice, ctx->stream));
  *dev = static_cast<const float*>(p);
  return TOD_OK;
}

// Automatic batching (SURVEY 8(a) level 3): the query-dependent
// device workspace of one run_knn call, per query row, from the plan.
size_t knn_bytes_per_row(const Plan& p, int k) {
  size_t b = (size_t)p.lists * p.kp * 12 + (size_t)p.lists * 4;  // pass-1 lists + thresholds
  if (p.kind == PASS_TC && p.S > 1) b += (size_t)p.lists * p.kp * 8;  // parked list state (B_STLIST)
  if (p.two) {
    const int parts = std::max(1, tc3_parts(p.dpad));
    b += (size_t)parts * ((size_t)p.cap * 2 / parts * 8 + 4);  // main-pass buffers + counts
    b += (size_t)parts * 8 * 4;                                 // key-only sample minima (B_SAMP)
  }
  b += (size_t)(p.dpad + 16) * 2 + 16;  // query image row + its bounds
  b += (size_t)k * 24 + 64;             // staged outputs, fail list and bounds
  // fallback: threshold tier (1024 candidates x 12 B) + per-slice lists, for
  // every row in the worst case (the tier only runs on failing rows)
  b += 1024 * 12 + (size_t)k * 12 * 8;
  if (p.kind == PASS_TC && rerank_use_split(p.dpad))
    b += rerank_split_ws(1024) / 1024;  // split re-rank: visited groups, kept columns, tasks
  return b;
}

// run_knn over [q_begin, q_begin + q_count), in chunks of 128-row multiples when
// ctx->cfg.workspace_bytes is set and one call would exceed it.  Rows are
// independent (per-row thresholds, bounds and certificate; the reference-side
// quantization constants are global), so the outputs are bit-identical.
tod_status run_knn_auto(tod_ctx* ctx, const float* dX, int64_t n, const float* dQ, int64_t q_begin,
                        int64_t q_count, int d, int k, KnnOutDev out, tod_stats* stats, Timer& tm,
                        int* launches) {
  int64_t rows = q_count;
  if (ctx->cfg.workspace_bytes > 0 && q_count > 128) {
    Plan plan;
    TOD_TRY(make_plan(ctx, n, q_count, d, k, &plan));
    const size_t per = knn_bytes_per_row(plan, k);
    rows = std::max<int64_t>(128, (int64_t)(ctx->cfg.workspace_bytes / per) / 128 * 128);
  }
  RefPrep ref;
  ref.dQall = dQ;
  ref.nq_all = dQ ? q_count : 0;
  if (rows >= q_count) {
    TOD_TRY(run_knn(ctx, dX, n, dQ, q_begin, q_count, d, k, out, stats, tm, launches, &ref));
    if (stats) stats->query_chunks = 1;
    return TOD_OK;
  }
  Timer off{ctx, false};
  tm.mark();  // 1: chunked mode reports the whole compute as one phase (see finish_stats)
  tod_stats acc{};
  int nch = 0;
  for (int64_t r0 = 0; r0 < q_count; r0 += rows, ++nch) {
    const int64_t qc = std::min<int64_t>(rows, q_count - r0);
    KnnOutDev o = out;
    auto sh = [&](auto* p, int64_t per_row) { return p ? p + r0 * per_row : p; };
    o.idx = sh(out.idx, k);
    o.dist = sh(out.dist, k);
    o.dist64 = sh(out.dist64, k);
    o.score_kth = sh(out.score_kth, 1);
    o.score_mean = sh(out.score_mean, 1);
    o.kdist64 = sh(out.kdist64, 1);
    o.tier = sh(out.tier, 1);
    tod_stats cs{};
    TOD_TRY(run_knn(ctx, dX, n, dQ ? dQ + r0 * d : nullptr, dQ ? 0 : q_begin + r0, qc, d, k, o,
                    stats ? &cs : nullptr, off, launches, &ref));
    if (nch == 0) acc = cs;
    else {
      acc.rows += cs.rows;
      acc.certified += cs.certified;
      acc.fallback_rows += cs.fallback_rows;
      acc.cand_groups += cs.cand_groups;
      acc.visited_groups += cs.visited_groups;
      acc.cand_columns += cs.cand_columns;
      acc.prebound_skipped += cs.prebound_skipped;
      acc.max_abs_err = std::max(acc.max_abs_err, cs.max_abs_err);
    }
  }
  for (int i = 0; i < 4; ++i) tm.mark();  // 2..5
  if (stats) {
    *stats = acc;
    stats->query_chunks = nch;
  }
  return TOD_OK;
}

void finish_stats(tod_stats* stats, Timer& tm, int launches, int i_lof_end) {
  if (!stats) return;
  stats->kernel_launches = launches;
  stats->ms_stage = tm.between(0, 1);
  stats->ms_prep = tm.between(1, 2);
  stats->ms_main = tm.between(2, 3);
  stats->ms_certify = tm.between(3, 4);
  stats->ms_fallback = tm.between(4, 5);
  stats->ms_lof = i_lof_end > 0 ? tm.between(5, i_lof_end) : 0.f;
  stats->ms_total = tm.between(0, tm.n - 1);
  if (stats->query_chunks > 1)  // chunked: phases interleave, only the totals are meaningful
    stats->ms_prep = stats->ms_main = stats->ms_certify = stats->ms_fallback = stats->ms_main_kernel = 0.f;
}

}  // namespace todapi

extern "C" {

int32_t tod_abi_version(void) { return TOD_ABI_VERSION; }
const char* tod_build_info(void) { return TOD_BUILD_INFO; }

const char* tod_status_str(tod_status s) {
  switch (s) {
    case TOD_OK: return "TOD_OK";
    case TOD_E_ARG: return "TOD_E_ARG: invalid argument";
    case TOD_E_NONFINITE: return "TOD_E_NONFINITE: NaN or Inf in input";
    case TOD_E_RANGE: return "TOD_E_RANGE: size or k out of range";
    case TOD_E_NOMEM: return "TOD_E_NOMEM: device allocation failed";
    case TOD_E_CUDA: return "TOD_E_CUDA: CUDA runtime error";
    case TOD_E_NCCL: return "TOD_E_NCCL: NCCL error";
    case TOD_E_UNSUPPORTED: return "TOD_E_UNSUPPORTED: not supported by this build";
    case TOD_E_INTERNAL: return "TOD_E_INTERNAL: internal error";
  }
  return "unknown tod_status";
}

const char* tod_last_message(const tod_ctx* ctx) { return ctx ? ctx->msg.c_str() : ""; }

tod_status tod_create(const tod_config* cfg, tod_ctx** out) {
  if (!out) return TOD_E_ARG;
  *out = nullptr;
  tod_ctx* ctx = new (std::nothrow) tod_ctx();
  if (!ctx) return TOD_E_NOMEM;
  if (cfg) ctx->cfg = *cfg;
  ctx->device = ctx->cfg.device;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0 || ctx->device < 0 || ctx->device >= ndev) {
    cudaGetLastError();
    delete ctx;
    return TOD_E_CUDA;
  }
  cudaDeviceProp prop;
  if (cudaSetDevice(ctx->device) != cudaSuccess ||
      cudaGetDeviceProperties(&prop, ctx->device) != cudaSuccess) {
    delete ctx;
    return TOD_E_CUDA;
  }
  if (prop.major != 10 || prop.minor != 0) {
    delete ctx;
    return TOD_E_UNSUPPORTED;  // built for sm_100a only
  }
  ctx->num_sms = prop.multiProcessorCount;
  if (ctx->cfg.stream) {
    ctx->stream = static_cast<cudaStream_t>(ctx->cfg.stream);
  } else {
    // A BLOCKING stream: it waits for work the caller queued on the legacy
    // default stream (e.g. torch kernels producing X) before each of our
    // kernels starts, so device inputs are never read stale.
    if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamDefault) != cudaSuccess) {
      delete ctx;
      return TOD_E_CUDA;
    }
    ctx->own_stream = true;
  }
  for (auto& ev : ctx->ev) cudaEventCreate(&ev);
  for (auto& ev : ctx->evk) cudaEventCreate(&ev);
  *out = ctx;
  return TOD_OK;
}

tod_status tod_destroy(tod_ctx* ctx) {
  if (!ctx) return TOD_OK;
  cudaSetDevice(ctx->device);
  if (ctx->stream) cudaStreamSynchronize(ctx->stream);
  ctx->ws.release();
  for (auto& ev : ctx->ev)
    if (ev) cudaEventDestroy(ev);
  for (auto ev : ctx->evk)
    if (ev) cudaEventDestroy(ev);
  if (ctx->own_stream) cudaStreamDestroy(ctx->stream);
  for (auto& w : ctx->rank_ws) w.release();
  if (ctx->nccl_comm) tod_comm_release(ctx);
  if (ctx->comm_stream) cudaStreamDestroy(ctx->comm_stream);
  delete ctx;
  return TOD_OK;
}

tod_status tod_knn(tod_ctx* ctx, const float* X, int64_t n, int32_t d, int32_t k, int64_t q_begin,
                   int64_t q_count, const tod_knn_out* out, tod_stats* stats) {
  TOD_TRY(validate_common(ctx, n, d, k));
  if (n < 2 || k > n - 1) return fail(ctx, TOD_E_RANGE, "need 1 <= k <= n-1 (n=%lld k=%d)", (long long)n, k);
  if (q_begin < 0 || q_count < 0 || q_begin + q_count > n)
    return fail(ctx, TOD_E_RANGE, "query rows [%lld, %lld) outside [0, %lld)", (long long)q_begin,
                (long long)(q_begin + q_count), (long long)n);
  TOD_CUDA(cudaSetDevice(ctx->device));
  if (stats) memset(stats, 0, sizeof *stats);
  Timer tm{ctx, (ctx->cfg.flags & TOD_F_TIMING) != 0};
  int launches = 0;
  tm.mark();  // 0
  const float* dX;
  TOD_TRY(stage_input(ctx, X, (size_t)n * d, B_X, &dX));
  OutStage os;
  TOD_TRY(stage_outputs(ctx, out, q_count, k, &os));
  if (q_count > 0) TOD_TRY(run_knn_auto(ctx, dX, n, nullptr, q_begin, q_count, d, k, os.dev, stats, tm, &launches));
  TOD_TRY(unstage_outputs(ctx, out, q_count, k, os));
  tm.mark();
  TOD_CUDA(cudaStreamSynchronize(ctx->stream));
  finish_stats(stats, tm, launches, 0);
  ctx->msg.clear();
  return TOD_OK;
}

tod_status tod_knn_query(tod_ctx* ctx, const float* Q, int64_t nq, const float* X, int64_t n,
                         int32_t d, int32_t k, const tod_knn_out* out, tod_stats* stats) {
  TOD_TRY(validate_common(ctx, n, d, k));
  if (k > n) return fail(ctx, TOD_E_RANGE, "need 1 <= k <= n (n=%lld k=%d)", (long long)n, k);
  if (nq < 0 || nq > INT32_MAX) return fail(ctx, TOD_E_RANGE, "nq=%lld out of range", (long long)nq);
  TOD_CUDA(cudaSetDevice(ctx->device));
  if (stats) memset(stats, 0, sizeof *stats);
  Timer tm{ctx, (ctx->cfg.flags & TOD_F_TIMING) != 0};
  int launches = 0;
  tm.mark();
  const float *dX, *dQ;
  TOD_TRY(stage_input(ctx, X, (size_t)n * d, B_X, &dX));
  if (nq > 0) TOD_TRY(stage_input(ctx, Q, (size_t)nq * d, B_Q, &dQ));
  OutStage os;
  TOD_TRY(stage_outputs(ctx, out, nq, k, &os));
  if (nq > 0) TOD_TRY(run_knn_auto(ctx, dX, n, dQ, 0, nq, d, k, os.dev, stats, tm, &launches));
  TOD_TRY(unstage_outputs(ctx, out, nq, k, os));
  tm.mark();
  TOD_CUDA(cudaStreamSynchronize(ctx->stream));
  finish_stats(stats, tm, launches, 0);
  ctx->msg.clear();
  return TOD_OK;
}

tod_status tod_nwr(tod_ctx* ctx, const float* X, int64_t n, int32_t d, double phi,
                   int64_t q_begin, int64_t q_count, int64_t* counts, int64_t* row_ptr,
                   int32_t* cols, int64_t capacity, int64_t* total, tod_stats* stats) {
  TOD_TRY(validate_common(ctx, n, d, 1));
  if (!(phi == phi) || phi == INFINITY) return fail(ctx, TOD_E_ARG, "phi must be finite");
  if (q_begin < 0 || q_count < 0 || q_begin + q_count > n)
    return fail(ctx, TOD_E_RANGE, "query rows [%lld, %lld) outside [0, %lld)", (long long)q_begin,
                (long long)(q_begin + q_count), (long long)n);
  if (!total) return fail(ctx, TOD_E_ARG, "total must not be NULL");
  if (cols && capacity < 0) return fail(ctx, TOD_E_ARG, "negative capacity");
  TOD_CUDA(cudaSetDevice(ctx->device));
  if (stats) memset(stats, 0, sizeof *stats);
  *total = 0;
  Timer tm{ctx, (ctx->cfg.flags & TOD_F_TIMING) != 0};
  int launches = 0;
  tm.mark();  // 0
  const float* dX;
  TOD_TRY(stage_input(ctx, X, (size_t)n * d, B_X, &dX));
  int64_t *dcounts, *dptr;
  int32_t* dcols;
  bool st_c, st_p, st_l;
  // counts and row_ptr are always computed (device temporaries when not requested)
  void* p;
  TOD_TRY(dev_view(ctx, counts, (size_t)q_count, B_NWRCNT, &dcounts, &st_c));
  if (!dcounts) {
    TOD_TRY(ensure(ctx, B_NWRCNT, (size_t)std::max<int64_t>(q_count, 1) * 8, &p));
    dcounts = static_cast<int64_t*>(p);
  }
  TOD_TRY(dev_view(ctx, row_ptr, (size_t)q_count + 1, B_NWRPTR, &dptr, &st_p));
  if (!dptr) {
    TOD_TRY(ensure(ctx, B_NWRPTR, (size_t)(q_count + 1) * 8, &p));
    dptr = static_cast<int64_t*>(p);
  }
  TOD_TRY(dev_view(ctx, cols, (size_t)std::max<int64_t>(capacity, 1), B_NWRCOLS, &dcols, &st_l));
  if (q_count > 0) {
    TOD_TRY(run_nwr(ctx, dX, n, d, phi, q_begin, q_count, dcounts, dptr, dcols, capacity, total,
                    stats, tm, &launches));
  } else {
    TOD_CUDA(cudaMemsetAsync(dptr, 0, 8, ctx->stream));
  }
  cudaStream_t st = ctx->stream;
  if (st_c) TOD_CUDA(cudaMemcpyAsync(counts, dcounts, (size_t)q_count * 8, cudaMemcpyDeviceToHost, st));
  if (st_p)
    TOD_CUDA(cudaMemcpyAsync(row_ptr, dptr, (size_t)(q_count + 1) * 8, cudaMemcpyDeviceToHost, st));
  const bool fits = *total <= capacity;
  if (st_l && fits && *total > 0)
    TOD_CUDA(cudaMemcpyAsync(cols, dcols, (size_t)*total * 4, cudaMemcpyDeviceToHost, st));
  tm.mark();
  TOD_CUDA(cudaStreamSynchronize(st));
  finish_stats(stats, tm, launches, 0);
  if (cols && !fits)
    return fail(ctx, TOD_E_RANGE, "cols capacity %lld < %lld neighbour pairs (counts, row_ptr and "
                "total are valid)", (long long)capacity, (long long)*total);
  ctx->msg.clear();
  return TOD_OK;
}

tod_status tod_abod(tod_ctx* ctx, const float* X, int64_t n, int32_t d, int32_t k,
                    int64_t q_begin, int64_t q_count, float* score, const tod_knn_out* knn_out,
                    tod_stats* stats) {
  TOD_TRY(validate_common(ctx, n, d, k));
  if (n < 2 || k > n - 1) return fail(ctx, TOD_E_RANGE, "need 1 <= k <= n-1 (n=%lld k=%d)", (long long)n, k);
  if (k > abod_max_k()) return fail(ctx, TOD_E_UNSUPPORTED, "ABOD supports k <= %d", abod_max_k());
  if (q_begin < 0 || q_count < 0 || q_begin + q_count > n)
    return fail(ctx, TOD_E_RANGE, "query rows outside [0, n)");
  if (!score) return fail(ctx, TOD_E_ARG, "score must not be NULL");
  TOD_CUDA(cudaSetDevice(ctx->device));
  if (stats) memset(stats, 0, sizeof *stats);
  Timer tm{ctx, (ctx->cfg.flags & TOD_F_TIMING) != 0};
  int launches = 0;
  tm.mark();
  const float* dX;
  TOD_TRY(stage_input(ctx, X, (size_t)n * d, B_X, &dX));
  OutStage os;
  TOD_TRY(stage_outputs(ctx, knn_out, q_count, k, &os));
  void* p;
  if (!os.dev.idx) {  // ABOD needs the neighbour indices on the device
    TOD_TRY(ensure(ctx, B_IDX, (size_t)std::max<int64_t>(q_count, 1) * k * 8, &p));
    os.dev.idx = static_cast<int64_t*>(p);
  }
  float* dscore;
  bool st_s;
  TOD_TRY(dev_view(ctx, score, (size_t)q_count, B_ABOD, &dscore, &st_s));
  if (q_count > 0) {
    TOD_TRY(run_knn_auto(ctx, dX, n, nullptr, q_begin, q_count, d, k, os.dev, stats, tm, &launches));
    TOD_CUDA(launch_abod(dX, q_begin, q_count, d, k, os.dev.idx, dscore, ctx->stream, &launches));
  }
  TOD_TRY(unstage_outputs(ctx, knn_out, q_count, k, os));
  if (st_s) TOD_CUDA(cudaMemcpyAsync(score, dscore, (size_t)q_count * 4, cudaMemcpyDeviceToHost, ctx->stream));
  tm.mark();
  TOD_CUDA(cudaStreamSynchronize(ctx->stream));
  finish_stats(stats, tm, launches, 0);
  ctx->msg.clear();
  return TOD_OK;
}

tod_status tod_knn_classify(tod_ctx* ctx, const float* Q, int64_t nq, const float* X, int64_t n,
                            int32_t d, int32_t k, const int32_t* labels, int32_t* pred,
                            tod_stats* stats) {
  TOD_TRY(validate_common(ctx, n, d, k));
  if (k > n) return fail(ctx, TOD_E_RANGE, "need 1 <= k <= n (n=%lld k=%d)", (long long)n, k);
  if (nq < 0 || nq > INT32_MAX) return fail(ctx, TOD_E_RANGE, "nq out of range");
  if (!labels || !pred) return fail(ctx, TOD_E_ARG, "labels and pred must not be NULL");
  TOD_CUDA(cudaSetDevice(ctx->device));
  if (stats) memset(stats, 0, sizeof *stats);
  Timer tm{ctx, (ctx->cfg.flags & TOD_F_TIMING) != 0};
  int launches = 0;
  tm.mark();
  const float *dX, *dQ = nullptr;
  TOD_TRY(stage_input(ctx, X, (size_t)n * d, B_X, &dX));
  if (nq > 0) TOD_TRY(stage_input(ctx, Q, (size_t)nq * d, B_Q, &dQ));
  void* p;
  const int32_t* dlab;
  if (is_device_ptr(labels, ctx->device)) {
    dlab = labels;
  } else {
    TOD_TRY(ensure(ctx, B_LABELS, (size_t)n * 4, &p));
    TOD_CUDA(cudaMemcpyAsync(p, labels, (size_t)n * 4, cudaMemcpyHostToDevice, ctx->stream));
    dlab = static_cast<const int32_t*>(p);
  }
  int32_t* dpred;
  bool st_p;
  TOD_TRY(dev_view(ctx, pred, (size_t)std::max<int64_t>(nq, 1), B_PRED, &dpred, &st_p));
  KnnOutDev kd{};
  TOD_TRY(ensure(ctx, B_IDX, (size_t)std::max<int64_t>(nq, 1) * k * 8, &p));
  kd.idx = static_cast<int64_t*>(p);
  if (nq > 0) {
    TOD_TRY(run_knn_auto(ctx, dX, n, dQ, 0, nq, d, k, kd, stats, tm, &launches));
    TOD_CUDA(launch_knn_classify(nq, k, kd.idx, dlab, dpred, ctx->stream, &launches));
  }
  if (st_p && nq > 0)
    TOD_CUDA(cudaMemcpyAsync(pred, dpred, (size_t)nq * 4, cudaMemcpyDeviceToHost, ctx->stream));
  tm.mark();
  TOD_CUDA(cudaStreamSynchronize(ctx->stream));
  finish_stats(stats, tm, launches, 0);
  ctx->msg.clear();
  return TOD_OK;
}

tod_status tod_lof(tod_ctx* ctx, const float* X, int64_t n, int32_t d, int32_t k, float* lof,
                   float* lrd, const tod_knn_out* knn_out, tod_stats* stats) {
  TOD_TRY(validate_common(ctx, n, d, k));
  if (n < 2 || k > n - 1) return fail(ctx, TOD_E_RANGE, "need 1 <= k <= n-1 (n=%lld k=%d)", (long long)n, k);
  TOD_CUDA(cudaSetDevice(ctx->device));
  if (stats) memset(stats, 0, sizeof *stats);
  Timer tm{ctx, (ctx->cfg.flags & TOD_F_TIMING) != 0};
  int launches = 0;
  tm.mark();
  const float* dX;
  TOD_TRY(stage_input(ctx, X, (size_t)n * d, B_X, &dX));
  OutStage os;
  TOD_TRY(stage_outputs(ctx, knn_out, n, k, &os));
  // LOF needs idx, dist64 and kdist64 on the device even if the caller did not ask.
  void* p;
  if (!os.dev.idx) {
    TOD_TRY(ensure(ctx, B_IDX, (size_t)n * k * 8, &p));
    os.dev.idx = static_cast<int64_t*>(p);
  }
  if (!os.dev.dist64) {
    TOD_TRY(ensure(ctx, B_DIST64, (size_t)n * k * 8, &p));
    os.dev.dist64 = static_cast<double*>(p);
  }
  if (!os.dev.kdist64) {
    TOD_TRY(ensure(ctx, B_KD64, (size_t)n * 8, &p));
    os.dev.kdist64 = static_cast<double*>(p);
  }
  TOD_TRY(run_knn_auto(ctx, dX, n, nullptr, 0, n, d, k, os.dev, stats, tm, &launches));
  TOD_TRY(ensure(ctx, B_LRD64, (size_t)n * 8, &p));
  double* lrd64 = static_cast<double*>(p);
  float *dlof, *dlrd;
  bool st_lof, st_lrd;
  TOD_TRY(dev_view(ctx, lof, (size_t)n, B_LOF, &dlof, &st_lof));
  TOD_TRY(dev_view(ctx, lrd, (size_t)n, B_LRD32, &dlrd, &st_lrd));
  TOD_CUDA(launch_lof_lrd(n, k, os.dev.idx, os.dev.dist64, os.dev.kdist64, lrd64, ctx->stream, &launches));
  TOD_CUDA(launch_lof_finish(0, n, k, os.dev.idx, lrd64, dlof, dlrd, ctx->stream, &launches));
  tm.mark();  // 6: LOF end
  TOD_TRY(unstage_outputs(ctx, knn_out, n, k, os));
  if (st_lof) TOD_CUDA(cudaMemcpyAsync(lof, dlof, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
  if (st_lrd) TOD_CUDA(cudaMemcpyAsync(lrd, dlrd, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
  tm.mark();
  TOD_CUDA(cudaStreamSynchronize(ctx->stream));
  finish_stats(stats, tm, launches, 6);
  ctx->msg.clear();
  return TOD_OK;
}

tod_status tod_debug_mainpass(tod_ctx* ctx, const float* X, int64_t n, int32_t d, float* w,
                              float* a_ops, float* b_ops, int32_t* K_out, int32_t* main_kernel) {
  TOD_TRY(validate_common(ctx, n, d, 1));
  if (n < 128) return fail(ctx, TOD_E_RANGE, "tod_debug_mainpass needs n >= 128");
  if (!X || !w || !a_ops || !b_ops || !K_out)
    return fail(ctx, TOD_E_ARG, "null pointer");
  for (const void* q : {(const void*)X, (const void*)w, (const void*)a_ops, (const void*)b_ops})
    if (!is_device_ptr(q, ctx->device)) return fail(ctx, TOD_E_ARG, "tod_debug_mainpass takes device pointers");
  TOD_CUDA(cudaSetDevice(ctx->device));
  Plan plan;
  TOD_TRY(make_plan(ctx, n, 128, d, 1, &plan));
  if (plan.kind != PASS_TC || !tc3_fits(plan.dpad))
    return fail(ctx, TOD_E_UNSUPPORTED, "tensor-core main pass not used for this shape/format");
  cudaStream_t st = ctx->stream;
  int launches = 0;
  void* p;
  TOD_TRY(ensure(ctx, B_SMALL, sizeof(SmallDev), &p));
  SmallDev* small = static_cast<SmallDev*>(p);
  TOD_CUDA(cudaMemsetAsync(small, 0, sizeof(SmallDev), st));
  CertParams cp{};
  Image A, B;
  RefPrep ref;
  TOD_TRY(prep_tc(ctx, X, n, nullptr, 0, 128, d, plan.fmt, plan.dpad, &small->g, &A, &B, &cp, &ref,
                  &launches));
  MainPass mp;
  mp.S = 1;
  mp.R = 0;
  mp.parts = tc3_parts(plan.dpad);
  mp.tau_v = nullptr;
  mp.tau_lists = 0;
  mp.buf = reinterpret_cast<uint2*>(w);  // dump: [128 x n] fp32, ld = n
  mp.cap = (int)n;
  mp.cnt = nullptr;
  const char* pe = getenv("TOD_MAIN_PAIR");
  const bool pair = (pe ? atoi(pe) != 0 : tc4_preferred(plan.dpad) != 0) &&
                    !(ctx->cfg.flags & TOD_F_MAIN_1SM) && tc4_fits(plan.dpad, mp.parts);
  if (pair) TOD_CUDA(launch_knn_tc4(A, B, 0, 128, true, plan.fmt, mp, ctx->num_sms, 4, st, &launches));
  else TOD_CUDA(launch_knn_tc3(A, B, 0, 128, true, plan.fmt, mp, ctx->num_sms, 4, st, &launches));
  TOD_CUDA(launch_image_decode(A, plan.fmt, 128, a_ops, st, &launches));
  TOD_CUDA(launch_image_decode(B, plan.fmt, n, b_ops, st, &launches));
  TOD_CUDA(cudaStreamSynchronize(st));
  *K_out = plan.dpad + 16;
  if (main_kernel) *main_kernel = pair ? 4 : 3;
  ctx->msg.clear();
  return TOD_OK;
}

tod_status tod_lof_lrd(tod_ctx* ctx, int64_t n, int32_t k, int64_t q_count, const int64_t* idx,
                       const double* dist64, const double* kdist64_all, double* lrd64_out) {
  if (!ctx) return TOD_E_ARG;
  if (n < 2 || k < 1 || k > n - 1 || q_count < 0 || q_count > n)
    return fail(ctx, TOD_E_RANGE, "bad sizes n=%lld k=%d q=%lld", (long long)n, k, (long long)q_count);
  if (!idx || !dist64 || !kdist64_all || !lrd64_out) return fail(ctx, TOD_E_ARG, "null pointer");
  TOD_CUDA(cudaSetDevice(ctx->device));
  int launches = 0;
  const size_t qk = (size_t)q_count * k;
  // stage (host -> device) as needed
  const int64_t* di = idx;
  const double *dd = dist64, *dk = kdist64_all;
  double* dl = lrd64_out;
  void* p;
  cudaStream_t st = ctx->stream;
  if (!is_device_ptr(idx, ctx->device)) {
    TOD_TRY(ensure(ctx, B_IDX, qk * 8, &p));
    TOD_CUDA(cudaMemcpyAsync(p, idx, qk * 8, cudaMemcpyHostToDevice, st));
    di = static_cast<int64_t*>(p);
  }
  if (!is_device_ptr(dist64, ctx->device)) {
    TOD_TRY(ensure(ctx, B_DIST64, qk * 8, &p));
    TOD_CUDA(cudaMemcpyAsync(p, dist64, qk * 8, cudaMemcpyHostToDevice, st));
    dd = static_cast<double*>(p);
  }
  if (!is_device_ptr(kdist64_all, ctx->device)) {
    TOD_TRY(ensure(ctx, B_KDALL, (size_t)n * 8, &p));
    TOD_CUDA(cudaMemcpyAsync(p, kdist64_all, n * 8, cudaMemcpyHostToDevice, st));
    dk = static_cast<double*>(p);
  }
  const bool st_out = !is_device_ptr(lrd64_out, ctx->device);
  if (st_out) {
    TOD_TRY(ensure(ctx, B_LRD64, (size_t)std::max<int64_t>(q_count, 1) * 8, &p));
    dl = static_cast<double*>(p);
  }
  TOD_CUDA(launch_lof_lrd(q_count, k, di, dd, dk, dl, st, &launches));
  if (st_out) TOD_CUDA(cudaMemcpyAsync(lrd64_out, dl, q_count * 8, cudaMemcpyDeviceToHost, st));
  TOD_CUDA(cudaStreamSynchronize(st));
  return TOD_OK;
}

tod_status tod_lof_finish(tod_ctx* ctx, int64_t n, int32_t k, int64_t q_begin, int64_t q_count,
                          const int64_t* idx, const double* lrd64_all, float* lof_out,
                          float* lrd_out) {
  if (!ctx) return TOD_E_ARG;
  if (n < 2 || k < 1 || k > n - 1 || q_begin < 0 || q_count < 0 || q_begin + q_count > n)
    return fail(ctx, TOD_E_RANGE, "bad sizes");
  if (!idx || !lrd64_all) return fail(ctx, TOD_E_ARG, "null pointer");
  TOD_CUDA(cudaSetDevice(ctx->device));
  int launches = 0;
  const size_t qk = (size_t)q_count * k;
  cudaStream_t st = ctx->stream;
  void* p;
  const int64_t* di = idx;
  const double* dl = lrd64_all;
  if (!is_device_ptr(idx, ctx->device)) {
    TOD_TRY(ensure(ctx, B_IDX, qk * 8, &p));
    TOD_CUDA(cudaMemcpyAsync(p, idx, qk * 8, cudaMemcpyHostToDevice, st));
    di = static_cast<int64_t*>(p);
  }
  if (!is_device_ptr(lrd64_all, ctx->device)) {
    TOD_TRY(ensure(ctx, B_KDALL, (size_t)n * 8, &p));
    TOD_CUDA(cudaMemcpyAsync(p, lrd64_all, n * 8, cudaMemcpyHostToDevice, st));
    dl = static_cast<double*>(p);
  }
  float *dlof, *dlrd;
  bool st_lof, st_lrd;
  TOD_TRY(dev_view(ctx, lof_out, (size_t)q_count, B_LOF, &dlof, &st_lof));
  TOD_TRY(dev_view(ctx, lrd_out, (size_t)q_count, B_LRD32, &dlrd, &st_lrd));
  TOD_CUDA(launch_lof_finish(q_begin, q_count, k, di, dl, dlof, dlrd, st, &launches));
  if (st_lof) TOD_CUDA(cudaMemcpyAsync(lof_out, dlof, q_count * 4, cudaMemcpyDeviceToHost, st));
  if (st_lrd) TOD_CUDA(cudaMemcpyAsync(lrd_out, dlrd, q_count * 4, cudaMemcpyDeviceToHost, st));
  TOD_CUDA(cudaStreamSynchronize(st));
  return TOD_OK;
}

}  // extern "C"
