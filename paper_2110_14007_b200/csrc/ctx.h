// ctx.h — library-internal context, workspace and planning types shared by
// api.cu (single-process entry points) and shard.cu (the sharded multi-GPU
// path).  Not part of the ABI.
#pragma once
#include <cuda_runtime.h>

#include <cstddef>
#include <string>
#include <vector>

#include "../../include/tod.h"
#include "internal.h"

namespace todapi {
using namespace tod;

struct Buf {
  void* p = nullptr;
  size_t bytes = 0;
};

struct Workspace {
  Buf bufs[64];
  void release() {
    for (auto& b : bufs) {
      if (b.p) cudaFree(b.p);
      b = Buf{};
    }
  }
};

enum BufId {
  B_X = 0, B_Q, B_IMG_B, B_A2_B, B_E_B, B_IMG_A, B_A2_A, B_E_A, B_MU, B_PART,
  B_G, B_CIDX, B_CV, B_FAIL, B_SMALL, B_IDX, B_DIST, B_DIST64, B_KTH, B_MEAN, B_KD64,
  B_LRD64, B_LOF, B_LRD32, B_KDALL, B_STLIST, B_STDONE, B_FBPART, B_CKEY, B_TRACE, B_MBUF, B_MCNT,
  B_FAILUB, B_NWRTAU, B_NWRCNT, B_NWRPTR, B_NWRCOLS, B_SCAN, B_ABOD, B_LABELS, B_PRED, B_SAMP,
  B_NWRBLK, B_NWRTASK, B_RRWS, B_T2ROWS, B_T2Q, B_T2IDX, B_T2D64, B_TIER, B_EG,
  // sharded path (shard.cu)
  B_XALL, B_XSEND, B_XSLOT, B_SHTAB, B_PARTALL, B_GATHER, B_GATHER2,
  B_NBUF
};
static_assert(B_NBUF <= 64, "Workspace::bufs too small");

}  // namespace todapi

struct tod_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  tod_config cfg{};
  int num_sms = 148;
  std::string msg;
  todapi::Workspace ws;
  cudaEvent_t ev[8] = {};
  cudaEvent_t evk[2] = {};  // around the main-pass kernel (two-pass mode)
  // ---- sharded path (shard.cu): communicator of the SPMD job
  int rank = 0, world = 1;
  int loopback = 0;                          // 1: `world` virtual ranks run in this process (testing)
  void* nccl_comm = nullptr;                 // ncclComm_t when a real NCCL communicator is attached
  cudaStream_t comm_stream = nullptr;        // NCCL transfers overlap compute on this stream
  std::vector<todapi::Workspace> rank_ws;    // per (virtual) rank state of a sharded call
  int tier_depth = 0;                        // > 0 inside a second-tier re-run (no nesting)
};

namespace todapi {

tod_status fail(tod_ctx* ctx, tod_status s, const char* fmt, ...);

#define TOD_CUDA(call)                                                                    \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(ctx, e_ == cudaErrorMemoryAllocation ? TOD_E_NOMEM : TOD_E_CUDA,       \
                  "%s: %s (%s:%d)", #call, cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)

#define TOD_TRY(expr)                  \
  do {                                 \
    tod_status s_ = (expr);            \
    if (s_ != TOD_OK) return s_;       \
  } while (0)

tod_status ensure_ws(tod_ctx* ctx, Workspace& ws, int id, size_t bytes, void** out);
inline tod_status ensure(tod_ctx* ctx, int id, size_t bytes, void** out) {
  return ensure_ws(ctx, ctx->ws, id, bytes, out);
}
bool is_device_ptr(const void* p, int device);
inline int roundup(int x, int m) { return (x + m - 1) / m * m; }

struct Plan {
  int fmt;       // 1 fp16, 2 bf16, 3 fp32 simt
  int kind;      // PASS_TC / PASS_SIMT
  int dpad;
  int kp;
  int S;
  int lists;     // candidate lists per row (TC: epilogue split; SIMT: S)
  int two;       // TC: two-pass candidate selection (sample pass + append-only main pass)
  int R;         // two-pass: sample stride over 256-column reference tiles
  int main_S;    // two-pass: main-pass reference chunks
  int kp_target; // two-pass: K' (target count of kept groups)
  int cap;       // two-pass: main-pass buffer slots per (row, column half)
};
tod_status make_plan(tod_ctx* ctx, int64_t n_ref, int64_t q_count, int d, int k, Plan* p);
int main_vote(int64_t n_ref);   // main-pass filter: part-minimum vote first (rare appends)
int main_nb(const MainPass& mp);  // CTA-pair main pass: 256-column tiles x 2 or 160 x 3
int main_colmode(const MainPass& mp, int dpad);  // main pass appends column candidates
int main_ring3(int dpad, const MainPass& mp, int dbg);  // use knn_tc5 (3-deep accumulator ring)

struct Timer {
  tod_ctx* ctx;
  bool on;
  int n = 0;
  void mark() {
    if (on && n < 8) cudaEventRecord(ctx->ev[n++], ctx->stream);
  }
  float between(int a, int b) {
    if (!on || b >= n) return 0.f;
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ctx->ev[a], ctx->ev[b]);
    return ms;
  }
};

struct SmallDev {
  PrepGlobals g;
  int32_t fail_count;
  int32_t pad;
  double max_err;
  unsigned long long counters[4];  // re-rank telemetry: staged groups, visited groups, kept columns, pre-bound skips
};

// Reference-side prep shared by the query chunks of one call (automatic
// batching): computed by the first chunk, reused by the others.  A bf16 second
// tier overwrites the reference image and the globals, so it clears `ready`.
struct RefPrep {
  bool ready = false;
  const float* dQall = nullptr;  // query mode: every query row of the call (finite / absmax)
  int64_t nq_all = 0;
};

// What pass 1 did (stats only).
struct PassInfo {
  int main_kernel = 0;  // 3 single-SM, 4 CTA pairs
  int sample_pass = 0;  // 1 list-based, 2 key-only
  bool main_timed = false;
};

struct OutStage {
  KnnOutDev dev{};
  bool st_idx = false, st_dist = false, st_d64 = false, st_kth = false, st_mean = false,
       st_kd = false, st_tier = false;
};

tod_status run_knn(tod_ctx* ctx, const float* dX, int64_t n, const float* dQ, int64_t q_begin,
                   int64_t q_count, int d, int k, KnnOutDev out, tod_stats* stats, Timer& tm,
                   int* launches, RefPrep* ref);
// Steps a3-a5 (re-rank + certificate, second tier, fallback, scores, stats)
// for rows whose pass-1 candidates are in `cands` / `mp`; dX holds every
// reference row.  `small` holds the prep globals and the row counters.
tod_status finish_rows(tod_ctx* ctx, const float* dX, int64_t n, const float* dQ, int64_t q_begin,
                       int64_t q_count, int d, int k, const Plan& plan, Cands cands,
                       const MainPass* mp, CertParams cp, SmallDev* small, KnnOutDev out,
                       tod_stats* stats, Timer& tm, int* launches, RefPrep* ref,
                       const PassInfo& pi);
tod_status run_knn_auto(tod_ctx* ctx, const float* dX, int64_t n, const float* dQ, int64_t q_begin,
                        int64_t q_count, int d, int k, KnnOutDev out, tod_stats* stats, Timer& tm,
                        int* launches);
tod_status validate_common(tod_ctx* ctx, int64_t n, int32_t d, int32_t k);
tod_status stage_outputs(tod_ctx* ctx, const tod_knn_out* o, int64_t q, int k, OutStage* s);
tod_status unstage_outputs(tod_ctx* ctx, const tod_knn_out* o, int64_t q, int k, const OutStage& s);
tod_status stage_input(tod_ctx* ctx, const float* user, size_t count, int id, const float** dev);
size_t knn_bytes_per_row(const Plan& p, int k);
void finish_stats(tod_stats* stats, Timer& tm, int launches, int i_lof_end);
void tod_comm_release(tod_ctx* ctx);  // shard.cu: destroy the NCCL communicator

// Resolve a caller buffer: device pointer as is, host pointer -> staging buffer.
template <class T>
tod_status dev_view(tod_ctx* ctx, T* user, size_t count, int id, T** dev, bool* staged) {
  *staged = false;
  if (!user) {
    *dev = nullptr;
    return TOD_OK;
  }
  if (is_device_ptr(user, ctx->device)) {
    *dev = user;
    return TOD_OK;
  }
  void* p;
  TOD_TRY(ensure(ctx, id, count * sizeof(T), &p));
  *dev = static_cast<T*>(p);
  *staged = true;
  return TOD_OK;
}

}  // namespace todapi
