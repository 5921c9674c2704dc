// shard.cu — the sharded multi-GPU path (§6.2 P:475-484:
// "subtasks are split equally", one process per GPU).
//
// Rank r of a world of W processes holds only its row block X_r = rows
// [off_r, off_r + cnt_r) of X (off_r % 256 == 0).  It answers the kNN of its own
// rows (the query shard stays put) while the quantized reference blocks
// circulate around an NCCL ring over NVLink, double-buffered so each transfer
// overlaps the tensor-core pass over the previous block:
//
//   a1  global quantization constants from collectives on tiny data:
//       column partial sums of every rank's 128-row blocks are all-gathered and
//       reduced in global block order (the same mean as one process, bit for
//       bit); max|x - mu|, max ||xhat||^2, max e, the norm-piece residual and the
//       NaN flag are all-reduced with MAX (order-free).  Each rank then
//       quantizes ONLY its own block: the reference image B_r (xhat | norm
//       pieces) and the query image A_r (-2 xhat | constants).
//   a2  ring of 2W steps; at step s rank r holds block b = (r - s) mod W:
//         s <  W: key-only sample pass (running minima accumulate over blocks),
//         s == W: tau = the j-th smallest sample minimum per row,
//         s >= W: append-only main pass (group candidates with GLOBAL indices);
//       while step s computes, block b is sent to rank r+1 and block b-1 is
//       received from rank r-1 on the communication stream.
//   a3+ the exact fp64 re-rank needs the fp32 rows of arbitrary candidates:
//       X is all-gathered once (SURVEY §8(e) option A; 2.56 GB at C4), on the
//       communication stream, overlapped with the ring.  Then re-rank,
//       certificate, second tier and fallback run on the rank's rows exactly as
//       in one process (api.cu finish_rows), and the scores are all-gathered.
//
// Because every returned neighbour set is certified exact (or recomputed in
// fp64), the outputs are bit-identical for every W.
//
// Transports: a real NCCL communicator (libnccl.so.2 loaded with dlopen, so
// the library does not depend on NCCL for single-process use), or a LOOPBACK
// of W virtual ranks in one process on one GPU (testing): the same schedule,
// every collective replaced by device-to-device copies between the virtual
// ranks' buffers.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstddef>
#include <cstring>
#include <vector>

#include "../../include/tod.h"
#include "ctx.h"
#include "internal.h"

using namespace tod;
using namespace todapi;

namespace {

// ------------------------------------------------------------------ NCCL
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

// The process's NCCL: if torch (or anyone) already loaded libnccl.so.2, dlopen
// returns that same library.
const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    auto sym = [&](const char* n) { return dlsym(h, n); };
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(sym("ncclAllGather"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(sym("ncclAllReduce"));
    a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
    a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
    a.ok = a.GetUniqueId && a.CommInitRank && a.CommDestroy && a.AllGather && a.AllReduce &&
           a.Send && a.Recv && a.GroupStart && a.GroupEnd && a.GetErrorString;
    return a;
  }();
  return api;
}

#define TOD_NCCL(call)                                                                   \
  do {                                                                                   \
    ncclResult_t r_ = (call);                                                            \
    if (r_ != ncclSuccess)                                                               \
      return fail(ctx, TOD_E_NCCL, "%s: %s (%s:%d)", #call, nccl().GetErrorString(r_),   \
                  __FILE__, __LINE__);                                                   \
  } while (0)

constexpr int kAlign = 256;  // shard offsets: reference tile (256 rows) boundaries

// loopback all-reduce: tmp[0..count) = max over the W rank slots of tmp
__global__ void k_u64_max_fold(unsigned long long* tmp, size_t count, int W) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  unsigned long long m = tmp[i];
  for (int v = 1; v < W; ++v) m = max(m, tmp[(size_t)v * count + i]);
  tmp[i] = m;
}
cudaError_t launch_u64_max_fold(unsigned long long* tmp, size_t count, int W, cudaStream_t st,
                                int* launches) {
  k_u64_max_fold<<<(unsigned)((count + 255) / 256), 256, 0, st>>>(tmp, count, W);
  *launches += 1;
  return cudaGetLastError();
}

// Balanced split of n rows into W blocks on 256-row boundaries.
void shard_rows(int64_t n, int W, int r, int64_t* off, int64_t* cnt) {
  const int64_t tiles = (n + kAlign - 1) / kAlign;
  const int64_t t0 = tiles * r / W, t1 = tiles * (r + 1) / W;
  const int64_t b = std::min<int64_t>(n, t0 * kAlign), e = std::min<int64_t>(n, t1 * kAlign);
  *off = b;
  *cnt = e - b;
}

// Per (virtual) rank state of one sharded call.
struct RankSt {
  int r = 0;
  int64_t off = 0, cnt = 0;
  const float* Xl = nullptr;  // device, own rows
  Workspace* ws = nullptr;
  SmallDev* small = nullptr;
  Image A, blk[2];
  double* part = nullptr;      // own column partials [nb_own x d]
  MainPass sm, mp;
  float* tau = nullptr;
  CertParams cp{};
  KnnOutDev out{};
  tod_stats st{};
};

enum RankBuf {  // ids inside a rank's Workspace
  R_SMALL = 0, R_IMGA, R_A2A, R_EA, R_BLK0, R_BLK1, R_BA2, R_BE, R_PART, R_SAMP, R_TAU, R_MBUF,
  R_MCNT, R_SEND, R_RECV, R_OUTIDX, R_OUTD64, R_OUTKD, R_OUTKTH, R_OUTMEAN, R_LRD, R_LOF, R_LRD32,
  R_TIER, R_NBUF
};

struct Shard {
  tod_ctx* ctx;
  int W;                     // ranks in the job
  bool loop;                 // loopback: all W ranks live here
  std::vector<RankSt> rk;    // W (loopback) or 1 (this rank)
  std::vector<int64_t> off, cnt;  // block table of all ranks
  int64_t cnt_max = 0;
  int launches = 0;
  cudaStream_t st, cs;       // compute / communication stream
  ncclComm_t comm = nullptr;

  tod_status rens(RankSt& R, int id, size_t bytes, void** p) {
    return ensure_ws(ctx, *R.ws, id, bytes, p);
  }

  // ---- collectives (device buffers)
  // MAX over ranks of `count` uint64 (non-negative doubles order like their bits)
  tod_status allreduce_max_u64(std::vector<unsigned long long*> bufs, size_t count) {
    if (W == 1) return TOD_OK;
    if (!loop) {
      TOD_NCCL(nccl().AllReduce(bufs[0], bufs[0], count, ncclUint64, ncclMax, comm, st));
      return TOD_OK;
    }
    // loopback: fold every rank into rank 0, then broadcast back (max is order-free)
    void* p;
    TOD_TRY(ensure(ctx, B_GATHER2, count * 8 * W, &p));
    unsigned long long* tmp = static_cast<unsigned long long*>(p);
    for (int v = 0; v < W; ++v)
      TOD_CUDA(cudaMemcpyAsync(tmp + v * count, bufs[v], count * 8, cudaMemcpyDeviceToDevice, st));
    TOD_CUDA(launch_u64_max_fold(tmp, count, W, st, &launches));
    for (int v = 0; v < W; ++v)
      TOD_CUDA(cudaMemcpyAsync(bufs[v], tmp, count * 8, cudaMemcpyDeviceToDevice, st));
    return TOD_OK;
  }

  // Gather per-rank row blocks (rows_r = cnt_r or a per-rank count) of
  // row_bytes each into `all` in rank order.  send[v] are the local blocks of
  // the ranks living here.
  tod_status allgather_rows(const std::vector<const void*>& send, const std::vector<int64_t>& rows,
                            size_t row_bytes, void* all, cudaStream_t stream,
                            int id_send = B_GATHER, int id_recv = B_GATHER2) {
    std::vector<int64_t> pre(W + 1, 0);
    for (int v = 0; v < W; ++v) pre[v + 1] = pre[v] + rows[v];
    char* dst = static_cast<char*>(all);
    if (loop || W == 1) {
      for (int v = 0; v < W; ++v)
        if (rows[v] > 0 && send[v] != dst + pre[v] * row_bytes)
          TOD_CUDA(cudaMemcpyAsync(dst + pre[v] * row_bytes, send[v], rows[v] * row_bytes,
                                   cudaMemcpyDeviceToDevice, stream));
      return TOD_OK;
    }
    int64_t mx = 0;
    for (int v = 0; v < W; ++v) mx = std::max(mx, rows[v]);
    const size_t slot = (size_t)std::max<int64_t>(mx, 1) * row_bytes;
    void *ps, *pr;
    TOD_TRY(ensure(ctx, id_send, slot, &ps));
    TOD_TRY(ensure(ctx, id_recv, slot * W, &pr));
    const int me = rk[0].r;
    if (rows[me] > 0)
      TOD_CUDA(cudaMemcpyAsync(ps, send[0], rows[me] * row_bytes, cudaMemcpyDeviceToDevice, stream));
    TOD_NCCL(nccl().AllGather(ps, pr, slot, ncclUint8, comm, stream));
    for (int v = 0; v < W; ++v)
      if (rows[v] > 0)
        TOD_CUDA(cudaMemcpyAsync(dst + pre[v] * row_bytes, static_cast<char*>(pr) + v * slot,
                                 rows[v] * row_bytes, cudaMemcpyDeviceToDevice, stream));
    return TOD_OK;
  }
};

}  // namespace

namespace todapi {

// ------------------------------------------------------------------ the call
// One sharded kNN; X_local: this rank's rows (loopback: all of
// X); out: this rank's rows (loopback: all rows).  Scores of ALL rows are
// gathered into kth_all / mean_all when non-null (device pointers).
tod_status run_sharded(tod_ctx* ctx, const float* dXl, int64_t n_local, int64_t row_offset,
                       int64_t n, int d, int k, KnnOutDev out_local, float* kth_all,
                       float* mean_all, double* kd_all, tod_stats* stats, Timer& tm, int* launches,
                       std::vector<RankSt>* keep) {
  Shard sh;
  sh.ctx = ctx;
  sh.W = ctx->world;
  sh.loop = ctx->loopback != 0;
  sh.st = ctx->stream;
  sh.cs = (sh.loop || sh.W == 1 || !ctx->comm_stream) ? ctx->stream : ctx->comm_stream;
  sh.comm = static_cast<ncclComm_t>(ctx->nccl_comm);
  const int W = sh.W;
  cudaStream_t st = sh.st;
  void* p;

  // ---- block table
  sh.off.assign(W, 0);
  sh.cnt.assign(W, 0);
  if (sh.loop || W == 1) {
    if (row_offset != 0 || n_local != n)
      return fail(ctx, TOD_E_ARG, "loopback / single-rank sharded call takes all rows (row_offset 0, n_local n)");
    for (int v = 0; v < W; ++v) shard_rows(n, W, v, &sh.off[v], &sh.cnt[v]);
  } else {
    // every rank reports (row_offset, n_local); the table must tile [0, n) in rank order
    TOD_TRY(ensure(ctx, B_SHTAB, (size_t)W * 16 + 16, &p));
    int64_t* dtab = static_cast<int64_t*>(p);
    int64_t mine[2] = {row_offset, n_local};
    TOD_CUDA(cudaMemcpyAsync(dtab + 2 * W, mine, 16, cudaMemcpyHostToDevice, st));
    TOD_NCCL(nccl().AllGather(dtab + 2 * W, dtab, 2, ncclInt64, sh.comm, st));
    std::vector<int64_t> tab(2 * W);
    TOD_CUDA(cudaMemcpyAsync(tab.data(), dtab, (size_t)W * 16, cudaMemcpyDeviceToHost, st));
    TOD_CUDA(cudaStreamSynchronize(st));
    for (int v = 0; v < W; ++v) {
      sh.off[v] = tab[2 * v];
      sh.cnt[v] = tab[2 * v + 1];
    }
  }
  int64_t expect = 0;
  for (int v = 0; v < W; ++v) {
    if (sh.off[v] != expect || sh.cnt[v] < 0 || (sh.off[v] % kAlign) != 0)
      return fail(ctx, TOD_E_ARG, "rank %d rows [%lld, +%lld): shards must tile [0, n) in rank order "
                  "on %d-row boundaries (tod_shard_rows)", v, (long long)sh.off[v],
                  (long long)sh.cnt[v], kAlign);
    expect += sh.cnt[v];
    sh.cnt_max = std::max(sh.cnt_max, sh.cnt[v]);
  }
  if (expect != n) return fail(ctx, TOD_E_ARG, "shards cover %lld rows, n = %lld", (long long)expect, (long long)n);

  // ---- rank states
  const int nloc = sh.loop ? W : 1;
  if ((int)ctx->rank_ws.size() < nloc) ctx->rank_ws.resize(nloc);
  sh.rk.resize(nloc);
  for (int i = 0; i < nloc; ++i) {
    RankSt& R = sh.rk[i];
    R.r = sh.loop ? i : ctx->rank;
    R.off = sh.off[R.r];
    R.cnt = sh.cnt[R.r];
    R.Xl = sh.loop ? dXl + R.off * d : dXl;
    R.ws = &ctx->rank_ws[i];
    R.out = out_local;
    if (sh.loop) {  // slice of the all-rows output
      auto shf = [&](auto* q, int64_t per) { return q ? q + R.off * per : q; };
      R.out.idx = shf(out_local.idx, k);
      R.out.dist = shf(out_local.dist, k);
      R.out.dist64 = shf(out_local.dist64, k);
      R.out.score_kth = shf(out_local.score_kth, 1);
      R.out.score_mean = shf(out_local.score_mean, 1);
      R.out.kdist64 = shf(out_local.kdist64, 1);
      R.out.tier = shf(out_local.tier, 1);
    }
    TOD_TRY(sh.rens(R, R_SMALL, sizeof(SmallDev), &p));
    R.small = static_cast<SmallDev*>(p);
    TOD_CUDA(cudaMemsetAsync(R.small, 0, sizeof(SmallDev), st));
  }

  Plan plan;
  TOD_TRY(make_plan(ctx, n, std::max<int64_t>(sh.cnt_max, 1), d, k, &plan));
  const bool ring = plan.kind == PASS_TC && plan.two && tc3_fits(plan.dpad);

  // ---- X all-gather (re-rank / fallback need the fp32 rows of any candidate:
  // SURVEY §8(e) option A).  On the communication stream, after the last
  // collective of the compute stream, so no two NCCL operations of the
  // communicator are ever in flight at once; it overlaps the ring's compute.
  const float* dXall = dXl;
  cudaEvent_t ev_x = nullptr;
  auto gather_x = [&]() -> tod_status {
    if (W == 1) return TOD_OK;
    TOD_TRY(ensure(ctx, B_XALL, (size_t)n * d * 4, &p));
    float* xa = static_cast<float*>(p);
    if (!sh.loop) {
      TOD_CUDA(cudaEventCreateWithFlags(&ev_x, cudaEventDisableTiming));
      cudaEvent_t ev0;
      TOD_CUDA(cudaEventCreateWithFlags(&ev0, cudaEventDisableTiming));
      TOD_CUDA(cudaEventRecord(ev0, st));
      TOD_CUDA(cudaStreamWaitEvent(sh.cs, ev0, 0));
      cudaEventDestroy(ev0);
      std::vector<const void*> send = {dXl};
      TOD_TRY(sh.allgather_rows(send, sh.cnt, (size_t)d * 4, xa, sh.cs, B_XSEND, B_XSLOT));
      TOD_CUDA(cudaEventRecord(ev_x, sh.cs));
    } else {
      // loopback: the virtual ranks' slices are gathered into a separate buffer
      // too, so the re-rank reads the gathered copy exactly as a real rank does
      std::vector<const void*> send(W);
      for (int v = 0; v < W; ++v) send[v] = sh.rk[v].Xl;
      TOD_TRY(sh.allgather_rows(send, sh.cnt, (size_t)d * 4, xa, st));
    }
    dXall = xa;
    return TOD_OK;
  };

  tm.mark();  // 1: prep
  if (!ring) {
    // Small or non-tensor-core problems: the replicated reference (every rank
    // answers its rows against all of X) -- no ring.
    TOD_TRY(gather_x());
    if (ev_x) TOD_CUDA(cudaStreamWaitEvent(st, ev_x, 0));
    tm.mark();  // 2
    tm.mark();  // 3
    tod_stats acc{};
    for (auto& R : sh.rk) {
      Timer off{ctx, false};
      tod_stats rs{};
      if (R.cnt > 0)
        TOD_TRY(run_knn_auto(ctx, dXall, n, nullptr, R.off, R.cnt, d, k, R.out, &rs, off, launches));
      acc.rows += rs.rows;
      acc.certified += rs.certified;
      acc.fallback_rows += rs.fallback_rows;
      acc.kprime = rs.kprime;
      acc.format = rs.format;
      acc.dpad = rs.dpad;
      acc.scale = rs.scale;
      acc.max_abs_err = std::max(acc.max_abs_err, rs.max_abs_err);
      R.st = rs;
    }
    tm.mark();  // 4
    tm.mark();  // 5
    if (stats) *stats = acc;
  } else {
    // ---------------------------------------------------------------- a1
    const int srows = prep_stat_rows();
    const int nb_all = (int)((n + srows - 1) / srows);
    TOD_TRY(ensure(ctx, B_MU, (size_t)d * 8 * nloc, &p));
    double* mu_base = static_cast<double*>(p);
    TOD_TRY(ensure(ctx, B_PARTALL, (size_t)nb_all * d * 8, &p));
    double* part_all = static_cast<double*>(p);
    std::vector<const void*> psend(nloc);
    std::vector<int64_t> prow(W);
    for (int v = 0; v < W; ++v) prow[v] = (sh.cnt[v] + srows - 1) / srows;
    for (int i = 0; i < nloc; ++i) {
      RankSt& R = sh.rk[i];
      TOD_TRY(sh.rens(R, R_PART, (size_t)std::max<int64_t>(prow[R.r], 1) * d * 8, &p));
      R.part = static_cast<double*>(p);
      TOD_CUDA(launch_prep_colsum(R.Xl, R.cnt, d, R.part, &R.small->g, st, launches));
      psend[i] = R.part;
    }
    // partials in global block order (every shard but the last is a whole number of blocks)
    TOD_TRY(sh.allgather_rows(psend, prow, (size_t)d * 8, part_all, st));
    std::vector<unsigned long long*> gbits(nloc);
    for (int i = 0; i < nloc; ++i) {
      RankSt& R = sh.rk[i];
      double* mu = mu_base + (size_t)i * d;
      TOD_CUDA(launch_prep_colmean(part_all, nb_all, n, d, mu, st, launches));
      TOD_CUDA(launch_prep_absmax(R.Xl, R.cnt, d, mu, &R.small->g, st, launches));
    }
    // max|x - mu| and the NaN flag: order-free MAX over ranks
    static_assert(offsetof(PrepGlobals, nonfinite) == offsetof(PrepGlobals, absmax_bits) + 8,
                  "absmax_bits and nonfinite are reduced together");
    for (int i = 0; i < nloc; ++i)
      gbits[i] = reinterpret_cast<unsigned long long*>(&sh.rk[i].small->g.absmax_bits);
    TOD_TRY(sh.allreduce_max_u64(gbits, 2));
    const int64_t blk_pad = (sh.cnt_max + 255) / 256 * 256;
    auto init_img = [&](Image& im, int64_t rows, int64_t rows_pad) {
      im.n = rows;
      im.n_pad = rows_pad;
      im.dpad = plan.dpad;
      im.rb = std::min(128, plan.dpad * 2);
      im.nkb = plan.dpad * 2 / im.rb;
      im.layout = im.rb == 128 ? 2 : (im.rb == 64 ? 4 : 6);
    };
    for (int i = 0; i < nloc; ++i) {
      RankSt& R = sh.rk[i];
      double* mu = mu_base + (size_t)i * d;
      TOD_CUDA(launch_prep_scale(&R.small->g, plan.fmt, plan.dpad, st, launches));
      // own reference block (ring buffer 0) and own query image
      for (int b = 0; b < 2; ++b) {
        init_img(R.blk[b], R.cnt, blk_pad);
        TOD_TRY(sh.rens(R, b ? R_BLK1 : R_BLK0, R.blk[b].total_bytes(), &p));
        R.blk[b].data = static_cast<uint16_t*>(p);
      }
      TOD_TRY(sh.rens(R, R_BA2, (size_t)blk_pad * 8, &p));
      R.blk[0].a2 = static_cast<double*>(p);
      TOD_TRY(sh.rens(R, R_BE, (size_t)blk_pad * 8, &p));
      R.blk[0].e = static_cast<double*>(p);
      TOD_CUDA(launch_prep_quant(R.Xl, R.cnt, d, mu, &R.small->g, plan.fmt, R.blk[0], 0, st, launches));
      init_img(R.A, R.cnt, std::max<int64_t>(256, (R.cnt + 255) / 256 * 256));
      TOD_TRY(sh.rens(R, R_IMGA, R.A.total_bytes(), &p));
      R.A.data = static_cast<uint16_t*>(p);
      TOD_TRY(sh.rens(R, R_A2A, (size_t)std::max<int64_t>(R.cnt, 1) * 8, &p));
      R.A.a2 = static_cast<double*>(p);
      TOD_TRY(sh.rens(R, R_EA, (size_t)std::max<int64_t>(R.cnt, 1) * 8, &p));
      R.A.e = static_cast<double*>(p);
      TOD_CUDA(launch_prep_quant(R.Xl, R.cnt, d, mu, &R.small->g, plan.fmt, R.A, 1, st, launches));
    }
    // amax2, emax, repmax: order-free MAX over ranks
    static_assert(offsetof(PrepGlobals, emax) == offsetof(PrepGlobals, amax2) + 8 &&
                  offsetof(PrepGlobals, repmax) == offsetof(PrepGlobals, amax2) + 16,
                  "amax2, emax and repmax are reduced together");
    for (int i = 0; i < nloc; ++i)
      gbits[i] = reinterpret_cast<unsigned long long*>(&sh.rk[i].small->g.amax2);
    TOD_TRY(sh.allreduce_max_u64(gbits, 3));
    TOD_TRY(gather_x());

    // ---------------------------------------------------------------- a2
    tm.mark();  // 2: ring
    const int parts = tc3_parts(plan.dpad);
    const int jw = std::max(4, (2 * plan.kp_target + plan.R - 1) / plan.R);
    const int samp_t = jw > 3 * parts ? 8 : 4;
    const int nv = parts * samp_t;
    const char* pe = getenv("TOD_MAIN_PAIR");
    const bool pair = (pe ? atoi(pe) != 0 : tc4_preferred(plan.dpad) != 0) &&
                      !(ctx->cfg.flags & TOD_F_MAIN_1SM) && tc4_fits(plan.dpad, parts);
    const double blk_bytes = (double)blk_pad * (plan.dpad + 16) * 2;
    const int blk_S = std::max(1, (int)std::ceil(blk_bytes / (48.0 * 1024 * 1024)));
    for (int i = 0; i < nloc; ++i) {
      RankSt& R = sh.rk[i];
      const int64_t q = std::max<int64_t>(R.cnt, 1);
      R.sm.S = 1;
      R.sm.R = plan.R;
      R.sm.parts = parts;
      R.sm.samp_t = samp_t;
      TOD_TRY(sh.rens(R, R_SAMP, (size_t)q * nv * 4, &p));
      R.sm.samp = static_cast<float*>(p);
      TOD_TRY(sh.rens(R, R_TAU, (size_t)q * 4, &p));
      R.tau = static_cast<float*>(p);
      R.mp.S = blk_S;
      R.mp.R = 0;
      R.mp.tau_v = R.tau;
      R.mp.tau_lists = 1;
      R.mp.parts = parts;
      R.mp.cap = plan.cap * 2 / parts;
      R.mp.vote = main_vote(n);
      TOD_TRY(sh.rens(R, R_MBUF, (size_t)q * parts * R.mp.cap * 8, &p));
      R.mp.buf = static_cast<uint2*>(p);
      TOD_TRY(sh.rens(R, R_MCNT, (size_t)q * parts * 4, &p));
      R.mp.cnt = static_cast<int*>(p);
      TOD_CUDA(cudaMemsetAsync(R.mp.cnt, 0, (size_t)q * parts * 4, st));
    }
    cudaEvent_t ev_done[2] = {}, ev_recv[2] = {};
    const bool async = !sh.loop && W > 1;
    if (async) {
      for (int b = 0; b < 2; ++b) {
        TOD_CUDA(cudaEventCreateWithFlags(&ev_done[b], cudaEventDisableTiming));
        TOD_CUDA(cudaEventCreateWithFlags(&ev_recv[b], cudaEventDisableTiming));
      }
      TOD_CUDA(cudaEventRecord(ev_done[1], st));  // prep done: buffer 0 holds the own block
    }
    const size_t xfer = sh.rk[0].blk[0].total_bytes();
    for (int s = 0; s < 2 * W; ++s) {
      const int cur = s & 1, nxt = cur ^ 1;
      // post the transfer for step s+1 (send the block in hand onward, receive the previous rank's)
      if (s + 1 < 2 * W && W > 1) {
        if (async) {
          RankSt& R = sh.rk[0];
          TOD_CUDA(cudaStreamWaitEvent(sh.cs, ev_done[nxt], 0));  // step s-1 finished reading nxt
          TOD_NCCL(nccl().GroupStart());
          TOD_NCCL(nccl().Send(R.blk[cur].data, xfer, ncclUint8, (R.r + 1) % W, sh.comm, sh.cs));
          TOD_NCCL(nccl().Recv(R.blk[nxt].data, xfer, ncclUint8, (R.r + W - 1) % W, sh.comm, sh.cs));
          TOD_NCCL(nccl().GroupEnd());
          TOD_CUDA(cudaEventRecord(ev_recv[nxt], sh.cs));
        }
      }
      if (s == W) {  // sample ring done: per-row threshold
        for (auto& R : sh.rk)
          if (R.cnt > 0)
            TOD_CUDA(launch_tau_combine(R.cnt, nv, std::min(nv, jw), R.sm.samp, R.tau, st, launches));
        if (tm.on) cudaEventRecord(ctx->evk[0], st);
      }
      if (async && s > 0) TOD_CUDA(cudaStreamWaitEvent(st, ev_recv[cur], 0));
      for (auto& R : sh.rk) {
        const int b = (int)(((R.r - s) % W + W) % W);  // block in hand at step s
        Image B = R.blk[cur];
        B.n = sh.cnt[b];
        if (R.cnt > 0 && B.n > 0) {
          if (s < W) {
            MainPass m = R.sm;
            m.col0 = sh.off[b];
            m.samp_acc = s > 0;
            TOD_CUDA(launch_knn_tc3(R.A, B, R.off, R.cnt, true, plan.fmt, m, ctx->num_sms, 0, st,
                                    launches));
          } else {
            MainPass m = R.mp;
            m.col0 = sh.off[b];
            if (pair)
              TOD_CUDA(launch_knn_tc4(R.A, B, R.off, R.cnt, true, plan.fmt, m, ctx->num_sms, 0, st,
                                      launches));
            else
              TOD_CUDA(launch_knn_tc3(R.A, B, R.off, R.cnt, true, plan.fmt, m, ctx->num_sms, 0, st,
                                      launches));
          }
        }
      }
      if (async) TOD_CUDA(cudaEventRecord(ev_done[cur], st));
      // loopback transport: rank v receives rank v-1's block (all on one stream)
      if (sh.loop && W > 1 && s + 1 < 2 * W)
        for (int v = 0; v < W; ++v)
          TOD_CUDA(cudaMemcpyAsync(sh.rk[v].blk[nxt].data, sh.rk[(v + W - 1) % W].blk[cur].data,
                                   xfer, cudaMemcpyDeviceToDevice, st));
    }
    if (tm.on) cudaEventRecord(ctx->evk[1], st);
    if (async) {
      for (int b = 0; b < 2; ++b) {
        cudaEventDestroy(ev_done[b]);
        cudaEventDestroy(ev_recv[b]);
      }
    }
    // -------------------------------------------------------- a3 .. a5
    if (ev_x) TOD_CUDA(cudaStreamWaitEvent(st, ev_x, 0));
    tm.mark();  // 3: certify
    tod_stats acc{};
    for (int i = 0; i < nloc; ++i) {
      RankSt& R = sh.rk[i];
      if (R.cnt == 0) continue;
      Cands c;
      c.v = R.tau;
      c.key = R.tau;  // no pass-1 lists (kp = 0): never read, must be non-null
      c.idx = reinterpret_cast<int32_t*>(R.tau);
      c.lists = 1;
      c.kp = 0;
      c.S = plan.S;
      c.R = plan.R;
      CertParams cp{};
      cp.kind = PASS_TC;
      cp.d = d;
      cp.dpad = plan.dpad;
      cp.s = 1.0;
      cp.g = &R.small->g;
      cp.qa2 = R.A.a2;
      cp.qe = R.A.e;
      cp.force_fail = (ctx->cfg.flags & TOD_F_NO_CERTIFY) ? 1 : 0;
      PassInfo pi;
      pi.main_kernel = pair ? 4 : 3;
      pi.sample_pass = 2;
      pi.main_timed = false;
      RefPrep ref;
      ref.ready = false;
      Timer off{ctx, false};
      tod_stats rs{};
      TOD_TRY(finish_rows(ctx, dXall, n, nullptr, R.off, R.cnt, d, k, plan, c, &R.mp, cp, R.small,
                          R.out, &rs, off, launches, &ref, pi));
      acc.rows += rs.rows;
      acc.certified += rs.certified;
      acc.fallback_rows += rs.fallback_rows;
      acc.cand_groups += rs.cand_groups;
      acc.visited_groups += rs.visited_groups;
      acc.cand_columns += rs.cand_columns;
      acc.max_abs_err = std::max(acc.max_abs_err, rs.max_abs_err);
      acc.kprime = rs.kprime;
      acc.format = rs.format;
      acc.chunks = blk_S;
      acc.dpad = rs.dpad;
      acc.scale = rs.scale;
      acc.main_kernel = rs.main_kernel;
      acc.sample_pass = 2;
      R.st = rs;
    }
    tm.mark();  // 4
    tm.mark();  // 5
    if (stats) {
      *stats = acc;
      if (tm.on) cudaEventElapsedTime(&stats->ms_main_kernel, ctx->evk[0], ctx->evk[1]);
    }
  }
  if (ev_x) cudaEventDestroy(ev_x);

  // ---- gathered per-row outputs of every rank
  auto gather = [&](float* all, float* KnnOutDev::*field) -> tod_status {
    if (!all) return TOD_OK;
    std::vector<const void*> send(nloc);
    for (int i = 0; i < nloc; ++i) send[i] = sh.rk[i].out.*field;
    return sh.allgather_rows(send, sh.cnt, 4, all, st);
  };
  TOD_TRY(gather(kth_all, &KnnOutDev::score_kth));
  TOD_TRY(gather(mean_all, &KnnOutDev::score_mean));
  if (kd_all) {
    std::vector<const void*> send(nloc);
    for (int i = 0; i < nloc; ++i) send[i] = sh.rk[i].out.kdist64;
    TOD_TRY(sh.allgather_rows(send, sh.cnt, 8, kd_all, st));
  }
  if (stats) stats->rows = sh.loop ? n : n_local;
  *launches += sh.launches;
  if (keep) *keep = sh.rk;
  return TOD_OK;
}

// LOF stages over the shards (after run_sharded): all-gather kdist64, lrd of
// own rows, all-gather lrd64, LOF of own rows, all-gather LOF / lrd (fp32).
tod_status lof_sharded_tail(tod_ctx* ctx, std::vector<RankSt>& rk, int64_t n, int k,
                            const double* kd_all, float* lof_all, float* lrd_all, int* launches) {
  Shard sh;
  sh.ctx = ctx;
  sh.W = ctx->world;
  sh.loop = ctx->loopback != 0;
  sh.st = ctx->stream;
  sh.cs = ctx->stream;
  sh.comm = static_cast<ncclComm_t>(ctx->nccl_comm);
  sh.rk = rk;
  sh.off.assign(sh.W, 0);
  sh.cnt.assign(sh.W, 0);
  for (int v = 0; v < sh.W; ++v) shard_rows(n, sh.W, v, &sh.off[v], &sh.cnt[v]);
  if (!sh.loop && sh.W > 1) {  // the real table (validated by run_sharded)
    // ranks' counts: rk[0] is this rank; others follow tod_shard_rows only if the
    // caller used it -- gather the counts to be safe
    void* p;
    TOD_TRY(ensure(ctx, B_SHTAB, (size_t)sh.W * 16 + 16, &p));
    int64_t* dtab = static_cast<int64_t*>(p);
    int64_t mine[2] = {rk[0].off, rk[0].cnt};
    TOD_CUDA(cudaMemcpyAsync(dtab + 2 * sh.W, mine, 16, cudaMemcpyHostToDevice, sh.st));
    TOD_NCCL(nccl().AllGather(dtab + 2 * sh.W, dtab, 2, ncclInt64, sh.comm, sh.st));
    std::vector<int64_t> tab(2 * sh.W);
    TOD_CUDA(cudaMemcpyAsync(tab.data(), dtab, (size_t)sh.W * 16, cudaMemcpyDeviceToHost, sh.st));
    TOD_CUDA(cudaStreamSynchronize(sh.st));
    for (int v = 0; v < sh.W; ++v) {
      sh.off[v] = tab[2 * v];
      sh.cnt[v] = tab[2 * v + 1];
    }
  }
  cudaStream_t st = sh.st;
  void* p;
  TOD_TRY(ensure(ctx, B_LRD64, (size_t)n * 8, &p));
  double* lrd_all64 = static_cast<double*>(p);
  std::vector<const void*> s_lrd(rk.size()), s_lof(rk.size()), s_lrd32(rk.size());
  for (size_t i = 0; i < rk.size(); ++i) {
    RankSt& R = rk[i];
    const int64_t q = std::max<int64_t>(R.cnt, 1);
    TOD_TRY(sh.rens(R, R_LRD, (size_t)q * 8, &p));
    double* lrd = static_cast<double*>(p);
    if (R.cnt > 0)
      TOD_CUDA(launch_lof_lrd(R.cnt, k, R.out.idx, R.out.dist64, kd_all, lrd, st, launches));
    s_lrd[i] = lrd;
  }
  TOD_TRY(sh.allgather_rows(s_lrd, sh.cnt, 8, lrd_all64, st));
  for (size_t i = 0; i < rk.size(); ++i) {
    RankSt& R = rk[i];
    const int64_t q = std::max<int64_t>(R.cnt, 1);
    TOD_TRY(sh.rens(R, R_LOF, (size_t)q * 4, &p));
    float* lof = static_cast<float*>(p);
    TOD_TRY(sh.rens(R, R_LRD32, (size_t)q * 4, &p));
    float* lrd32 = static_cast<float*>(p);
    if (R.cnt > 0)
      TOD_CUDA(launch_lof_finish(R.off, R.cnt, k, R.out.idx, lrd_all64, lof, lrd32, st, launches));
    s_lof[i] = lof;
    s_lrd32[i] = lrd32;
  }
  if (lof_all) TOD_TRY(sh.allgather_rows(s_lof, sh.cnt, 4, lof_all, st));
  if (lrd_all) TOD_TRY(sh.allgather_rows(s_lrd32, sh.cnt, 4, lrd_all, st));
  *launches += sh.launches;
  return TOD_OK;
}

void tod_comm_release(tod_ctx* ctx) {
  if (ctx->nccl_comm && nccl().ok) nccl().CommDestroy(static_cast<ncclComm_t>(ctx->nccl_comm));
  ctx->nccl_comm = nullptr;
}

}  // namespace todapi

extern "C" {

tod_status tod_shard_rows(int64_t n, int32_t world, int32_t rank, int64_t* row_offset,
                          int64_t* n_local) {
  if (n < 0 || world < 1 || rank < 0 || rank >= world || !row_offset || !n_local) return TOD_E_ARG;
  shard_rows(n, world, rank, row_offset, n_local);
  return TOD_OK;
}

tod_status tod_comm_id_create(tod_comm_id* id) {
  if (!id) return TOD_E_ARG;
  static_assert(sizeof(tod_comm_id) == sizeof(ncclUniqueId), "tod_comm_id must hold an ncclUniqueId");
  if (!nccl().ok) return TOD_E_NCCL;
  ncclUniqueId u;
  if (nccl().GetUniqueId(&u) != ncclSuccess) return TOD_E_NCCL;
  memcpy(id, &u, sizeof u);
  return TOD_OK;
}

tod_status tod_comm_init(tod_ctx* ctx, const tod_comm_id* id, int32_t rank, int32_t world) {
  if (!ctx) return TOD_E_ARG;
  if (!id || world < 1 || rank < 0 || rank >= world)
    return fail(ctx, TOD_E_ARG, "bad rank %d / world %d", rank, world);
  if (ctx->nccl_comm || ctx->loopback) return fail(ctx, TOD_E_ARG, "context already has a communicator");
  TOD_CUDA(cudaSetDevice(ctx->device));
  if (!nccl().ok) return fail(ctx, TOD_E_NCCL, "libnccl.so.2 not found or incomplete");
  ncclUniqueId u;
  memcpy(&u, id, sizeof u);
  ncclComm_t c = nullptr;
  TOD_NCCL(nccl().CommInitRank(&c, world, u, rank));
  ctx->nccl_comm = c;
  ctx->rank = rank;
  ctx->world = world;
  if (!ctx->comm_stream)
    TOD_CUDA(cudaStreamCreateWithFlags(&ctx->comm_stream, cudaStreamNonBlocking));
  return TOD_OK;
}

tod_status tod_comm_init_loopback(tod_ctx* ctx, int32_t world) {
  if (!ctx) return TOD_E_ARG;
  if (world < 1) return fail(ctx, TOD_E_ARG, "bad world %d", world);
  if (ctx->nccl_comm) return fail(ctx, TOD_E_ARG, "context already has an NCCL communicator");
  ctx->loopback = 1;
  ctx->rank = 0;
  ctx->world = world;
  return TOD_OK;
}

tod_status tod_knn_sharded(tod_ctx* ctx, const float* X_local, int64_t n_local, int64_t row_offset,
                           int64_t n, int32_t d, int32_t k, const tod_knn_out* out,
                           float* score_kth_all, float* score_mean_all, tod_stats* stats) {
  TOD_TRY(validate_common(ctx, n, d, k));
  if (n < 2 || k > n - 1) return fail(ctx, TOD_E_RANGE, "need 1 <= k <= n-1 (n=%lld k=%d)", (long long)n, k);
  if (n_local < 0 || row_offset < 0 || row_offset + n_local > n)
    return fail(ctx, TOD_E_RANGE, "rows [%lld, +%lld) outside [0, %lld)", (long long)row_offset,
                (long long)n_local, (long long)n);
  TOD_CUDA(cudaSetDevice(ctx->device));
  if (stats) memset(stats, 0, sizeof *stats);
  Timer tm{ctx, (ctx->cfg.flags & TOD_F_TIMING) != 0};
  int launches = 0;
  tm.mark();  // 0
  const float* dX;
  TOD_TRY(stage_input(ctx, X_local, (size_t)n_local * d, B_X, &dX));
  OutStage os;
  TOD_TRY(stage_outputs(ctx, out, n_local, k, &os));
  float *dk = nullptr, *dm = nullptr;
  bool st_k = false, st_m = false;
  TOD_TRY(dev_view(ctx, score_kth_all, (size_t)n, B_KTH, &dk, &st_k));
  TOD_TRY(dev_view(ctx, score_mean_all, (size_t)n, B_MEAN, &dm, &st_m));
  // gathering a score needs the local score
  void* p;
  if (dk && !os.dev.score_kth) {
    TOD_TRY(ensure(ctx, B_LRD32, (size_t)std::max<int64_t>(n_local, 1) * 4, &p));
    os.dev.score_kth = static_cast<float*>(p);
  }
  if (dm && !os.dev.score_mean) {
    TOD_TRY(ensure(ctx, B_LOF, (size_t)std::max<int64_t>(n_local, 1) * 4, &p));
    os.dev.score_mean = static_cast<float*>(p);
  }
  TOD_TRY(run_sharded(ctx, dX, n_local, row_offset, n, d, k, os.dev, dk, dm, nullptr, stats, tm,
                      &launches, nullptr));
  TOD_TRY(unstage_outputs(ctx, out, n_local, k, os));
  if (st_k) TOD_CUDA(cudaMemcpyAsync(score_kth_all, dk, (size_t)n * 4, cudaMemcpyDeviceToHost, ctx->stream));
  if (st_m) TOD_CUDA(cudaMemcpyAsync(score_mean_all, dm, (size_t)n * 4, cudaMemcpyDeviceToHost, ctx->stream));
  tm.mark();
  TOD_CUDA(cudaStreamSynchronize(ctx->stream));
  finish_stats(stats, tm, launches, 0);
  ctx->msg.clear();
  return TOD_OK;
}

tod_status tod_lof_sharded(tod_ctx* ctx, const float* X_local, int64_t n_local, int64_t row_offset,
                           int64_t n, int32_t d, int32_t k, float* lof_all, float* lrd_all,
                           const tod_knn_out* out, tod_stats* stats) {
  TOD_TRY(validate_common(ctx, n, d, k));
  if (n < 2 || k > n - 1) return fail(ctx, TOD_E_RANGE, "need 1 <= k <= n-1 (n=%lld k=%d)", (long long)n, k);
  if (n_local < 0 || row_offset < 0 || row_offset + n_local > n)
    return fail(ctx, TOD_E_RANGE, "rows outside [0, n)");
  TOD_CUDA(cudaSetDevice(ctx->device));
  if (stats) memset(stats, 0, sizeof *stats);
  Timer tm{ctx, (ctx->cfg.flags & TOD_F_TIMING) != 0};
  int launches = 0;
  tm.mark();
  const float* dX;
  TOD_TRY(stage_input(ctx, X_local, (size_t)n_local * d, B_X, &dX));
  OutStage os;
  TOD_TRY(stage_outputs(ctx, out, n_local, k, &os));
  void* p;
  // LOF needs idx, dist64 and kdist64 of the local rows on the device
  if (!os.dev.idx) {
    TOD_TRY(ensure(ctx, B_IDX, (size_t)std::max<int64_t>(n_local, 1) * k * 8, &p));
    os.dev.idx = static_cast<int64_t*>(p);
  }
  if (!os.dev.dist64) {
    TOD_TRY(ensure(ctx, B_DIST64, (size_t)std::max<int64_t>(n_local, 1) * k * 8, &p));
    os.dev.dist64 = static_cast<double*>(p);
  }
  if (!os.dev.kdist64) {
    TOD_TRY(ensure(ctx, B_KD64, (size_t)std::max<int64_t>(n_local, 1) * 8, &p));
    os.dev.kdist64 = static_cast<double*>(p);
  }
  TOD_TRY(ensure(ctx, B_KDALL, (size_t)n * 8, &p));
  double* kd_all = static_cast<double*>(p);
  float *dlof, *dlrd;
  bool st_lof, st_lrd;
  TOD_TRY(dev_view(ctx, lof_all, (size_t)n, B_ABOD, &dlof, &st_lof));
  TOD_TRY(dev_view(ctx, lrd_all, (size_t)n, B_PRED, &dlrd, &st_lrd));
  std::vector<RankSt> rk;
  TOD_TRY(run_sharded(ctx, dX, n_local, row_offset, n, d, k, os.dev, nullptr, nullptr, kd_all, stats,
                      tm, &launches, &rk));
  TOD_TRY(lof_sharded_tail(ctx, rk, n, k, kd_all, dlof, dlrd, &launches));
  tm.mark();  // 6: LOF end
  TOD_TRY(unstage_outputs(ctx, out, n_local, k, os));
  if (st_lof) TOD_CUDA(cudaMemcpyAsync(lof_all, dlof, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
  if (st_lrd) TOD_CUDA(cudaMemcpyAsync(lrd_all, dlrd, n * 4, cudaMemcpyDeviceToHost, ctx->stream));
  tm.mark();
  TOD_CUDA(cudaStreamSynchronize(ctx->stream));
  finish_stats(stats, tm, launches, 6);
  ctx->msg.clear();
  return TOD_OK;
}

size_t tod_workspace_size(int64_t n, int32_t d, int32_t k, int64_t q_count, const tod_config* cfg) {
  if (n < 2 || d < 1 || k < 1 || q_count < 0) return 0;
  tod_ctx tmp;
  if (cfg) tmp.cfg = *cfg;
  tmp.num_sms = 148;
  Plan plan;
  if (make_plan(&tmp, n, std::max<int64_t>(q_count, 1), d, k, &plan) != TOD_OK) return 0;
  size_t b = knn_bytes_per_row(plan, k) * (size_t)std::max<int64_t>(q_count, 1);
  if (plan.kind == PASS_TC) {
    const size_t npad = (size_t)((n + 255) / 256 * 256);
    b += npad * (plan.dpad + 16) * 2 + (size_t)n * 16;            // reference image + a2, e
    b += (size_t)((n + 127) / 128) * d * 8 + (size_t)d * 8 + 4096;  // column partials, mu, globals
  }
  return b;
}

}  // extern "C"
