/*
 * tod.h — C ABI of the B200-native exact kNN / LOF hot path of TOD
 * (Zhao et al., "TOD: GPU-accelerated Outlier Detection via Tensor Operations",
 * arXiv 2110.14007).  Implemented in paper_2110_14007_b200/csrc (CUDA sm_100a),
 * built as paper_2110_14007_b200/libtod.so.
 *
 * Citations are PAPER.md line numbers (P:nnn) of /root/reference/PAPER.md and
 * DESIGN.md section names.
 *
 * Problem statement: given X in R^{n x d} (rows = samples) without
 * labels, output outlier scores O in R^n, higher = more outlying, "roughly
 * deterministic and irrespective of the underlying system".  Here the scores
 * are EXACT: neighbour indices equal the fp64 brute-force oracle bit for bit
 * (DESIGN.md "Parity contract").
 *
 * Conventions for every entry point
 * ---------------------------------
 *  - Every call returns tod_status; TOD_OK == 0.  No C++ exception crosses
 *    the ABI.  On error the contents of output buffers are unspecified, and
 *    tod_last_message(ctx) returns a one-line human-readable reason.
 *  - Pointers may be DEVICE memory (cudaMalloc / torch CUDA tensors on the
 *    context's device) or HOST memory (pageable or pinned); the library
 *    detects which with cudaPointerGetAttributes and stages host buffers
 *    through its own device workspace (host<->device copies are inside the
 *    call).  Device pointers must be on cfg->device.
 *  - Layout: all matrices are row-major and contiguous.  X is fp32 n x d;
 *    per-row outputs are [q_count] and per-neighbour outputs [q_count x k].
 *  - Ownership: the caller owns X and every output buffer; X is read-only.
 *    The library owns only its workspace (allocated lazily, grown on demand,
 *    freed by tod_destroy).
 *  - Synchronisation: the call enqueues work on the context stream and
 *    synchronises that stream before returning, so results are valid on
 *    return.  A context must not be used by two threads at once.
 *  - Self-join semantics (P:270 kNN = cdist -> topk; DESIGN.md readings
 *    A3/A4/A13): row i's neighbours are all j != i (self excluded by INDEX,
 *    duplicates of i remain valid neighbours), ordered by the exact fp64
 *    squared distance D64(i,j) (DESIGN.md "Oracle" O1), ties broken by the
 *    smaller index, k smallest kept.
 */
#ifndef TOD_H_
#define TOD_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TOD_ABI_VERSION 4

/* Largest k (neighbours per row) this build serves; larger k -> TOD_E_UNSUPPORTED. */
#define TOD_MAX_K 128

typedef enum {
  TOD_OK = 0,
  TOD_E_ARG = -1,          /* null/misaligned pointer, bad enum, inconsistent sizes */
  TOD_E_NONFINITE = -2,    /* NaN or Inf in X (checked on device before any output) */
  TOD_E_RANGE = -3,        /* k < 1, k > n-1 (k > n for queries), n > 2^31-1, d < 1 or d > 4096, q range outside [0,n) */
  TOD_E_NOMEM = -4,        /* workspace allocation failed */
  TOD_E_CUDA = -5,         /* a CUDA runtime error (message has cudaGetErrorString) */
  TOD_E_NCCL = -6,         /* an NCCL error in the sharded path, or libnccl.so.2 not loadable */
  TOD_E_UNSUPPORTED = -7,  /* valid request this build cannot serve (message says why) */
  TOD_E_INTERNAL = -8      /* invariant violated inside the library (a bug) */
} tod_status;

/* Low-precision format of the first (tensor-core) pass — the "input
 * quantization" step (i) of provable quantization. */
typedef enum {
  TOD_FMT_AUTO = 0,   /* planner's choice: FP32 SIMT for small d, else FP16 */
  TOD_FMT_FP16 = 1,   /* tcgen05 kind::f16, power-of-two scaled fp16 operands, fp32 accumulate */
  TOD_FMT_BF16 = 2,   /* tcgen05 kind::f16 with bf16 operands, fp32 accumulate */
  TOD_FMT_FP32 = 3    /* CUDA-core fp32 difference-form tile path (no quantization) */
} tod_format;

/* Flags for tod_config.flags. */
#define TOD_F_NO_CERTIFY   0x1u  /* testing: treat every row as uncertified -> fp64 brute-force tier */
#define TOD_F_TIMING       0x2u  /* record per-phase CUDA-event times in tod_stats */
#define TOD_F_DEBUG_NULL_EPILOGUE 0x100u  /* profiling only: pass 1 skips its epilogue (results invalid) */
#define TOD_F_MAIN_1SM     0x20u  /* testing: run the main pass on single SMs (knn_tc3.cu) instead of CTA pairs */
#define TOD_F_PASS1_V1     0x10u   /* testing: force the single-query-tile tensor-core schedule (knn_tc.cu) */
#define TOD_F_DEBUG_TRACE  0x800u  /* profiling only: per-tile clock64 stamps of CTA 0 written to $TOD_TRACE_FILE */

typedef struct {
  int32_t device;          /* CUDA device ordinal */
  int32_t format;          /* tod_format */
  int32_t kprime;          /* K' candidates kept per row by the low-precision pass; 0 = auto */
  uint32_t flags;          /* TOD_F_* */
  void* stream;            /* cudaStream_t to run on; NULL = a stream the library creates, BLOCKING
                              with respect to the legacy default stream (it waits for work queued
                              there, e.g. by torch, before running) */
  int32_t chunks;          /* reference chunks S per query tile (load balance); 0 = auto */
  int32_t epilogue_split;  /* tensor-core pass: epilogue warps per TMEM lane quarter (1 or 2; 2 splits each
                              tile's columns into two per-row lists of K'/2+8); 0 = auto */
  size_t workspace_bytes;  /* automatic batching ("store as many samples as possible"):
                              budget for the query-dependent device workspace of tod_knn /
                              tod_knn_query / tod_lof (candidate buffers and lists, per-row bounds,
                              the query image); when one call's estimate exceeds it, the query rows
                              are processed in chunks of 128-row multiples (>= 128 rows), with
                              results bit-identical to one unchunked call.  0 = no limit.  The
                              reference-side buffers (X, its quantized image) are not covered. */
} tod_config;

typedef struct {
  int64_t rows;            /* query rows answered */
  int64_t certified;       /* rows whose top-k was certified by the low-precision pass (P:342-343 step iii) */
  int64_t fallback_rows;   /* rows recomputed by the fp64 brute-force tier ("recalculate on the subset") */
  int32_t kprime;          /* K' used */
  int32_t format;          /* tod_format actually used */
  int32_t chunks;          /* S used */
  int32_t dpad;            /* padded feature count of the tensor-core operands */
  double scale;            /* power-of-two scale s applied before quantization (1 for FP32) */
  double max_abs_err;      /* largest per-row pass-1 error term (E_i + quantization), scaled units */
  float ms_stage, ms_prep, ms_main, ms_certify, ms_fallback, ms_lof, ms_total;  /* with TOD_F_TIMING */
  int64_t kernel_launches; /* kernels launched by this call */
  int64_t cand_groups;     /* 8-column candidate groups kept by pass 1, summed over rows (tensor-core pass) */
  int64_t visited_groups;  /* groups the re-rank expanded to exact fp64 distances, summed over rows */
  int64_t cand_columns;    /* exact distances at or below the per-row bound kept for the final selection */
  float ms_main_kernel;    /* two-pass mode, TOD_F_TIMING: the main-pass kernel alone (ms_main also has the sample pass) */
  int32_t main_kernel;     /* main-pass kernel used: 0 = none (single pass), 3 = single-SM, 4 = CTA pairs,
                              5 = single-SM with a 3-deep accumulator ring */
  int32_t sample_pass;     /* two-pass sample: 0 = none, 1 = list-based (main pass skips the sample
                              tiles), 2 = key-only (main pass covers every tile), 3 = three-stage
                              (key-only pre-sample; the main-pass kernel over the sample tiles,
                              then over the others) */
  int32_t query_chunks;    /* query-row chunks the call was split into (workspace_bytes); 1 = none */
  int64_t prebound_skipped;/* columns of visited groups the re-rank's per-column pre-bound excluded
                              without their exact fp64 distance (ABI 4), summed over rows */
} tod_stats;

/* Per-neighbour and per-row outputs of the kNN functional operator (P:270,
 * P:448-455) and the kNN outlier scores (Table 1; reading A1: both the
 * k-th-neighbour distance and the mean kNN distance).  Every pointer is
 * nullable; non-null ones are filled for the q_count query rows. */
typedef struct {
  int64_t* idx;         /* [q_count x k] neighbour indices, ascending (D64, index) */
  float* dist;          /* [q_count x k] Euclidean distance fp32(sqrt_RN(D64)) */
  double* dist64;       /* [q_count x k] sqrt_RN(D64) in fp64 (bit-identical to the oracle) */
  float* score_kth;     /* [q_count] fp32(dist64[:, k-1]) */
  float* score_mean;    /* [q_count] fp32((sum_m dist64[:, m], sequential in m) / k) */
  double* kdist64;      /* [q_count] dist64[:, k-1] (k-distance; input of the LOF stage) */
  int32_t* row_tier;    /* [q_count] diagnostics: which step answered each row -- 0 = certified by the
                           low-precision pass (P:342 step iii), 1 = re-answered by the second tier
                           (the fp16 two-pass path on just the failing rows: bf16 -> fp16, fp16 ->
                           twice K'), 2 = the fp64 tiers ("recalculate on the subset") */
} tod_knn_out;

typedef struct tod_ctx tod_ctx;

/* Create a context bound to cfg->device.  cfg may be NULL (all defaults). */
tod_status tod_create(const tod_config* cfg, tod_ctx** out);

/* Free the context and its workspace.  NULL is a no-op. */
tod_status tod_destroy(tod_ctx* ctx);

/* Static string for a status code. */
const char* tod_status_str(tod_status s);

/* Reason for the last non-OK status returned on ctx ("" if none). */
const char* tod_last_message(const tod_ctx* ctx);

/* ABI version (TOD_ABI_VERSION) and build string (arch, git describe). */
int32_t tod_abi_version(void);
const char* tod_build_info(void);

/*
 * tod_knn — exact kNN self-join with fused distance + top-K' (P:452-459 operator
 * fusion; Eq. 3 P:350-355 for the tensor-core distance form) and re-derived
 * provable quantization.
 *
 *   X        fp32 [n x d] row-major, the whole dataset (references = all rows).
 *   q_begin, q_count   query rows [q_begin, q_begin+q_count) of X answered by
 *            this call (a process in a multi-GPU job passes its shard; a single
 *            process passes 0, n).  0 <= q_begin, q_begin+q_count <= n.
 *   k        1 <= k <= n-1.
 *   out      per-row outputs for the q_count rows (see tod_knn_out), may be NULL
 *            (then nothing is written — useful only for timing).
 *   stats    nullable.
 * Errors: TOD_E_RANGE, TOD_E_NONFINITE, TOD_E_ARG, TOD_E_NOMEM, TOD_E_CUDA,
 * TOD_E_UNSUPPORTED (e.g. d > 4096).
 */
tod_status tod_knn(tod_ctx* ctx, const float* X, int64_t n, int32_t d, int32_t k,
                   int64_t q_begin, int64_t q_count, const tod_knn_out* out,
                   tod_stats* stats);

/*
 * tod_lof — Local Outlier Factor over the whole dataset in one process
 * (Table 1 P:158, P:184 citing Breunig et al. 2000; DESIGN.md "Oracle" O4 and
 * readings A5/A6):
 *   kdist(o) = dist(o, o_k);  reach(p,o) = max(kdist(o), dist(p,o));
 *   lrd(p) = k / sum_m reach(p, o_m)   (+inf when the sum is 0);
 *   LOF(p) = (sum_m lrd(o_m)) / (k * lrd(p))   (1 when lrd(p) = +inf),
 * fp64 throughout, rounded to fp32 on output.
 *   lof, lrd  [n] fp32, nullable (lrd = +inf allowed).
 *   knn_out   nullable; if given, also receives the kNN outputs for all n rows.
 */
tod_status tod_lof(tod_ctx* ctx, const float* X, int64_t n, int32_t d, int32_t k,
                   float* lof, float* lrd, const tod_knn_out* knn_out, tod_stats* stats);

/*
 * Sharded LOF stages, for SPMD multi-GPU jobs (one process per GPU):
 * each rank runs tod_knn on its rows (with dist64 and kdist64), all-gathers
 * kdist64 to kdist64_all[n], calls tod_lof_lrd, all-gathers lrd64 to
 * lrd64_all[n], then calls tod_lof_finish.  Bit-identical to tod_lof.
 *
 * tod_lof_lrd:    lrd64_out[r] = k / sum_m max(kdist64_all[idx[r,m]], dist64[r,m])
 *                 for r < q_count (idx, dist64: [q_count x k] from tod_knn).
 * tod_lof_finish: lof_out[r] = fp32(LOF) with lrd(p) = lrd64_all[q_begin+r] and
 *                 neighbour lrds from lrd64_all; lrd_out[r] = fp32(lrd) (nullable).
 */
tod_status tod_lof_lrd(tod_ctx* ctx, int64_t n, int32_t k, int64_t q_count,
                       const int64_t* idx, const double* dist64, const double* kdist64_all,
                       double* lrd64_out);
tod_status tod_lof_finish(tod_ctx* ctx, int64_t n, int32_t k, int64_t q_begin, int64_t q_count,
                          const int64_t* idx, const double* lrd64_all, float* lof_out,
                          float* lrd_out);

/*
 * tod_knn_query — test-set scoring (the detector's decision_function on new
 * rows): kNN of each row of Q [nq x d] among the rows of
 * X [n x d], nothing excluded, 1 <= k <= n.  Same ordering and outputs as
 * tod_knn (indices refer to rows of X).
 */
/*
 * tod_nwr — neighbours within range (NWR, a functional operator of the paper's
 * programming model; §5.3, the paper's provable-quantization
 * case study).  For every query row i in [q_begin, q_begin + q_count) of X
 * (self-join), the rows j != i with  D_ij <= phi, where D_ij is the SQUARED
 * Euclidean distance of Eq. (3) evaluated exactly as the oracle's O1
 * (sequential fp64, no FMA) -- the output equals the fp64 brute force exactly.
 * Method (§5.1): fp16 tensor-core evaluation (the append-only main
 * pass) with a per-row rigorous bound selects candidate 8-column groups; every
 * candidate pair is decided in fp64; rows whose candidate buffers overflow are
 * recomputed by fp64 brute force ("recalculate on the subset").
 *   phi        finite threshold on the squared distance (phi < 0 => no pairs).
 *   counts     [q_count] int64 neighbour counts (nullable).
 *   row_ptr    [q_count + 1] int64 CSR offsets, row_ptr[0] = 0 (nullable).
 *   cols       [capacity] int32 neighbour indices, ascending within each row
 *              (nullable: call once without to size it, then again).
 *   total      (required) total number of pairs.
 * Pointers may be host or device (host buffers are staged).  Errors: as
 * tod_knn; TOD_E_RANGE if cols != NULL and capacity < *total (counts, row_ptr
 * and *total are still written); TOD_E_UNSUPPORTED for d > 64 or the FP32
 * format.
 */
tod_status tod_nwr(tod_ctx* ctx, const float* X, int64_t n, int32_t d, double phi,
                   int64_t q_begin, int64_t q_count, int64_t* counts, int64_t* row_ptr,
                   int32_t* cols, int64_t capacity, int64_t* total, tod_stats* stats);

/*
 * tod_abod — angle-based outlier scores (§4.2, Fig. 3(a):
 * the kNN functional operator followed by cosine similarity; Kriegel 2008,
 * cited P:182).  For each query row i in [q_begin, q_begin+q_count) of X
 * (self-join, exact neighbours as tod_knn): with a = x_a - x_i, b = x_b - x_i,
 * score_i = -Var over neighbour pairs (a < b) of <a,b> / (||a||^2 ||b||^2)
 * (Kriegel's distance-weighted angle factor, as PyOD's fast ABOD over the
 * k-exact neighbour set), pairs with a coincident neighbour skipped, 0 if none
 * remain (reading A20; higher = more outlying).
 * fp64 with the oracle's operation order; fp32 out.
 *   score    [q_count] fp32 (required).  knn_out: optional neighbour outputs.
 * Errors: as tod_knn; TOD_E_UNSUPPORTED for k > 48.
 */
tod_status tod_abod(tod_ctx* ctx, const float* X, int64_t n, int32_t d, int32_t k,
                    int64_t q_begin, int64_t q_count, float* score, const tod_knn_out* knn_out,
                    tod_stats* stats);

/*
 * tod_knn_classify — kNN classifier (Appendix B: cdist ->
 * topk -> majority vote).  For each row of Q (nq x d) the k nearest rows of X
 * (exact, as tod_knn_query) vote with labels[] (int32 per row of X); ties go to
 * the tied class whose first neighbour is nearest (reading A21).
 *   pred     [nq] int32 (required).
 */
tod_status tod_knn_classify(tod_ctx* ctx, const float* Q, int64_t nq, const float* X, int64_t n,
                            int32_t d, int32_t k, const int32_t* labels, int32_t* pred,
                            tod_stats* stats);

tod_status tod_knn_query(tod_ctx* ctx, const float* Q, int64_t nq, const float* X, int64_t n,
                         int32_t d, int32_t k, const tod_knn_out* out, tod_stats* stats);

/*
 * tod_debug_mainpass — diagnostics for the certificate's tensor-core error
 * model (reading A9; the verification step (iii) of PAPER.md
 * P:341-343 rests on it).  Quantizes X as tod_knn would (cfg->format), runs the
 * production main-pass kernel (single-SM or CTA-pair, as tod_knn would) for
 * query rows [0, 128) against all n rows, and returns:
 *   w      [128 x n] fp32: the raw tensor-core accumulators w~_ij (self and
 *          padding unmasked);
 *   a_ops  [128 x K] fp32: the query operand row i as multiplied (-2 xhat_i, then
 *          the norm-piece constants), K = dpad + 16;
 *   b_ops  [n x K] fp32: the reference operand row j (xhat_j, then the norm pieces),
 * so that w_ij = sum_c a_ops[i,c] b_ops[j,c] exactly (every product is exact in
 * fp32) and |w~_ij - w_ij| can be checked against the model.  All pointers are
 * DEVICE pointers; n >= 128.  *K_out = K; *main_kernel = 3 (single SM) or 4 (pair).
 */
tod_status tod_debug_mainpass(tod_ctx* ctx, const float* X, int64_t n, int32_t d, float* w,
                              float* a_ops, float* b_ops, int32_t* K_out, int32_t* main_kernel);

/* ===================================================================== *
 * Sharded multi-GPU path (§6.2: one process per GPU,    *
 * "subtasks are split equally").     *
 * ===================================================================== *
 * Rank r of W holds only its row block X_r = rows [row_offset, row_offset +
 * n_local) of X.  It answers the kNN of its own rows while the quantized
 * reference blocks circulate over an NCCL ring (double-buffered, overlapped with
 * the tensor-core pass); the fp32 rows the exact re-rank needs are all-gathered
 * once.  Outputs are bit-identical to tod_knn / tod_lof for every W.
 *
 * Communicator: the library creates its own NCCL communicator (libnccl.so.2 is
 * loaded at run time; when torch is loaded it is torch's copy) from an id that
 * rank 0 creates with tod_comm_id_create and the job broadcasts (e.g. with
 * torch.distributed).  Every rank then calls tod_comm_init on its context.  A
 * context without a communicator runs the sharded calls as a world of 1.
 * tod_comm_init_loopback (testing) makes the context run `world` VIRTUAL ranks
 * in this one process on its one GPU: the same schedule, every collective and
 * ring transfer replaced by device-to-device copies; the sharded calls then take
 * all rows (row_offset 0, n_local n) and write every rank's outputs.
 *
 * Shards must tile [0, n) in rank order with row_offset % 256 == 0; use
 * tod_shard_rows for the balanced split.  Every rank must make the same
 * sequence of sharded calls with the same (n, d, k).
 */

/* Opaque 128-byte communicator id (an ncclUniqueId). */
typedef struct {
  char bytes[128];
} tod_comm_id;

/* Rank 0: a fresh id (TOD_E_NCCL if libnccl.so.2 cannot be loaded). */
tod_status tod_comm_id_create(tod_comm_id* id);

/* Attach an NCCL communicator of `world` ranks to ctx (collective: every rank
 * calls it with the same id).  ctx's device must be this rank's GPU. */
tod_status tod_comm_init(tod_ctx* ctx, const tod_comm_id* id, int32_t rank, int32_t world);

/* Testing: `world` virtual ranks in this process (see above). */
tod_status tod_comm_init_loopback(tod_ctx* ctx, int32_t world);

/* Balanced split of n rows over `world` ranks on 256-row boundaries (host-only). */
tod_status tod_shard_rows(int64_t n, int32_t world, int32_t rank, int64_t* row_offset,
                          int64_t* n_local);

/*
 * tod_knn_sharded — tod_knn for this rank's rows of a sharded X.
 *   X_local          fp32 [n_local x d], rows [row_offset, row_offset + n_local) of X.
 *   n                global row count; 1 <= k <= n-1.
 *   out              this rank's rows (n_local), as tod_knn_out (nullable fields).
 *   score_kth_all, score_mean_all   [n] fp32 scores of ALL rows, gathered (nullable).
 * Errors: as tod_knn; TOD_E_ARG if the shards do not tile [0, n); TOD_E_NCCL.
 */
tod_status tod_knn_sharded(tod_ctx* ctx, const float* X_local, int64_t n_local, int64_t row_offset,
                           int64_t n, int32_t d, int32_t k, const tod_knn_out* out,
                           float* score_kth_all, float* score_mean_all, tod_stats* stats);

/*
 * tod_lof_sharded — tod_lof over a sharded X: kNN of own rows (ring), k-distances
 * all-gathered, lrd of own rows, lrd all-gathered, LOF of own rows, then LOF and
 * lrd of ALL rows gathered into lof_all / lrd_all ([n] fp32, nullable).
 *   out      this rank's kNN outputs (nullable).
 */
tod_status tod_lof_sharded(tod_ctx* ctx, const float* X_local, int64_t n_local, int64_t row_offset,
                           int64_t n, int32_t d, int32_t k, float* lof_all, float* lrd_all,
                           const tod_knn_out* out, tod_stats* stats);

/*
 * tod_workspace_size — estimated device bytes one tod_knn call over q_count
 * query rows of an n x d dataset allocates (reference image, per-row candidate
 * state, re-rank and fallback bookkeeping; excluding X and caller outputs), for
 * choosing cfg->workspace_bytes.  0 if the request is invalid.  Host-only.
 */
size_t tod_workspace_size(int64_t n, int32_t d, int32_t k, int64_t q_count, const tod_config* cfg);

#ifdef __cplusplus
}
#endif
#endif /* TOD_H_ */
