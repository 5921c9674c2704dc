// internal.h — shared structs and kernel launchers of libtod (not part of the ABI).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace tod {

// Quantized operand image of a row set in HBM ("input quantization", step (i)
// of provable quantization).  16-bit elements laid out exactly as
// tcgen05 K-major swizzled shared-memory tiles, so a contiguous bulk copy of
// rows [r0, r0+R) of one K region lands as a ready UMMA operand.  K = dpad + 16:
//   main regions kb = 0..nkb-1: 64-element K blocks (or one block of dpad < 64
//     elements), n_pad rows x rb bytes, rb = min(128, 2*dpad), swizzle
//     SW128/SW64/SW32 (16-byte chunks XOR-swizzled within 8-row atoms);
//   extra region (16 elements, 32-byte rows, SW32): the fp16/bf16 pieces of
//     ||xhat_j||^2 (reference image "B") or the power-of-two constants that
//     multiply them (query image "A"), so the tensor core itself produces
//     w_ij = ||xhat_j||^2 - 2 xhat_i.xhat_j (the A image stores -2 xhat_i).
struct Image {
  uint16_t* data = nullptr;
  double* a2 = nullptr;     // [n] ||xhat_r||^2 in fp64 (B: references; A: queries)
  double* e = nullptr;      // [n] upper bound on ||xhat_r - s(x_r - mu)||
  int64_t n = 0, n_pad = 0;
  int dpad = 0, rb = 0, nkb = 0, layout = 0;  // layout: 2=SW128, 4=SW64, 6=SW32
  __host__ __device__ size_t region_bytes() const { return (size_t)n_pad * rb; }
  __host__ __device__ size_t extra_offset() const { return (size_t)nkb * n_pad * rb; }
  // + 256 rows of slack after the last (extra) region: kernels whose reference
  // tiles are not 256-row aligned (knn_tc5.cu, 160-row tiles) read up to one
  // tile past n_pad (masked columns).
  __host__ __device__ size_t total_bytes() const { return extra_offset() + (size_t)(n_pad + 256) * 32; }
};

// Global prep scalars, device resident.
struct PrepGlobals {
  double s;          // power-of-two scale
  double amax2;      // max_j ||xhat_j||^2 over references
  double emax;       // max_j e_j over references
  double repmax;     // max_j |sum_q c_q p_jq - ||xhat_j||^2| (norm-piece representation error)
  unsigned long long absmax_bits;  // max |x - mu| (fp64 bits) over queries and references
  int nonfinite;     // any NaN/Inf seen in X (or Q)
  int pad;
};

// Candidate lists written by the pass-1 kernels: per (query row, list) K'
// column indices (-1 = empty) and the threshold v (keys of non-kept >= v).
// The tensor-core kernel keeps ONE list per row across all S reference chunks
// (state parked in st_list between chunks); the SIMT kernel writes S lists.
struct Cands {
  int32_t* idx = nullptr;   // [q_count][lists][kp]
  float* v = nullptr;       // [q_count][lists]
  float* key = nullptr;     // TC: [q_count][lists][kp] group-min w~ of each kept group (ascending)
  int kp = 0, S = 0;        // S = reference chunks
  int lists = 1;            // lists per row (TC: epilogue split 1|2; SIMT: S)
  uint2* st_list = nullptr; // TC: [q tiles][kp][128] parked (key, index) state
  int* st_done = nullptr;   // TC: [q tiles] chunks completed
  int R = 1;                // tile stride (sample pass: every R-th 256-column tile)
  int dbg = 0;  // profiling aid bits (TOD_F_DEBUG_*), 0 in production
  long long* trace = nullptr;  // TOD_F_DEBUG_TRACE: [4096 tiles][8] clock64 stamps of CTA 0
};

enum PassKind : int { PASS_TC = 0, PASS_SIMT = 1 };

// ---- prep.cu
cudaError_t launch_prep_stats(const float* X, int64_t n, int d, double* mu, double* partial,
                              int partial_blocks, PrepGlobals* g, cudaStream_t st, int* launches);
cudaError_t launch_prep_absmax(const float* X, int64_t n, int d, const double* mu, PrepGlobals* g,
                               cudaStream_t st, int* launches);
cudaError_t launch_prep_scale(PrepGlobals* g, int fmt, int dpad, cudaStream_t st, int* launches);
// side 0 = reference image B (xhat | norm pieces; updates amax2/emax/repmax),
// side 1 = query image A (-2 xhat | constants).
cudaError_t launch_prep_quant(const float* X, int64_t n, int d, const double* mu, PrepGlobals* g,
                              int fmt, Image img, int side, cudaStream_t st, int* launches);
cudaError_t launch_prep_colsum(const float* X, int64_t n, int d, double* partial, PrepGlobals* g,
                               cudaStream_t st, int* launches);
cudaError_t launch_prep_colmean(const double* partial, int blocks, int64_t n, int d, double* mu,
                                cudaStream_t st, int* launches);
int prep_stat_rows();  // rows per column-sum partial block (128)
// eg[g] = max of e[8g .. 8g+7] (rows < n): per-group residual bound for the re-rank
cudaError_t launch_group_emax(const double* e, int64_t n, double* eg, cudaStream_t st, int* launches);
cudaError_t launch_image_decode(const Image& img, int fmt, int64_t rows, float* out, cudaStream_t st,
                                int* launches);  // diagnostics: 16-bit image -> fp32 [rows][dpad+16]
cudaError_t launch_finite_check(const float* X, int64_t n, int d, PrepGlobals* g, cudaStream_t st,
                                int* launches);

// ---- knn_tc.cu  (tcgen05 fused distance + top-K')
int tc_split_fits(int dpad, int kp, int split);  // 1 if the split epilogue fits in smem with K''=kp
cudaError_t launch_knn_tc(const Image& A, const Image& B, int64_t q_begin, int64_t q_count,
                          bool self_join, int fmt, Cands c, int num_sms, cudaStream_t st,
                          int* launches);

// ---- knn_tc3.cu  (main pass: tcgen05 distance + fixed-threshold filter, append-only)
// Two-pass candidate selection: the sample pass (launch_knn_tc with
// Cands.R = R) keeps a small list per row over every R-th 256-column reference
// tile; its threshold v is tau for the main pass, which appends every group of
// the remaining tiles whose minimum is below tau to a per-(row, column half)
// HBM buffer.
struct MainPass {
  int S = 1;                  // reference chunks (L2 locality)
  int R = 0;                  // sample stride: tiles t % R == 0 are skipped (0 = none)
  const float* tau_v = nullptr;  // [q_count][tau_lists] sample-list thresholds
  int tau_lists = 1;
  uint2* buf = nullptr;       // [q_count][parts][cap] (key bits, group index)
  int* cnt = nullptr;         // [q_count][parts] appended counts (may exceed cap = overflow)
  int cap = 0;
  int parts = 2;              // column parts per tile (one buffer per (row, part))
  float* samp = nullptr;      // sample mode (knn_tc3; knn_tc4 K-pipelined with smode 1): [q_count][parts][samp_t] smallest
                              // group minima over the sample tiles t = 0, R, 2R, ... (no appends)
  int samp_t = 4;             // 4 or 8
  int samp_acc = 0;           // sample mode: merge into the minima already in samp (ring of blocks)
  int64_t col0 = 0;           // global index of reference row 0 of the image (a ring block; % 256 == 0)
  int vote = 0;               // filter: test each part's minimum with one warp vote first (rare appends)
  long long* trace = nullptr; // profiling (TOD_F_DEBUG_TRACE): CTA 0's per-tile clock64 stamps
  int colmode = 0;            // appends are (w~, column) of each column below tau, not group minima
  int nb = 256;               // CTA-pair main pass tile: 256 columns x 2 accumulators, or 160 x 3
  int smode = 0;              // CTA-pair main pass: 1 = sweep only the sample tiles t % R == 0
};
cudaError_t launch_tau_from_appends(int64_t q, int parts, int cap, const int* cnt, const uint2* buf,
                                    int j, float* tau, cudaStream_t st, int* launches);
cudaError_t launch_tau_combine(int64_t q, int nv, int j, const float* samp, float* tau,
                               cudaStream_t st, int* launches);
int tc3_fits(int dpad);
int tc3_parts(int dpad);      // column parts (= filter warps / 4) the main pass uses
// ---- knn_tc4.cu  (the same main pass on CTA pairs: tcgen05 cta_group::2, M = 256)
// ---- knn_tc5.cu  (single-SM main pass, three 160-column accumulators; MainPass.R == 0 only)
int tc5_fits(int dpad);
cudaError_t launch_knn_tc5(const Image& A, const Image& B, int64_t q_begin, int64_t q_count,
                           bool self_join, int fmt, const MainPass& m, int num_sms, cudaStream_t st,
                           int* launches);
int tc4_fits(int dpad, int parts);
int tc4_preferred(int dpad);   // shapes where the pair beats the single-SM main pass
cudaError_t launch_knn_tc4(const Image& A, const Image& B, int64_t q_begin, int64_t q_count,
                           bool self_join, int fmt, const MainPass& m, int num_sms, int dbg,
                           cudaStream_t st, int* launches);
cudaError_t launch_knn_tc3(const Image& A, const Image& B, int64_t q_begin, int64_t q_count,
                           bool self_join, int fmt, const MainPass& m, int num_sms, int dbg,
                           cudaStream_t st, int* launches);

// ---- knn_simt.cu  (CUDA-core fp32 difference-form fused distance + top-K')
cudaError_t launch_knn_simt(const float* Q, int64_t q_begin, int64_t q_count, const float* X,
                            int64_t n, int d, bool self_join, Cands c, cudaStream_t st,
                            int* launches);

// ---- rerank.cu  (fp64 re-rank + certificate, fp64 brute-force fallback)
struct CertParams {
  int kind;        // PassKind
  int d, dpad;
  double s;        // scale (tensor path)
  const PrepGlobals* g;  // device: amax2, emax (tensor path)
  const double* qa2;     // query ||xhat||^2 (tensor path)
  const double* qe;      // query residual bound (tensor path)
  const double* eg;      // per 8-row reference group: max residual bound (nullable: emax)
  const double* ecol;    // per reference row: residual bound e_j (column candidates; nullable: eg/emax)
  int force_fail;        // TOD_F_NO_CERTIFY
  int colmode;           // two-pass candidates are single columns (MainPass.colmode), not 8-column groups
  // The reference operand image (self-join, single process; nullable): the
  // re-rank's per-column pre-bound reads xhat rows from it (DESIGN.md §5 "Re-rank").
  const uint8_t* bimg;
  size_t b_region;       // bytes per 64-element K region
  int b_rb;              // bytes per row per region (128 / 64 / 32)
  int fmt;               // 1 fp16, 2 bf16
};
struct KnnOutDev {
  int64_t* idx;
  float* dist;
  double* dist64;
  float* score_kth;
  float* score_mean;
  double* kdist64;
  int32_t* tier;   // [q] diagnostics (nullable): 0 certified by pass 1, 1 second tier, 2 fp64 tiers
};
size_t rerank_split_ws(int64_t q);  // bytes of the split re-rank's workspace (tensor-core pass)
int rerank_use_split(int d);        // the split re-rank is used at this width (d > 256)
cudaError_t launch_rerank(const float* Q, int64_t q_begin, int64_t q_count, const float* X,
                          int64_t n, int d, int k, bool self_join, Cands c, const MainPass* mp,
                          CertParams cp,
                          KnnOutDev out, int32_t* fail_rows, double* fail_ub, int32_t* fail_count,
                          double* max_err, unsigned long long* counters, void* split_ws, cudaStream_t st,
                          int* launches);
int fallback_slices(int nfail, int64_t n, int num_sms);
size_t fallback_workspace(int nfail, int k, int64_t n, int num_sms);
// second tier for bf16 passes (rerank.cu)
cudaError_t launch_gather_rows(const float* src, int64_t base, const int32_t* rows, int nr, int d,
                               float* dst, cudaStream_t st, int* launches);
cudaError_t launch_mark_rows(const int32_t* rows, int nr, int32_t value, int32_t* dst,
                             cudaStream_t st, int* launches);
cudaError_t launch_tier2_scatter(const int32_t* rows, int nr, int64_t q_begin, bool self_join, int k,
                                 int k2, const int64_t* idx2, const double* dd2, KnnOutDev out,
                                 cudaStream_t st, int* launches);
cudaError_t launch_fallback(const float* Q, int64_t q_begin, const float* X, int64_t n, int d,
                            int k, bool self_join, const int32_t* fail_rows,
                            const double* fail_ub, int nfail,
                            KnnOutDev out, void* ws, int num_sms, cudaStream_t st, int* launches);

// ---- rerank.cu: NWR (neighbours within range, §5.3)
cudaError_t launch_nwr_tau(int64_t q_count, double phi, CertParams cp, float* tau,
                           cudaStream_t st, int* launches);
cudaError_t launch_nwr_verify(const float* Q, int64_t q_begin, int64_t q_count, const float* X,
                              int64_t n, int d, bool self_join, double phi, const MainPass& mp,
                              int mode, int64_t* counts, const int64_t* row_ptr, int32_t* cols,
                              int32_t* ovf_rows, int32_t* ovf_count, int64_t* tasks_ws,
                              void* scan_ws, int num_sms, cudaStream_t st, int* launches);
size_t nwr_tasks_ws(int64_t q_count, const MainPass& mp);  // int64 words
cudaError_t launch_nwr_brute(const float* Q, int64_t q_begin, const float* X, int64_t n, int d,
                             bool self_join, double phi, const int32_t* rows, int nrows, int mode,
                             int64_t* counts, const int64_t* row_ptr, int32_t* cols, int64_t* bcnt,
                             cudaStream_t st, int* launches);
int nwr_brute_slices();       // bcnt holds nrows x nwr_brute_slices() counts
size_t scan_workspace(int64_t q);
cudaError_t launch_scan(const int64_t* counts, int64_t q, int64_t* row_ptr, void* ws,
                        cudaStream_t st, int* launches);

// ---- consumers.cu (ABOD, kNN classifier on the exact neighbour lists)
cudaError_t launch_abod(const float* X, int64_t q_begin, int64_t q_count, int d, int k,
                        const int64_t* idx, float* score, cudaStream_t st, int* launches);
int abod_max_k();
cudaError_t launch_knn_classify(int64_t nq, int k, const int64_t* idx, const int32_t* labels,
                                int32_t* pred, cudaStream_t st, int* launches);

// ---- lof.cu
cudaError_t launch_lof_lrd(int64_t q_count, int k, const int64_t* idx, const double* dist64,
                           const double* kdist64_all, double* lrd64_out, cudaStream_t st,
                           int* launches);
cudaError_t launch_lof_finish(int64_t q_begin, int64_t q_count, int k, const int64_t* idx,
                              const double* lrd64_all, float* lof_out, float* lrd_out,
                              cudaStream_t st, int* launches);

}  // namespace tod
