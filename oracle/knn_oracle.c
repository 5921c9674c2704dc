/*
 * knn_oracle.c — the plain, slow, obviously-correct CPU oracle for exact kNN.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.  The
 * product path (paper_2110_14007_b200/) never links, imports or calls it, and
 * the two share no code, header, table or constant.
 *
 * What it computes:
 *
 *   O1  D64(i,j) = sum_{c=0..d-1, ascending c, from +0.0} t*t,
 *       t = fl64(x_ic - x_jc), every op IEEE-754 binary64 round-to-nearest,
 *       no FMA contraction (compiled with -ffp-contract=off).
 *       This is the difference form of Eq. (3)'s left-hand side,
 *       ||X_i - X_j||^2 (§5.3).  The paper reaches this
 *       result exactly ("the result is still exact"; "output results
 *       are exact and consistent across systems"), so the oracle is
 *       the definition itself, with no quantisation, batching or fusion.
 *   O2  Neighbours of row i: all j != i (self excluded by index, reading A3),
 *       sorted ascending by the key (D64(i,j), j) with a full sort (reading A4:
 *       ties broken by the smaller index), first k kept.  kNN = cdist then
 *       topk; topk returns the k smallest (reading A13).
 *
 * Query variant (tod_knn_query analogue, P:1114 decision_function): the same
 * O1/O2 between a query row and every reference row, with no self exclusion.
 *
 * Parity pins: tests/test_oracle.py (hand examples S:143/S:153/S:271, exact
 * integer brute force, sklearn brute-force cross-check, symmetry/scaling).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

typedef struct {
    double key;   /* D64(i,j) */
    int64_t j;    /* reference index */
} pair_t;

/* O2's strict total order: (D64, index) lexicographic. */
static int pair_cmp(const void* a, const void* b) {
    const pair_t* p = (const pair_t*)a;
    const pair_t* q = (const pair_t*)b;
    if (p->key < q->key) return -1;
    if (p->key > q->key) return 1;
    if (p->j < q->j) return -1;
    if (p->j > q->j) return 1;
    return 0;
}

/* O1: sequential fp64 sum of squared fp64 differences. */
double oracle_d64(const float* a, const float* b, int32_t d) {
    double acc = 0.0;
    for (int32_t c = 0; c < d; ++c) {
        double t = (double)a[c] - (double)b[c];
        double sq = t * t;
        acc = acc + sq;
    }
    return acc;
}

int oracle_num_threads(void) {
#ifdef _OPENMP
    return omp_get_max_threads();
#else
    return 1;
#endif
}

/*
 * kNN of the query rows `rows[0..nrows)` of X (n x d, row-major fp32) against
 * all rows of X, self excluded.  Writes idx_out[r*k + m] and d64_out[r*k + m]
 * for m = 0..k-1 (ascending key).  Returns 0, or -1 on bad arguments / OOM.
 */
int oracle_knn_rows(const float* X, int64_t n, int32_t d, int32_t k,
                    const int64_t* rows, int64_t nrows,
                    int64_t* idx_out, double* d64_out, int32_t nthreads) {
    if (!X || !rows || !idx_out || !d64_out) return -1;
    if (n < 2 || d < 1 || k < 1 || k > n - 1 || nrows < 0) return -1;
    int failed = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel
#endif
    {
        pair_t* buf = (pair_t*)malloc((size_t)(n - 1) * sizeof(pair_t));
        if (!buf) {
#ifdef _OPENMP
#pragma omp atomic write
#endif
            failed = 1;
        }
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
        for (int64_t r = 0; r < nrows; ++r) {
            if (!buf) continue;
            int64_t i = rows[r];
            if (i < 0 || i >= n) {
#ifdef _OPENMP
#pragma omp atomic write
#endif
                failed = 1;
                continue;
            }
            const float* xi = X + (size_t)i * d;
            int64_t m = 0;
            for (int64_t j = 0; j < n; ++j) {
                if (j == i) continue;
                buf[m].key = oracle_d64(xi, X + (size_t)j * d, d);
                buf[m].j = j;
                ++m;
            }
            qsort(buf, (size_t)m, sizeof(pair_t), pair_cmp);
            for (int32_t t = 0; t < k; ++t) {
                idx_out[r * k + t] = buf[t].j;
                d64_out[r * k + t] = buf[t].key;
            }
        }
        free(buf);
    }
    return failed ? -1 : 0;
}

/*
 * Query variant: kNN of each row of Q (nq x d) among all rows of X (n x d),
 * nothing excluded.  Requires 1 <= k <= n.
 */
int oracle_knn_query(const float* Q, int64_t nq, const float* X, int64_t n, int32_t d,
                     int32_t k, int64_t* idx_out, double* d64_out, int32_t nthreads) {
    if (!Q || !X || !idx_out || !d64_out) return -1;
    if (n < 1 || d < 1 || k < 1 || k > n || nq < 0) return -1;
    int failed = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel
#endif
    {
        pair_t* buf = (pair_t*)malloc((size_t)n * sizeof(pair_t));
        if (!buf) {
#ifdef _OPENMP
#pragma omp atomic write
#endif
            failed = 1;
        }
#ifdef _OPENMP
#pragma omp for schedule(dynamic, 1)
#endif
        for (int64_t r = 0; r < nq; ++r) {
            if (!buf) continue;
            const float* q = Q + (size_t)r * d;
            for (int64_t j = 0; j < n; ++j) {
                buf[j].key = oracle_d64(q, X + (size_t)j * d, d);
                buf[j].j = j;
            }
            qsort(buf, (size_t)n, sizeof(pair_t), pair_cmp);
            for (int32_t t = 0; t < k; ++t) {
                idx_out[r * k + t] = buf[t].j;
                d64_out[r * k + t] = buf[t].key;
            }
        }
        free(buf);
    }
    return failed ? -1 : 0;
}

/*
 * NWR -- neighbours within range (§5.3): "each pairwise
 * distance in D is compared with phi, and NWR outputs the indices of samples
 * where D_ij <= phi", D_ij the SQUARED Euclidean distance of Eq. (3), here its
 * exact definition O1 (oracle_d64).  Self excluded (reading A3).
 * Pass 1 (cols == NULL): counts_out[r] = |{j != rows[r] : D64 <= phi}|.
 * Pass 2: the neighbours of each row, ascending j, written at cols + offs[r].
 */
int oracle_nwr_rows(const float* X, int64_t n, int32_t d, double phi, const int64_t* rows,
                    int64_t nrows, int64_t* counts_out, const int64_t* offs, int64_t* cols,
                    int32_t nthreads) {
    if (!X || !rows || !counts_out || n < 1 || d < 1 || nrows < 0) return -1;
    if (cols && !offs) return -1;
    int failed = 0;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (int64_t r = 0; r < nrows; ++r) {
        const int64_t i = rows[r];
        if (i < 0 || i >= n) {
#ifdef _OPENMP
#pragma omp atomic write
#endif
            failed = 1;
            continue;
        }
        const float* xi = X + (size_t)i * d;
        int64_t c = 0;
        for (int64_t j = 0; j < n; ++j) {
            if (j == i) continue;
            if (oracle_d64(xi, X + (size_t)j * d, d) <= phi) {
                if (cols) cols[offs[r] + c] = j;
                ++c;
            }
        }
        counts_out[r] = c;
    }
    return failed ? -1 : 0;
}
