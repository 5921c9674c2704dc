"""CPU oracle for exact kNN outlier scores and LOF (TOD, arXiv 2110.14007).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` legs may import this
package.  The product package ``paper_2110_14007_b200`` never imports it; the
two share no code (the seeded generators live in ``datagen/``).

Definitions:
  O1 distance  ``D64(i,j)``: sequential fp64 sum of squared fp64 differences,
     no FMA (knn_oracle.c; Eq. (3) LHS).
  O2 neighbours: sort all j != i by (D64, j), keep k (A3, A4, A13).
  O3 kNN scores: score_kth = fp32(sqrt(D64_(k))); score_mean =
     fp32((sum_m sqrt(D64_(m)), sequential in m) / k)  ("higher = more
     outlying"; Table 1; reading A1 returns both, A2 Euclidean units).
  O4 LOF (Breunig 2000, cited at P:158/P:184 without restating):
     kdist(o) = dist_o,(k); reach(p,o) = max(kdist(o), dist(p,o));
     S_p = sum_m reach(p, o_m) sequential; lrd_p = k / S_p (= +inf when S_p = 0);
     LOF_p = (sum_m lrd_{o_m} sequential) / (k * lrd_p), LOF_p = 1 when
     lrd_p = +inf (reading A6); all fp64, rounded to fp32 at the end.
     Neighbourhoods are the k-exact sets of O2 (reading A5).
  O6 ABOD: -variance of the distance-weighted neighbour-pair
     angle factor <a,b>/(|a|^2 |b|^2) (Kriegel 2008; reading A20).
  O7 kNN classifier (Appendix B): majority vote, nearest-first ties.
  O5 NWR: {j != i : D64(i,j) <= phi}, phi on the squared distance
     of Eq. (3), neighbours ascending by j (CSR).

Every function here is pinned by tests/test_oracle.py against hand-derived
values, exact integer brute force, scipy/sklearn library routines and
invariants.  Nothing here is "parity unpinned".
"""
from __future__ import annotations

import ctypes
import math
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "knn_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

# Flags that make the C oracle follow O1 literally: IEEE binary64, no FMA
# contraction, no fast-math reassociation.
CFLAGS = ["-O2", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off", "-fno-fast-math",
          "-std=c11"]


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (idempotent)."""
    with _lock:
        if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
            tmp = _LIB + ".tmp%d" % os.getpid()
            subprocess.check_call(["gcc", *CFLAGS, _SRC, "-o", tmp, "-lm"])
            os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        build()
        lib = ctypes.CDLL(_LIB)
        lib.oracle_d64.restype = ctypes.c_double
        lib.oracle_d64.argtypes = [ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32]
        lib.oracle_knn_rows.restype = ctypes.c_int
        lib.oracle_knn_rows.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                        ctypes.c_int32, ctypes.c_void_p, ctypes.c_int64,
                                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32]
        lib.oracle_knn_query.restype = ctypes.c_int
        lib.oracle_knn_query.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_void_p,
                                         ctypes.c_int64, ctypes.c_int32, ctypes.c_int32,
                                         ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int32]
        lib.oracle_nwr_rows.restype = ctypes.c_int
        lib.oracle_nwr_rows.argtypes = [ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32,
                                        ctypes.c_double, ctypes.c_void_p, ctypes.c_int64,
                                        ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p,
                                        ctypes.c_int32]
        lib.oracle_num_threads.restype = ctypes.c_int
        _lib = lib
    return _lib


def _f32(x) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float32)
    if x.ndim != 2:
        raise ValueError("X must be 2-D (n, d)")
    return x


def num_threads() -> int:
    """OpenMP threads the C oracle uses (reported as cpu_baseline.cores)."""
    return int(_load().oracle_num_threads())


def d64(a, b) -> float:
    """O1 for two rows a, b (fp32 vectors)."""
    a = np.ascontiguousarray(a, dtype=np.float32).ravel()
    b = np.ascontiguousarray(b, dtype=np.float32).ravel()
    if a.shape != b.shape:
        raise ValueError("shape mismatch")
    return float(_load().oracle_d64(a.ctypes.data, b.ctypes.data, a.size))


def cdist64(X) -> np.ndarray:
    """Full O1 matrix (small n only): D[i, j] = D64(X_i, X_j)."""
    X = _f32(X)
    n = X.shape[0]
    out = np.empty((n, n), np.float64)
    for i in range(n):
        for j in range(n):
            out[i, j] = d64(X[i], X[j])
    return out


def knn(X, k: int, rows=None, threads: int = 0):
    """O2 for the query rows ``rows`` (default: all) of X against X, self excluded.

    Returns (idx int64 [r, k], d64 float64 [r, k]) in ascending (D64, j) order.
    """
    X = _f32(X)
    n, d = X.shape
    if not (1 <= k <= n - 1):
        raise ValueError("need 1 <= k <= n-1")
    if rows is None:
        rows = np.arange(n, dtype=np.int64)
    rows = np.ascontiguousarray(rows, dtype=np.int64).ravel()
    idx = np.empty((rows.size, k), np.int64)
    dd = np.empty((rows.size, k), np.float64)
    rc = _load().oracle_knn_rows(X.ctypes.data, n, d, k, rows.ctypes.data, rows.size,
                                 idx.ctypes.data, dd.ctypes.data, int(threads))
    if rc != 0:
        raise RuntimeError("oracle_knn_rows failed")
    return idx, dd


def knn_query(Q, X, k: int, threads: int = 0):
    """O2 for external queries Q against references X (no self exclusion)."""
    Q = _f32(Q)
    X = _f32(X)
    if Q.shape[1] != X.shape[1]:
        raise ValueError("dimension mismatch")
    nq, n = Q.shape[0], X.shape[0]
    if not (1 <= k <= n):
        raise ValueError("need 1 <= k <= n")
    idx = np.empty((nq, k), np.int64)
    dd = np.empty((nq, k), np.float64)
    rc = _load().oracle_knn_query(Q.ctypes.data, nq, X.ctypes.data, n, X.shape[1], k,
                                  idx.ctypes.data, dd.ctypes.data, int(threads))
    if rc != 0:
        raise RuntimeError("oracle_knn_query failed")
    return idx, dd


def nwr(X, phi: float, rows=None, threads: int = 0):
    """O5 NWR (§5.3): for each query row i (default: all),
    the rows j != i with D64(i, j) <= phi, phi a threshold on the SQUARED
    distance of Eq. (3).  Returns (counts int64 [r], row_ptr int64 [r+1],
    cols int64 [total]) in CSR form, neighbours ascending by j."""
    X = _f32(X)
    n, d = X.shape
    if rows is None:
        rows = np.arange(n, dtype=np.int64)
    rows = np.ascontiguousarray(rows, dtype=np.int64).ravel()
    counts = np.empty(rows.size, np.int64)
    lib = _load()
    if lib.oracle_nwr_rows(X.ctypes.data, n, d, float(phi), rows.ctypes.data, rows.size,
                           counts.ctypes.data, None, None, int(threads)) != 0:
        raise RuntimeError("oracle_nwr_rows failed")
    row_ptr = np.zeros(rows.size + 1, np.int64)
    np.cumsum(counts, out=row_ptr[1:])
    cols = np.empty(int(row_ptr[-1]), np.int64)
    c2 = np.empty_like(counts)
    if lib.oracle_nwr_rows(X.ctypes.data, n, d, float(phi), rows.ctypes.data, rows.size,
                           c2.ctypes.data, row_ptr.ctypes.data, cols.ctypes.data,
                           int(threads)) != 0:
        raise RuntimeError("oracle_nwr_rows failed")
    return counts, row_ptr, cols


def abod_from_knn(X, idx, rows=None):
    """O6 ABOD: the angle-based outlier factor of Kriegel et al. 2008 (cited
    PAPER.md P:182; built as kNN FO + angle FO; reading A20) over the
    k-exact neighbours, as in PyOD's fast ABOD: for row i with neighbours
    o_1..o_k (O2 order), v_m = x_{o_m} - x_i (fp64 of the fp32 inputs),
    q_m = sum_c v_mc^2 (sequential); for each pair (a < b), lexicographic, with
    q_a, q_b > 0:   w_ab = (sum_c v_ac * v_bc, sequential) / (q_a * q_b);
    mean = (sum w, pair order) / P;  var = (sum (w - mean)^2, pair order) / P;
    score_i = fp32(-var)  (0 when P = 0).  Higher = more outlying.
    Plain Python loops in fp64 (each op IEEE RN, no FMA)."""
    X = _f32(X).astype(np.float64)
    idx = np.asarray(idx)
    n, k = idx.shape
    rows = np.arange(n) if rows is None else np.asarray(rows)   # query row of idx[t]
    out = np.empty(n, np.float32)
    d = X.shape[1]
    for t in range(n):
        i = int(rows[t])
        V = [X[int(o)] - X[i] for o in idx[t]]
        q = []
        for v in V:
            acc = 0.0
            for c in range(d):
                acc = acc + float(v[c]) * float(v[c])
            q.append(acc)
        w = []
        for a in range(k):
            for b in range(a + 1, k):
                if q[a] > 0.0 and q[b] > 0.0:
                    dot = 0.0
                    for c in range(d):
                        dot = dot + float(V[a][c]) * float(V[b][c])
                    w.append(dot / (q[a] * q[b]))
        if not w:
            out[t] = 0.0
            continue
        s = 0.0
        for x in w:
            s = s + x
        mean = s / len(w)
        s2 = 0.0
        for x in w:
            u = x - mean
            s2 = s2 + u * u
        out[t] = np.float32(-(s2 / len(w)))
    return out


def knn_classify(idx, labels):
    """O7 kNN classifier (Appendix B: cdist -> topk ->
    majority vote): majority label among the k neighbours (O2 order); ties go to
    the tied class whose first neighbour is nearest (reading A21)."""
    idx = np.asarray(idx)
    labels = np.asarray(labels)
    out = np.empty(idx.shape[0], np.int32)
    for i in range(idx.shape[0]):
        ls = [int(labels[int(o)]) for o in idx[i]]
        cnt = {}
        for l in ls:
            cnt[l] = cnt.get(l, 0) + 1
        best = max(cnt.values())
        out[i] = next(l for l in ls if cnt[l] == best)
    return out


def euclid(d64_sorted) -> np.ndarray:
    """dist = sqrt_RN(D64) in fp64 (O1)."""
    return np.sqrt(np.asarray(d64_sorted, dtype=np.float64))


def scores(d64_sorted):
    """O3: (score_kth fp32, score_mean fp32) from the ascending D64 rows [r, k]."""
    dist = euclid(d64_sorted)
    r, k = dist.shape
    kth = dist[:, k - 1].astype(np.float32)
    acc = np.zeros(r, np.float64)
    for m in range(k):                      # sequential in rank order
        acc = acc + dist[:, m]
    mean = (acc / np.float64(k)).astype(np.float32)
    return kth, mean


def lof_from_knn(idx, d64_sorted):
    """O4 on a complete kNN table (rows 0..n-1).  Returns (lrd fp64, lof fp64)."""
    idx = np.asarray(idx, dtype=np.int64)
    dist = euclid(d64_sorted)
    n, k = dist.shape
    kdist = dist[:, k - 1]
    s = np.zeros(n, np.float64)
    for m in range(k):
        reach = np.maximum(kdist[idx[:, m]], dist[:, m])
        s = s + reach
    lrd = np.full(n, np.inf, np.float64)
    pos = s > 0
    lrd[pos] = np.float64(k) / s[pos]
    lsum = np.zeros(n, np.float64)
    for m in range(k):
        lsum = lsum + lrd[idx[:, m]]
    lof = np.ones(n, np.float64)
    fin = np.isfinite(lrd)
    with np.errstate(over="ignore", invalid="ignore"):
        lof[fin] = lsum[fin] / (np.float64(k) * lrd[fin])
    return lrd, lof


def lof_rows(X, k: int, rows, threads: int = 0):
    """O4 for selected rows only, via the exact neighbourhood closure.

    LOF_p needs lrd of p's neighbours, which needs the k-distance of their
    neighbours: kNN is run on rows ∪ N(rows) ∪ N(N(rows)) (at most
    |rows|·(1+k+k²) queries).  Returns dict with 'idx', 'd64', 'lrd', 'lof'
    (fp64) for ``rows`` in order.
    """
    rows = np.ascontiguousarray(rows, dtype=np.int64).ravel()
    table = {}

    def ensure(rs):
        need = np.array(sorted(set(int(r) for r in rs) - table.keys()), dtype=np.int64)
        if need.size:
            ii, dd = knn(X, k, need, threads)
            for t, r in enumerate(need):
                table[int(r)] = (ii[t], dd[t])

    ensure(rows)
    lvl1 = {int(o) for r in rows for o in table[int(r)][0]}
    ensure(lvl1)
    lvl2 = {int(q) for o in lvl1 for q in table[o][0]}
    ensure(lvl2)

    def kd(o):
        return float(np.sqrt(table[o][1][k - 1]))

    def lrd_of(p):
        ii, dd = table[p]
        dist = np.sqrt(dd)
        s = 0.0
        for m in range(k):
            s = s + max(kd(int(ii[m])), float(dist[m]))
        return float(k) / s if s > 0 else float("inf")

    out_lrd = np.empty(rows.size)
    out_lof = np.empty(rows.size)
    for t, p in enumerate(rows):
        p = int(p)
        lp = lrd_of(p)
        ls = 0.0
        for o in table[p][0]:
            ls = ls + lrd_of(int(o))
        out_lrd[t] = lp
        if np.isinf(lp):
            out_lof[t] = 1.0
        else:
            out_lof[t] = ls / (float(k) * lp)
    idx = np.stack([table[int(r)][0] for r in rows]) if rows.size else np.empty((0, k), np.int64)
    dd = np.stack([table[int(r)][1] for r in rows]) if rows.size else np.empty((0, k))
    return {"idx": idx, "d64": dd, "lrd": out_lrd, "lof": out_lof}
