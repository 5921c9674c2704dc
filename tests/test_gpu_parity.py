"""GPU parity: libtod.so (through the C ABI) vs the CPU oracle, element by element
on the same seeded inputs.  Bar (BASELINE.json north_star, DESIGN.md "Parity
contract"): neighbour indices bit-exact (order included); fp32 scores within
1e-5 relative (they are in fact bit-identical because the re-rank evaluates the
oracle's own fp64 formula, so the tests demand exact equality and report the
relative error on failure)."""
import os

import numpy as np
import pytest

import datagen
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pkg():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2110_14007_b200 import build
    build.build()
    import paper_2110_14007_b200 as p
    return p


def _ctx(pkg, **kw):
    return pkg.Context(device=0, **kw)


def _np(x):
    return x.cpu().numpy() if hasattr(x, "cpu") else np.asarray(x)


def _check_rows(res, X, k, rows, q_begin=0, ref=None):
    """Compare GPU outputs of global rows `rows` with the oracle."""
    if ref is None:
        ref = oracle.knn(X, k, rows=rows)
    ri, rd = ref
    loc = np.asarray(rows) - q_begin
    gi = _np(res.idx)[loc]
    bad = np.nonzero((gi != ri).any(1))[0]
    assert bad.size == 0, "rows %s: gpu %s oracle %s" % (np.asarray(rows)[bad[:3]], gi[bad[:1]], ri[bad[:1]])
    assert np.array_equal(_np(res.dist64)[loc], np.sqrt(rd))
    kth, mean = oracle.scores(rd)
    g_kth, g_mean = _np(res.score_kth)[loc], _np(res.score_mean)[loc]
    rel = np.max(np.abs(g_mean - mean) / np.maximum(np.abs(mean), 1e-30)) if mean.size else 0
    assert np.array_equal(g_kth, kth) and np.array_equal(g_mean, mean), "rel err %g" % rel
    assert np.array_equal(_np(res.dist)[loc], np.sqrt(rd).astype(np.float32))


# ----------------------------------------------------------- configs[0] (C1)
def test_c1_full_bitexact(pkg):
    X = datagen.gaussian_mixture(1000, 10, seed=0)
    with _ctx(pkg) as ctx:
        res = ctx.knn(torch.from_numpy(X).cuda(), 10)
    _check_rows(res, X, 10, np.arange(1000))
    assert res.stats["certified"] + res.stats["fallback_rows"] == 1000


@pytest.mark.parametrize("n,d,k,fmt", [
    (3000, 32, 20, "fp16"),     # C2 shape, small n, several tiles + ragged tail
    (2999, 64, 10, "fp16"),     # C3 shape, ragged
    (1000, 16, 10, "fp16"),     # SW32 operand layout
    (1500, 100, 12, "fp16"),    # dpad 128 (two K regions), d not a multiple of 16
    (2500, 64, 10, "bf16"),
    (777, 10, 5, "fp32"),
    (2000, 40, 30, "fp32"),
    (257, 33, 7, "fp16"),       # one query tile more than a reference tile
])
def test_knn_full_parity(pkg, n, d, k, fmt):
    X = datagen.gaussian_mixture(n, d, seed=n + d)
    with _ctx(pkg, fmt=fmt) as ctx:
        res = ctx.knn(torch.from_numpy(X).cuda(), k)
    _check_rows(res, X, k, np.arange(n))
    st = res.stats
    assert st["rows"] == n
    if fmt != "bf16":
        assert st["certified"] >= 0.95 * n, st


@pytest.mark.parametrize("d", [32, 64])
@pytest.mark.parametrize("fmt", ["fp16", "bf16"])
@pytest.mark.parametrize("split", [1, 2, 4])
@pytest.mark.parametrize("chunks", [1, 3])
def test_epilogue_variants_parity(pkg, d, fmt, split, chunks):
    # every epilogue layout of the single-query-tile schedule (1/2/4 lists per
    # row, pending widths 16/24/32, tile- and chunk-level reserves) and parked
    # state across chunks
    n, k = 2300, 10
    X = datagen.gaussian_mixture(n, d, seed=77 + d)
    with _ctx(pkg, fmt=fmt, split=split, chunks=chunks, flags=pkg.F_PASS1_V1) as ctx:
        res = ctx.knn(torch.from_numpy(X).cuda(), k)
    _check_rows(res, X, k, np.arange(n))


@pytest.mark.parametrize("n,d,k,fmt,chunks", [
    (20_000, 32, 20, "fp16", 0),   # two-pass: sample pass (every 8th tile) + main pass
    (20_000, 64, 10, "fp16", 0),   # d=64 (SW128 operands)
    (17_001, 32, 10, "fp16", 4),   # sample pass in 4 chunks, ragged tail
    (9_000, 16, 6, "fp16", 2),     # smallest two-pass size, SW32 layout
    (12_345, 64, 10, "bf16", 3),
    (5_000, 32, 20, "fp16", 3),    # below the two-pass threshold: single pass, 3 chunks
])
@pytest.mark.parametrize("pair", [True, False])
def test_two_pass_parity(pkg, n, d, k, fmt, chunks, pair):
    # sample pass (every 8th tile) + append-only main pass (two-pass selection),
    # main pass on CTA pairs (cta_group::2) or single SMs; full-table parity at
    # sizes that span the sampling and chunk logic
    X = datagen.gaussian_mixture(n, d, seed=n + 3 * d)
    flags = 0 if pair else pkg.F_MAIN_1SM
    os.environ["TOD_MAIN_PAIR"] = "1" if pair else "0"
    try:
        with _ctx(pkg, fmt=fmt, chunks=chunks, flags=flags) as ctx:
            res = ctx.knn(torch.from_numpy(X).cuda(), k)
    finally:
        os.environ.pop("TOD_MAIN_PAIR", None)
    _check_rows(res, X, k, np.arange(n))
    if fmt == "fp16":
        assert res.stats["certified"] >= 0.99 * n, res.stats


@pytest.mark.parametrize("n,d,k,fmt", [
    (20_000, 32, 20, "fp16"),    # C2 shape: the default main pass at dpad 32
    (17_001, 32, 10, "bf16"),    # ragged last 160-row tile, bf16
    (9_000, 16, 6, "fp16"),      # SW32 operands
    (20_000, 64, 10, "fp16"),    # dpad 64 (forced: the default there is the CTA pair)
    (12_345, 64, 10, "bf16"),
])
def test_main_ring3_parity(pkg, n, d, k, fmt):
    # knn_tc5: single-SM main pass with three 160-column accumulators (160-row
    # reference tiles; a query tile's own columns can straddle two of them)
    X = datagen.gaussian_mixture(n, d, seed=n + 5 * d)
    env = {"TOD_MAIN_RING3": "1", "TOD_SAMPLE_V1": "0", "TOD_MAIN_PAIR": "0"}
    os.environ.update(env)
    try:
        with _ctx(pkg, fmt=fmt) as ctx:
            res = ctx.knn(torch.from_numpy(X).cuda(), k)
    finally:
        for e in env:
            os.environ.pop(e, None)
    assert res.stats["main_kernel"] == 5, res.stats
    _check_rows(res, X, k, np.arange(n))
    if fmt == "fp16":
        assert res.stats["certified"] >= 0.99 * n, res.stats


@pytest.mark.parametrize("n,d,k,fmt,v1,pair", [
    (20_000, 32, 20, "fp16", "0", "0"),   # key-only sample: column candidates only (tc3)
    (17_001, 32, 10, "bf16", "0", "0"),   # bf16 (second tier), ragged tail
    (20_000, 64, 10, "fp16", "1", "1"),   # list sample (group candidates) + CTA-pair main pass (columns)
    (12_345, 64, 10, "bf16", "1", "0"),   # mixed candidates, single-SM main pass
    (9_000, 512, 20, "fp16", "0", "0"),   # d = 512: split re-rank with column tasks
])
def test_column_candidates_parity(pkg, n, d, k, fmt, v1, pair):
    _column_case(pkg, n, d, k, fmt, {"TOD_SAMPLE_V1": v1, "TOD_MAIN_PAIR": pair})


@pytest.mark.parametrize("n,d,k,fmt,kern", [
    (20_000, 64, 10, "fp16", 4),
    (12_345, 64, 10, "bf16", 4),     # ragged tail, second tier
    (17_001, 64, 20, "fp16", 4),
    (20_000, 32, 20, "fp16", 3),     # d <= 32: the single-SM kernel's MODE 2 / MODE 1 sweeps
    (12_345, 32, 10, "bf16", 3),
    (9_001, 16, 8, "fp16", 3),
])
def test_three_stage_selection_parity(pkg, n, d, k, fmt, kern):
    # the default at d = 64 (and d <= 32 from n = 3e5; forced here): key-only
    # pre-sample (every 64th tile) -> the main pass over the sample tiles below
    # tau0 -> tau -> the main pass over the rest
    X = datagen.gaussian_mixture(n, d, seed=n + 11 * d)
    os.environ["TOD_SAMPLE3"] = "1"
    try:
        with _ctx(pkg, fmt=fmt) as ctx:
            res = ctx.knn(torch.from_numpy(X).cuda(), k)
    finally:
        os.environ.pop("TOD_SAMPLE3", None)
    assert res.stats["sample_pass"] == 3 and res.stats["main_kernel"] == kern, res.stats
    _check_rows(res, X, k, np.arange(n))
    if fmt == "fp16":
        assert res.stats["certified"] >= 0.99 * n, res.stats


@pytest.mark.parametrize("n,d,k,fmt,col", [
    (20_000, 64, 10, "fp16", "0"),
    (12_345, 64, 10, "bf16", "1"),
    (17_001, 32, 10, "fp16", "1"),
    (9_000, 16, 6, "fp16", "0"),
])
def test_pair_ring3_parity(pkg, n, d, k, fmt, col):
    # CTA-pair main pass with 160-column tiles and three accumulators (key-only
    # sample: the main pass covers every tile), group or column candidates
    _column_case(pkg, n, d, k, fmt, {"TOD_SAMPLE_V1": "0", "TOD_MAIN_PAIR": "1", "TOD_MAIN_NB": "160",
                                     "TOD_COLMODE": col}, main_kernel=4)


@pytest.mark.parametrize("n,d,k,fmt,col", [
    (12_000, 100, 12, "fp16", "0"),   # dpad 128, group candidates
    (9_000, 200, 10, "fp16", "1"),    # dpad 256, column candidates
    (9_000, 512, 20, "fp16", "1"),    # dpad 512 (C5 width)
    (7_001, 512, 50, "fp16", "0"),    # dpad 512, k = 50, ragged n
    (8_003, 128, 10, "bf16", "1"),    # bf16 (second tier)
])
def test_pair_kpipelined_parity(pkg, n, d, k, fmt, col):
    # CTA-pair main pass, K-pipelined (dpad > 64): each SM streams its own A slice
    # and half of each B slice per 64-wide K region (knn_tc4.cu KP mode)
    _column_case(pkg, n, d, k, fmt, {"TOD_SAMPLE_V1": "0", "TOD_MAIN_PAIR": "1", "TOD_COLMODE": col},
                 main_kernel=4)


def _column_case(pkg, n, d, k, fmt, extra, main_kernel=None):
    # MainPass.colmode: the main pass appends each column below tau of a passing
    # group (the default for large n); forced on here at sizes the oracle checks
    X = datagen.gaussian_mixture(n, d, seed=n + 7 * d)
    env = {"TOD_COLMODE": "1", "TOD_VOTE": "1"}
    env.update(extra)
    os.environ.update(env)
    try:
        with _ctx(pkg, fmt=fmt) as ctx:
            res = ctx.knn(torch.from_numpy(X).cuda(), k)
    finally:
        for e in env:
            os.environ.pop(e, None)
    if main_kernel is not None:
        assert res.stats["main_kernel"] == main_kernel, res.stats
    rows = np.arange(n) if n <= 20_000 and d <= 64 else np.random.default_rng(1).choice(n, 500, replace=False)
    _check_rows(res, X, k, np.sort(rows))
    if fmt == "fp16":
        assert res.stats["certified"] >= 0.99 * n, res.stats


@pytest.mark.parametrize("n,d,k,fmt", [
    (20_000, 32, 20, "fp16"),
    (20_000, 64, 10, "bf16"),
    (7_777, 16, 8, "fp16"),
    (9_000, 128, 10, "fp16"),    # generic (runtime-dpad) image read
])
def test_rerank_prebound_parity(pkg, n, d, k, fmt):
    # the re-rank's per-column pre-bound from the operand image (opt-in): the
    # columns it excludes must not change a single output
    X = datagen.gaussian_mixture(n, d, seed=n + 3 * d)
    os.environ["TOD_RR_PREBOUND"] = "1"
    try:
        with _ctx(pkg, fmt=fmt) as ctx:
            res = ctx.knn(torch.from_numpy(X).cuda(), k)
    finally:
        os.environ.pop("TOD_RR_PREBOUND", None)
    assert res.stats["prebound_skipped"] > 0, res.stats
    rows = np.arange(n) if n <= 20_000 and d <= 64 else np.random.default_rng(2).choice(n, 500, replace=False)
    _check_rows(res, X, k, np.sort(rows))


@pytest.mark.parametrize("pair", ["1", "0"])   # CTA-pair (default) / single-SM K-pipelined pass
@pytest.mark.parametrize("n,d,k", [
    (3000, 200, 10),     # dpad 256, small n: two-pass forced (K-pipelined main pass)
    (12_000, 100, 12),   # dpad 128, K-pipelined two-pass
    (9000, 512, 20),     # dpad 512 (C5 width)
    (2000, 300, 50),     # C5's k
])
def test_high_dimensional_parity(pkg, n, d, k, pair):
    X = datagen.gaussian_mixture(n, d, seed=n + d)
    os.environ["TOD_MAIN_PAIR"] = pair
    try:
        with _ctx(pkg) as ctx:
            res = ctx.knn(torch.from_numpy(X).cuda(), k)
    finally:
        os.environ.pop("TOD_MAIN_PAIR", None)
    rows = np.arange(n) if n <= 3000 else np.random.default_rng(0).choice(n, 400, replace=False)
    _check_rows(res, X, k, np.sort(rows))
    assert res.stats["certified"] >= 0.95 * n, res.stats


@pytest.mark.parametrize("v1", ["0", "1"])
@pytest.mark.parametrize("d", [32, 64])
def test_sample_pass_variants_parity(pkg, v1, d):
    # key-only register sample (knn_tc3 sample mode) and the list-based sample
    # (knn_tc.cu) at both widths
    n, k = 15_000, 12
    X = datagen.gaussian_mixture(n, d, seed=d + 5)
    os.environ["TOD_SAMPLE_V1"] = v1
    try:
        with _ctx(pkg) as ctx:
            res = ctx.knn(torch.from_numpy(X).cuda(), k)
    finally:
        os.environ.pop("TOD_SAMPLE_V1", None)
    _check_rows(res, X, k, np.arange(n))
    assert res.stats["certified"] >= 0.99 * n


def test_single_and_two_pass_identical(pkg):
    X = datagen.gaussian_mixture(30_000, 32, seed=31)
    Xd = torch.from_numpy(X).cuda()
    outs = []
    for flags in (0, pkg.F_PASS1_V1):
        with _ctx(pkg, flags=flags) as ctx:
            outs.append(ctx.knn(Xd, 20))
    assert torch.equal(outs[0].idx, outs[1].idx) and torch.equal(outs[0].dist64, outs[1].dist64)


def test_forced_fallback_tier(pkg):
    X = datagen.gaussian_mixture(1200, 24, seed=5)
    with _ctx(pkg, flags=pkg.F_NO_CERTIFY) as ctx:
        res = ctx.knn(torch.from_numpy(X).cuda(), 9)
    assert res.stats["fallback_rows"] == 1200
    _check_rows(res, X, 9, np.arange(1200))


@pytest.mark.parametrize("fmt", ["fp16", "fp32"])
def test_ties_lattice_and_duplicates(pkg, fmt):
    X = datagen.lattice(2000, 20, seed=3, extent=2)
    X = datagen.with_duplicates(X, frac=0.05, seed=4)
    with _ctx(pkg, fmt=fmt) as ctx:
        res = ctx.knn(torch.from_numpy(X).cuda(), 12)
    _check_rows(res, X, 12, np.arange(2000))


def test_translated_far_from_origin(pkg):
    # cancellation stress for the norm expansion: |x| >> pairwise distances
    X = datagen.uniform(2000, 32, seed=2, offset=1000.0)
    with _ctx(pkg, fmt="fp16") as ctx:
        res = ctx.knn(torch.from_numpy(X).cuda(), 10)
    _check_rows(res, X, 10, np.arange(2000))


def test_query_range_and_chunk_invariance(pkg):
    X = datagen.gaussian_mixture(4000, 32, seed=8)
    Xd = torch.from_numpy(X).cuda()
    outs = []
    for chunks, kp, sp in ((1, 0, 1), (3, 0, 2), (2, 64, 0), (1, 48, 2), (5, 40, 1), (4, 32, 2)):
        with _ctx(pkg, chunks=chunks, kprime=kp, split=sp) as ctx:
            outs.append(ctx.knn(Xd, 20, q_begin=1000, q_count=1700))
    for o in outs[1:]:
        assert torch.equal(o.idx, outs[0].idx) and torch.equal(o.dist64, outs[0].dist64)
    _check_rows(outs[0], X, 20, np.arange(1000, 2700), q_begin=1000)


def test_host_pointer_path_matches_device(pkg):
    X = datagen.gaussian_mixture(2500, 48, seed=11)
    with _ctx(pkg) as ctx:
        dev = ctx.knn(torch.from_numpy(X).cuda(), 15)
        host = ctx.knn(X, 15)
    assert np.array_equal(host.idx, _np(dev.idx))
    assert np.array_equal(host.score_mean, _np(dev.score_mean))


def test_lof_full_bitexact(pkg):
    X = datagen.gaussian_mixture(3000, 32, seed=21)
    k = 20
    with _ctx(pkg) as ctx:
        lof, lrd, res, st = ctx.lof(torch.from_numpy(X).cuda(), k, want_knn=("idx",))
    ri, rd = oracle.knn(X, k)
    olrd, olof = oracle.lof_from_knn(ri, rd)
    assert np.array_equal(_np(res.idx), ri)
    assert np.array_equal(_np(lof), olof.astype(np.float32))
    assert np.array_equal(_np(lrd), olrd.astype(np.float32))


def test_lof_duplicates_inf_lrd(pkg):
    X = np.repeat(datagen.gaussian_mixture(50, 8, seed=1), 4, axis=0)   # 4 copies each
    with _ctx(pkg) as ctx:
        lof, lrd, _, _ = ctx.lof(torch.from_numpy(X).cuda(), 3)
    ri, rd = oracle.knn(X, 3)
    olrd, olof = oracle.lof_from_knn(ri, rd)
    assert np.all(np.isinf(_np(lrd))) and np.all(_np(lof) == 1.0)
    assert np.array_equal(_np(lof), olof.astype(np.float32))


@pytest.mark.parametrize("fmt", ["fp16", "fp32"])
def test_knn_query_parity(pkg, fmt):
    X = datagen.gaussian_mixture(3000, 24, seed=31)
    Q = datagen.gaussian_mixture(700, 24, seed=32)
    Q[:10] = X[:10]     # exact duplicates of references: distance 0
    with _ctx(pkg, fmt=fmt) as ctx:
        res = ctx.knn_query(torch.from_numpy(Q).cuda(), torch.from_numpy(X).cuda(), 11)
    ri, rd = oracle.knn_query(Q, X, 11)
    assert np.array_equal(_np(res.idx), ri)
    assert np.array_equal(_np(res.dist64), np.sqrt(rd))


def test_error_paths(pkg):
    X = datagen.gaussian_mixture(100, 8, seed=0)
    with _ctx(pkg) as ctx:
        for k in (0, 100):
            with pytest.raises(pkg.TodError) as e:
                ctx.knn(torch.from_numpy(X).cuda(), k)
            assert e.value.status == -3
        Y = X.copy()
        Y[5, 3] = np.nan
        with pytest.raises(pkg.TodError) as e:
            ctx.knn(torch.from_numpy(Y).cuda(), 5)
        assert e.value.status == -2
        r = ctx.knn(torch.from_numpy(X).cuda(), 99)    # k = n-1: every other row
        assert sorted(_np(r.idx)[0].tolist()) == list(range(1, 100))


# ------------------------------------------------ BASELINE full-size configs
def _sample_rows(n, labels, m, seed):
    rng = np.random.default_rng(seed)
    out_rows = np.nonzero(labels)[0]
    rows = np.concatenate([rng.choice(n, m - m // 4, replace=False),
                           rng.choice(out_rows, m // 4, replace=False), [0, n - 1]])
    return np.unique(rows)


# ------------------------------------------------------------ NWR (NEXT-2)
def _nwr_check(got, X, phi, rows):
    counts, ptr, cols, st = got
    rc, rp, rl = oracle.nwr(X, phi, rows=rows)
    assert np.array_equal(_np(counts), rc)
    assert np.array_equal(_np(ptr), rp)
    assert np.array_equal(_np(cols).astype(np.int64), rl)
    return st


@pytest.mark.parametrize("n,d,q", [(3000, 32, 8.0), (2999, 64, 12.0), (1000, 16, 5.0),
                                   (20_000, 32, 4.0), (777, 10, 6.0)])
def test_nwr_full_parity(pkg, n, d, q):
    # phi = the q-th percentile of squared k-NN-scale distances: a few to ~100
    # neighbours per row; bit-exact CSR against the fp64 brute force
    X = datagen.gaussian_mixture(n, d, seed=n + 11 * d)
    _, dd = oracle.knn(X, 10, rows=np.arange(0, n, max(1, n // 200)))
    phi = float(np.percentile(dd[:, -1], 50)) * (q / 8.0)
    with _ctx(pkg) as ctx:
        got = ctx.nwr(torch.from_numpy(X).cuda(), phi)
    st = _nwr_check(got, X, phi, np.arange(n))
    assert st["rows"] == n


def test_nwr_boundary_and_ties_lattice(pkg):
    # integer lattice + duplicates: many pairs exactly on phi (boundary inclusive)
    X = datagen.with_duplicates(datagen.lattice(3000, 16, seed=3, extent=2), frac=0.05, seed=4)
    for phi in (0.0, 2.0, 5.0):
        with _ctx(pkg) as ctx:
            got = ctx.nwr(torch.from_numpy(X).cuda(), phi)
        _nwr_check(got, X, phi, np.arange(3000))


def test_nwr_overflow_rows_brute_force_and_query_range(pkg):
    # a phi so large that every row overflows its candidate buffers (-> fp64
    # brute force), on a query-row subrange, host buffers
    X = datagen.gaussian_mixture(40_000, 32, seed=77)   # 5000 groups > 4 x 1024 slots
    phi = 1e9
    with _ctx(pkg) as ctx:
        got = ctx.nwr(X, phi, q_begin=100, q_count=50)
    st = _nwr_check(got, X, phi, np.arange(100, 150))
    assert st["fallback_rows"] == 50
    # small phi on the same range: no overflow
    with _ctx(pkg) as ctx:
        got = ctx.nwr(X, 1.0, q_begin=4000, q_count=3000)
    assert _nwr_check(got, X, 1.0, np.arange(4000, 7000))["fallback_rows"] == 0


def test_nwr_dense_rows_block_emit(pkg):
    # 750 groups in all (never overflows 4 x 1024 slots): phi = inf-like puts every
    # group of every row in the output (> 256 nonzero entries: the dense-row block
    # emitter), a mid phi mixes dense and light rows
    X = datagen.gaussian_mixture(6000, 16, seed=21)
    _, dd = oracle.knn(X, 10, rows=np.arange(0, 6000, 60))
    for phi in (1e9, float(np.percentile(dd[:, -1], 50)) * 40.0):
        with _ctx(pkg) as ctx:
            got = ctx.nwr(torch.from_numpy(X).cuda(), phi, q_begin=2000, q_count=1500)
        st = _nwr_check(got, X, phi, np.arange(2000, 3500))
        assert st["fallback_rows"] == 0


def test_nwr_capacity_error_reports_total(pkg):
    X = datagen.gaussian_mixture(2000, 16, seed=5)
    phi = 50.0
    with _ctx(pkg) as ctx:
        c, p, _, _ = ctx.nwr(torch.from_numpy(X).cuda(), phi, lists=False)
        total = int(p[-1])
        with pytest.raises(pkg.TodError) as e:
            ctx.nwr(torch.from_numpy(X).cuda(), phi, capacity=max(1, total - 1))
    assert e.value.status == -3 and total > 1


# ------------------------------------------------ ABOD, kNN classifier (NEXT-3)
@pytest.mark.parametrize("n,d,k", [(1500, 16, 10), (900, 32, 5), (700, 10, 2)])
def test_abod_bitexact(pkg, n, d, k):
    X = datagen.gaussian_mixture(n, d, seed=n + k)
    X = datagen.with_duplicates(X, frac=0.02, seed=1)     # coincident neighbours: skipped pairs
    ri, _ = oracle.knn(X, k)
    ref = oracle.abod_from_knn(X, ri)
    with _ctx(pkg) as ctx:
        s, res, st = ctx.abod(torch.from_numpy(X).cuda(), k, want_knn=("idx",))
    assert np.array_equal(_np(res.idx), ri)
    assert np.array_equal(_np(s), ref)


def test_abod_query_range_host_buffers(pkg):
    X = datagen.gaussian_mixture(12_000, 32, seed=4)       # two-pass kNN path
    rows = np.arange(3000, 3400)
    ri, _ = oracle.knn(X, 8, rows=rows)
    with _ctx(pkg) as ctx:
        s, _, _ = ctx.abod(X, 8, q_begin=3000, q_count=400)
    assert np.array_equal(s, oracle.abod_from_knn(X, ri, rows=rows))


def test_knn_classify_parity(pkg):
    rng = np.random.default_rng(3)
    Xtr = datagen.gaussian_mixture(5000, 24, seed=11)
    ytr = rng.integers(0, 4, 5000).astype(np.int32)
    Xte = datagen.gaussian_mixture(700, 24, seed=12)
    for k in (1, 6, 15):
        ri, _ = oracle.knn_query(Xte, Xtr, k)
        ref = oracle.knn_classify(ri, ytr)
        with _ctx(pkg) as ctx:
            pred = ctx.knn_classify(torch.from_numpy(Xte).cuda(), torch.from_numpy(Xtr).cuda(), ytr, k)
        assert np.array_equal(_np(pred), ref), k


# ------------------------------------------------ detector wrapper (NEXT-4)
def test_detectors_fit_labels_auc(pkg):
    from sklearn.metrics import roc_auc_score
    from paper_2110_14007_b200 import detectors
    X, lab = datagen.gaussian_mixture(6000, 16, seed=2, return_labels=True)
    k = 10
    ri, rd = oracle.knn(X, k)
    kth, mean = oracle.scores(rd)
    _, lof_ref = oracle.lof_from_knn(ri, rd)
    for det, ref in ((detectors.KNN(k, contamination=0.05), kth),
                     (detectors.KNN(k, method="mean", contamination=0.05), mean),
                     (detectors.LOF(k, contamination=0.05), lof_ref.astype(np.float32))):
        det.fit(torch.from_numpy(X).cuda())
        assert np.array_equal(det.decision_scores_.astype(np.float32), ref)
        assert abs(det.labels_.mean() - 0.05) < 0.01
        assert roc_auc_score(lab, det.decision_scores_) == roc_auc_score(lab, ref)
        assert roc_auc_score(lab, det.decision_scores_) > 0.9
        det.close()
    abod = detectors.ABOD(k, contamination=0.05).fit(torch.from_numpy(X).cuda())
    assert np.array_equal(abod.decision_scores_.astype(np.float32), oracle.abod_from_knn(X, ri))
    assert roc_auc_score(lab, abod.decision_scores_) > 0.8


def test_detector_decision_function_matches_query_oracle(pkg):
    from paper_2110_14007_b200 import detectors
    X = datagen.gaussian_mixture(4000, 24, seed=5)
    Xt = datagen.gaussian_mixture(300, 24, seed=6)
    det = detectors.KNN(7).fit(torch.from_numpy(X).cuda())
    s = det.decision_function(torch.from_numpy(Xt).cuda())
    ri, rd = oracle.knn_query(Xt, X, 7)
    assert np.array_equal(s.astype(np.float32), oracle.scores(rd)[0])
    assert np.array_equal(det.predict(torch.from_numpy(Xt).cuda()), (s > det.threshold_).astype(np.int64))
    det.close()


def test_forced_fallback_more_rows_than_grid_y(pkg):
    # > 65535 failing rows: the fallback grids put rows on x (gridDim.y <= 65535)
    n, k = 70_000, 5
    X = datagen.gaussian_mixture(n, 16, seed=17)
    with _ctx(pkg, flags=pkg.F_NO_CERTIFY) as ctx:
        res = ctx.knn(torch.from_numpy(X).cuda(), k)
    assert res.stats["fallback_rows"] == n
    rows = np.random.default_rng(0).choice(n, 64, replace=False)
    _check_rows(res, X, k, rows)


@pytest.mark.parametrize("dt", ["float16", "bfloat16"])
def test_tensor_core_accumulation_model(pkg, dt):
    # Reading A9: the certificate bounds the fp32 tensor-core accumulation error
    # by 17 ceil(K/16) 2^-23 sum|A B| (alignment-truncation model).  Guard it on
    # this device with cuBLAS tcgen05 GEMMs too (the library's own kernels are
    # checked by test_certificate_bound_on_product_kernel): the measured worst
    # error must stay below half the model.
    dtype = getattr(torch, dt)
    g = torch.Generator(device="cuda").manual_seed(1)
    for K in (48, 80, 144, 528):
        model = 17 * ((K + 15) // 16) * 2.0   # in units of 2^-24
        worst = 0.0
        for trial in range(3):
            A = torch.randn(1024, K, generator=g, device="cuda")
            B = torch.randn(1024, K, generator=g, device="cuda")
            if trial == 1:
                A, B = A + 30, -(B + 30)
            if trial == 2:
                A = A * torch.exp2(torch.randint(-8, 8, A.shape, generator=g, device="cuda").float())
            A, B = A.to(dtype), B.to(dtype)
            C = torch.mm(A, B.t(), out_dtype=torch.float32).double()
            Ad, Bd = A.double(), B.double()
            err = (C - Ad @ Bd.t()).abs() / (Ad.abs() @ Bd.abs().t() * 2.0 ** -24)
            worst = max(worst, err.max().item())
        assert worst < model / 2, (K, worst, model)


# ------------------------------------------------ automatic batching (workspace_bytes)
@pytest.mark.parametrize("d,fmt", [(32, "fp16"), (64, "bf16"), (10, "auto")])
def test_workspace_budget_chunks_queries_bit_identical(pkg, d, fmt):
    # SURVEY 8(a) level 3: a small workspace budget splits the query rows into
    # 128-row-multiple chunks; every output equals the unchunked call bit for bit
    n, k = 12_345, 15
    X = torch.from_numpy(datagen.gaussian_mixture(n, d, seed=3 + d)).cuda()
    with _ctx(pkg, fmt=fmt) as ctx:
        ref = ctx.knn(X, k)
        ref_q = ctx.knn_query(X[:1000] + 0.25, X, k)
        lof_ref = ctx.lof(X, k)
    with _ctx(pkg, fmt=fmt, workspace_bytes=3 << 20) as ctx:
        got = ctx.knn(X, k, q_begin=77, q_count=n - 77)
        got_q = ctx.knn_query(X[:1000] + 0.25, X, k)
        lof_got = ctx.lof(X, k)
    assert got.stats["query_chunks"] > 2, got.stats["query_chunks"]
    assert got.stats["rows"] == n - 77
    for f in ("idx", "dist", "dist64", "score_kth", "score_mean", "kdist64"):
        assert torch.equal(getattr(got, f), getattr(ref, f)[77:]), f
        assert torch.equal(getattr(got_q, f), getattr(ref_q, f)), f
    assert torch.equal(lof_got[0], lof_ref[0]) and torch.equal(lof_got[1], lof_ref[1])
    assert lof_got[3]["query_chunks"] > 2
    _check_rows(ref, _np(X), k, np.arange(0, n, n // 8))


@pytest.mark.parametrize("n,d,k", [(20_000, 32, 20), (9000, 300, 12)])
def test_split_rerank_matches_one_kernel_rerank(pkg, n, d, k, monkeypatch):
    # the split re-rank (plan -> flat expansion -> finish; default at d > 256) and
    # the one-kernel re-rank keep the same columns: outputs bit-identical, both
    # equal to the oracle on sampled rows
    X = torch.from_numpy(datagen.gaussian_mixture(n, d, seed=11 + d)).cuda()
    res = {}
    for split in ("0", "1"):
        monkeypatch.setenv("TOD_RR_SPLIT", split)
        with _ctx(pkg, fmt="fp16") as ctx:
            res[split] = ctx.knn(X, k)
    for f in ("idx", "dist64", "score_mean"):
        assert torch.equal(getattr(res["0"], f), getattr(res["1"], f)), f
    assert res["0"].stats["certified"] == res["1"].stats["certified"]
    _check_rows(res["1"], _np(X), k, np.arange(0, n, n // 6))


@pytest.mark.parametrize("case", ["mixture", "duplicates"])
def test_bf16_second_tier_matches_brute_force_tier(pkg, case, monkeypatch):
    # rows a bf16 pass cannot certify are re-answered by the fp16 pass on just
    # those rows (self dropped from k+1 neighbours); the outputs must equal the
    # fp64 brute-force tier's bit for bit, including rows with exact duplicates
    if case == "mixture":
        X = datagen.gaussian_mixture(60_000, 64, seed=8)
    else:
        X = datagen.with_duplicates(datagen.lattice(20_000, 64, seed=9, extent=3), frac=0.2, seed=10)
    Xd = torch.from_numpy(X).cuda()
    k = 10
    # duplicates: every row forced through the tiers (TOD_F_NO_CERTIFY; knob 2 keeps
    # the second tier on), so the self-drop among exact-duplicate neighbours runs
    flags, on = (0, "1") if case == "mixture" else (pkg.F_NO_CERTIFY, "2")
    res = {}
    for t2 in (on, "0"):
        monkeypatch.setenv("TOD_TIER2", t2)
        with _ctx(pkg, fmt="bf16", flags=flags) as ctx:
            res[t2] = ctx.knn(Xd, k)
    res["1"] = res[on]
    if case == "duplicates":  # query mode (no self to drop) through the same tier
        q = {}
        for t2 in (on, "0"):
            monkeypatch.setenv("TOD_TIER2", t2)
            with _ctx(pkg, fmt="bf16", flags=flags) as ctx:
                q[t2] = ctx.knn_query(Xd[:3000], Xd, k)
        for f in ("idx", "dist64", "score_mean"):
            assert torch.equal(getattr(q[on], f), getattr(q["0"], f)), f
    assert res["1"].stats["fallback_rows"] == res["0"].stats["fallback_rows"]
    print("bf16 uncertified rows:", res["1"].stats["fallback_rows"])
    for f in ("idx", "dist", "dist64", "score_kth", "score_mean", "kdist64"):
        assert torch.equal(getattr(res["1"], f), getattr(res["0"], f)), f
    _check_rows(res["1"], X, k, np.arange(0, X.shape[0], X.shape[0] // 8))


@pytest.mark.parametrize("case", ["mixture", "duplicates"])
def test_fp16_second_tier_matches_brute_force_tier(pkg, case, monkeypatch):
    # rows an fp16 two-pass call cannot certify are re-answered by the same path
    # on just those rows with twice its K' (references reused); outputs must
    # equal the fp64 tiers' bit for bit.  K' = 12 for k = 10 leaves many rows
    # uncertified by pass 1.
    if case == "mixture":  # TOD_TIER2=2: the re-run regardless of its cost estimate
        X = datagen.gaussian_mixture(40_000, 32, seed=18)
        flags, on = 0, "2"
    else:
        X = datagen.with_duplicates(datagen.lattice(20_000, 32, seed=19, extent=3), frac=0.2, seed=20)
        flags, on = pkg.F_NO_CERTIFY, "2"
    Xd = torch.from_numpy(X).cuda()
    k = 10
    res = {}
    for t2 in (on, "0"):
        monkeypatch.setenv("TOD_TIER2", t2)
        with _ctx(pkg, fmt="fp16", kprime=12, flags=flags) as ctx:
            res[t2] = ctx.knn(Xd, k, want=("idx", "dist", "dist64", "score_kth", "score_mean",
                                           "kdist64", "row_tier"))
    assert res[on].stats["fallback_rows"] == res["0"].stats["fallback_rows"] > 0
    tier = _np(res[on].row_tier)
    assert (tier == 1).sum() == res[on].stats["fallback_rows"], "every failing row went to the second tier"
    for f in ("idx", "dist", "dist64", "score_kth", "score_mean", "kdist64"):
        assert torch.equal(getattr(res[on], f), getattr(res["0"], f)), f
    rows = np.unique(np.concatenate([np.arange(0, X.shape[0], X.shape[0] // 8),
                                     np.nonzero(tier)[0][:200]]))
    _check_rows(res[on], X, k, rows)


def test_abod_weighted_golden_on_gpu(pkg, golden_dir):
    # the non-unit hand golden (tests/golden/abod_clf_examples.json): -2/81, not the
    # plain-cosine -2/9 (reading A20)
    import json
    g = json.load(open(os.path.join(golden_dir, "abod_clf_examples.json")))
    X = np.array(g["abod_weighted_X"], np.float32)
    with _ctx(pkg) as ctx:
        s, _, _ = ctx.abod(torch.from_numpy(X).cuda(), g["abod_weighted_k"])
    assert _np(s)[0] == np.float32(g["abod_weighted_row0"])
