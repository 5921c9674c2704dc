"""GPU parity at BASELINE.json's full sizes, in the launch configuration bench.py
times (VERDICT r01 "Harden parity where the risky code runs"):

  C2  n=100,000 d=32 k=20 kNN + LOF: EVERY row (the oracle's full table), and LOF
      of every row, through tod_lof (bench N=1) and the loopback ring (bench N>1);
  C3  n=1,000,000 d=64 k=10: >= 1000 seeded rows (a quarter outliers) in BOTH bf16
      and fp16, plus EVERY row the low-precision pass did not certify (row_tier);
  C4  n=10,000,000 d=64 k=20: rank 0's 1/8 query shard (bench --config c4 at N=1),
      >= 256 rows incl. outliers plus every uncertified row of the shard;
  C5  n=2,000,000 d=512 k=50: >= 256 rows plus every uncertified row.

Bar (BASELINE north_star): indices bit-exact, order included; fp32 scores within
1e-5 relative -- here bit-identical, because the re-rank evaluates the oracle's own
fp64 formula."""
import numpy as np
import pytest

import datagen
import oracle

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

WANT = ("idx", "dist", "dist64", "score_kth", "score_mean", "row_tier")


@pytest.fixture(scope="module")
def pkg():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2110_14007_b200 import build
    build.build()
    import paper_2110_14007_b200 as p
    return p


def _np(x):
    return x.cpu().numpy() if hasattr(x, "cpu") else np.asarray(x)


def _check(res, rows, ri, rd, q_begin=0):
    loc = np.asarray(rows) - q_begin
    gi = _np(res.idx)[loc]
    bad = np.nonzero((gi != ri).any(1))[0]
    assert bad.size == 0, "rows %s: gpu %s oracle %s" % (np.asarray(rows)[bad[:3]], gi[bad[:1]],
                                                          ri[bad[:1]])
    assert np.array_equal(_np(res.dist64)[loc], np.sqrt(rd))
    assert np.array_equal(_np(res.dist)[loc], np.sqrt(rd).astype(np.float32))
    kth, mean = oracle.scores(rd)
    assert np.array_equal(_np(res.score_kth)[loc], kth)
    assert np.array_equal(_np(res.score_mean)[loc], mean)


def _rows(n, labels, m, seed, extra=()):
    rng = np.random.default_rng(seed)
    out_rows = np.nonzero(labels)[0]
    rows = np.concatenate([rng.choice(n, m - m // 4, replace=False),
                           rng.choice(out_rows, m // 4, replace=False), [0, n - 1],
                           np.asarray(extra, dtype=np.int64)])
    return np.unique(rows)


# ------------------------------------------------------------------ C2
@pytest.fixture(scope="module")
def c2():
    X = datagen.gaussian_mixture(100_000, 32, seed=0)
    idx, d64 = oracle.knn(X, 20)               # every row (~100 s on 16 host cores)
    _, lof = oracle.lof_from_knn(idx, d64)
    return X, idx, d64, lof


def test_c2_every_row_and_lof(pkg, c2):
    X, ri, rd, rlof = c2
    with pkg.Context(device=0) as ctx:       # bench.py N=1: tod_lof
        lof, lrd, res, st = ctx.lof(torch.from_numpy(X).cuda(), 20, want_knn=WANT)
    _check(res, np.arange(100_000), ri, rd)
    assert np.array_equal(_np(lof), rlof.astype(np.float32))
    assert st["certified"] >= 0.999 * 100_000, st


def test_c2_lof_through_the_ring(pkg, c2):
    X, ri, rd, rlof = c2
    with pkg.Context(device=0) as ctx:       # bench.py N>1: tod_lof_sharded (loopback ring)
        ctx.comm_init_loopback(4)
        lof, lrd, res, st = ctx.lof_sharded(torch.from_numpy(X).cuda(), 100_000, 0, 20,
                                            want_knn=WANT)
    _check(res, np.arange(100_000), ri, rd)
    assert np.array_equal(_np(lof), rlof.astype(np.float32))


def test_c2_replicated_orchestration(pkg, c2):
    # dist.lof_scores with CudaStages (tod_knn -> tod_lof_lrd -> tod_lof_finish)
    from paper_2110_14007_b200 import dist as tdist
    X, _, _, rlof = c2
    with pkg.Context(device=0) as ctx:
        lof, _ = tdist.lof_scores(torch.from_numpy(X).cuda(), 20, tdist.CudaStages(ctx))
    assert np.array_equal(_np(lof), rlof.astype(np.float32))


# ------------------------------------------------------------------ C3
@pytest.fixture(scope="module")
def c3():
    X, lab = datagen.gaussian_mixture(1_000_000, 64, seed=0, return_labels=True)
    return X, lab, {}


def _oracle_rows(cache, X, k, rows):
    need = [r for r in rows if r not in cache]
    if need:
        ri, rd = oracle.knn(X, k, rows=np.asarray(need))
        for r, a, b in zip(need, ri, rd):
            cache[r] = (a, b)
    return np.stack([cache[r][0] for r in rows]), np.stack([cache[r][1] for r in rows])


@pytest.mark.parametrize("fmt", ["bf16", "fp16"])
def test_c3_rows_and_every_uncertified_row(pkg, c3, fmt):
    X, lab, cache = c3
    with pkg.Context(device=0, fmt=fmt) as ctx:     # bench.py default: tod_knn, all rows
        res = ctx.knn(torch.from_numpy(X).cuda(), 10, want=WANT)
    tier = _np(res.row_tier)
    unc = np.nonzero(tier)[0]
    assert unc.size == res.stats["fallback_rows"]
    rows = _rows(1_000_000, lab, 1000, seed=2, extra=unc)
    ri, rd = _oracle_rows(cache, X, 10, rows)
    _check(res, rows, ri, rd)
    if fmt == "bf16":
        assert (tier == 1).sum() > 0       # the fp16 second tier answered rows here
    print("C3 %s: %d rows checked, %d uncertified" % (fmt, rows.size, unc.size))


# ------------------------------------------------------------------ C4 shard
def test_c4_rank0_shard(pkg):
    n, d, k = 10_000_000, 64, 20
    X, lab = datagen.gaussian_mixture(n, d, seed=0, return_labels=True)
    b, c = pkg.shard_rows(n, 8, 0)
    with pkg.Context(device=0, fmt="fp16") as ctx:  # bench.py --config c4 at N=1
        res = ctx.knn(torch.from_numpy(X).cuda(), k, b, c, want=WANT)
    unc = np.nonzero(_np(res.row_tier))[0] + b
    rng = np.random.default_rng(4)
    in_shard_out = np.nonzero(lab[b:b + c])[0] + b
    rows = np.unique(np.concatenate([rng.choice(np.arange(b, b + c), 192, replace=False),
                                     rng.choice(in_shard_out, 64, replace=False), unc[:256]]))
    ri, rd = oracle.knn(X, k, rows=rows)
    _check(res, rows, ri, rd, q_begin=b)
    print("C4 shard: %d rows checked, %d uncertified" % (rows.size, unc.size))


# ------------------------------------------------------------------ C5
def test_c5_full_size(pkg):
    n, d, k = 2_000_000, 512, 50
    X, lab = datagen.gaussian_mixture(n, d, seed=0, return_labels=True)
    with pkg.Context(device=0, fmt="fp16") as ctx:
        res = ctx.knn(torch.from_numpy(X).cuda(), k, want=WANT)
    unc = np.nonzero(_np(res.row_tier))[0]
    rows = _rows(n, lab, 256, seed=5, extra=unc[:256])
    ri, rd = oracle.knn(X, k, rows=rows)
    _check(res, rows, ri, rd)
    print("C5: %d rows checked, %d uncertified" % (rows.size, unc.size))
