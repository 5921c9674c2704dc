"""GPU tests of the sharded multi-GPU path (tod_knn_sharded / tod_lof_sharded,
SURVEY §8(e), §6.2) on ONE B200: the loopback transport runs
W virtual ranks in this process with the real ring schedule (blocks circulate,
global statistics are gathered / max-reduced, X is all-gathered for the re-rank)
and every collective replaced by device copies; a real NCCL communicator of one
rank exercises the NCCL plumbing.  Bar: outputs bit-identical to the
single-process call (and hence to the oracle) for every W."""
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


def _np(x):
    return x.cpu().numpy() if hasattr(x, "cpu") else np.asarray(x)


WANT = ("idx", "dist64", "score_kth", "score_mean", "kdist64", "row_tier")


def _single(pkg, Xd, k, fmt):
    with pkg.Context(device=0, fmt=fmt) as ctx:
        return ctx.knn(Xd, k, want=WANT)


@pytest.mark.parametrize("n,d,k,fmt,W", [
    (20_000, 32, 20, "fp16", 1),
    (20_000, 32, 20, "fp16", 2),
    (20_000, 32, 20, "fp16", 3),
    (20_000 + 77, 32, 20, "fp16", 5),     # ragged last block
    (30_000, 64, 10, "bf16", 3),          # CTA-pair main pass + bf16 second tier
    (24_000, 64, 20, "fp16", 4),
    (12_000, 128, 16, "fp16", 2),         # K-pipelined main pass
])
def test_loopback_ring_bit_identical(pkg, n, d, k, fmt, W):
    X = datagen.gaussian_mixture(n, d, seed=3)
    Xd = torch.from_numpy(X).cuda()
    ref = _single(pkg, Xd, k, fmt)
    with pkg.Context(device=0, fmt=fmt) as ctx:
        ctx.comm_init_loopback(W)
        res, kth, mean = ctx.knn_sharded(Xd, n, 0, k, want=WANT)
    for f in ("idx", "dist64", "score_kth", "score_mean", "kdist64"):
        assert np.array_equal(_np(getattr(res, f)), _np(getattr(ref, f))), f
    assert np.array_equal(_np(kth), _np(ref.score_kth))
    assert np.array_equal(_np(mean), _np(ref.score_mean))
    # the ring really ran (not the replicated fallback) and answered every row
    assert res.stats["main_kernel"] in (3, 4) and res.stats["sample_pass"] == 2
    assert res.stats["certified"] + res.stats["fallback_rows"] == n
    # sampled rows against the oracle too, including every row not certified by pass 1
    tier = _np(res.row_tier)
    rows = np.unique(np.concatenate([np.random.default_rng(0).choice(n, 64, replace=False),
                                     np.nonzero(tier)[0][:64]]))
    ri, rd = oracle.knn(X, k, rows=rows)
    assert np.array_equal(_np(res.idx)[rows], ri)
    assert np.array_equal(_np(res.dist64)[rows], np.sqrt(rd))


@pytest.mark.parametrize("W", [2, 4])
def test_loopback_lof_bit_identical(pkg, W):
    n, d, k = 16_000, 32, 20
    X = datagen.gaussian_mixture(n, d, seed=5)
    Xd = torch.from_numpy(X).cuda()
    with pkg.Context(device=0) as ctx:
        lof_ref, lrd_ref, _, _ = ctx.lof(Xd, k)
    with pkg.Context(device=0) as ctx:
        ctx.comm_init_loopback(W)
        lof, lrd, _, st = ctx.lof_sharded(Xd, n, 0, k)
    assert np.array_equal(_np(lof), _np(lof_ref))
    assert np.array_equal(_np(lrd), _np(lrd_ref))
    rows = np.random.default_rng(1).choice(n, 40, replace=False)
    ref = oracle.lof_rows(X, k, rows)
    assert np.array_equal(_np(lof)[rows], ref["lof"].astype(np.float32))


def test_loopback_small_problem_replicated_form(pkg):
    # n too small for the two-pass plan: every virtual rank answers its rows
    # against the gathered X (no ring); still bit-identical
    n, d, k = 3000, 16, 8
    X = datagen.gaussian_mixture(n, d, seed=9)
    Xd = torch.from_numpy(X).cuda()
    ref = _single(pkg, Xd, k, "auto")
    with pkg.Context(device=0) as ctx:
        ctx.comm_init_loopback(3)
        res, kth, _ = ctx.knn_sharded(Xd, n, 0, k, want=WANT)
    assert np.array_equal(_np(res.idx), _np(ref.idx))
    assert np.array_equal(_np(kth), _np(ref.score_kth))


def test_loopback_duplicates_and_host_buffers(pkg):
    n, d, k = 20_000, 32, 10
    X = datagen.with_duplicates(datagen.gaussian_mixture(n, d, seed=11), frac=0.05, seed=2)
    ref = _single(pkg, torch.from_numpy(X).cuda(), k, "fp16")
    with pkg.Context(device=0, fmt="fp16") as ctx:
        ctx.comm_init_loopback(3)
        res, kth, mean = ctx.knn_sharded(X, n, 0, k, want=WANT)   # numpy: host buffers
    assert np.array_equal(res.idx, _np(ref.idx))
    assert np.array_equal(kth, _np(ref.score_kth))


def test_nccl_single_rank_communicator(pkg):
    # the NCCL plumbing (dlopen of the process's libnccl, id, CommInitRank,
    # all-gathers / all-reduces of one rank) with a real communicator
    n, d, k = 20_000, 32, 20
    X = datagen.gaussian_mixture(n, d, seed=4)
    Xd = torch.from_numpy(X).cuda()
    ref = _single(pkg, Xd, k, "fp16")
    cid = pkg.comm_id_create()
    assert len(cid) == 128
    with pkg.Context(device=0, fmt="fp16") as ctx:
        ctx.comm_init(0, 1, cid)
        res, kth, _ = ctx.knn_sharded(Xd, n, 0, k, want=WANT)
        lof, _, _, _ = ctx.lof_sharded(Xd, n, 0, k)
    assert np.array_equal(_np(res.idx), _np(ref.idx))
    assert np.array_equal(_np(kth), _np(ref.score_kth))
    with pkg.Context(device=0, fmt="fp16") as ctx:
        lof_ref, _, _, _ = ctx.lof(Xd, k)
    assert np.array_equal(_np(lof), _np(lof_ref))


def test_sharded_argument_errors(pkg):
    X = torch.from_numpy(datagen.gaussian_mixture(5000, 16, seed=1)).cuda()
    with pkg.Context(device=0) as ctx:
        ctx.comm_init_loopback(2)
        with pytest.raises(pkg.TodError) as e:
            ctx.knn_sharded(X[256:], 5000, 256, 5)   # loopback takes all rows
        assert e.value.status == -1
        with pytest.raises(pkg.TodError) as e:
            ctx.knn_sharded(X, 5000, 0, pkg.MAX_K + 1)
        assert e.value.status == -7
