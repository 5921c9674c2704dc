"""Multi-process (world_size 2, gloo, CPU) tests of the SPMD host logic in
paper_2110_14007_b200/dist.py: tile-aligned sharding, variable-length
all-gathers, and the sharded LOF stage order (kNN shard -> all-gather kdist ->
lrd shard -> all-gather lrd -> LOF shard).  The per-rank compute is the CPU
oracle injected through the same `stages` interface the CUDA path uses, so the
result must equal the single-process oracle bit for bit."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import datagen
import oracle
from paper_2110_14007_b200 import dist as tdist


class OracleStages:
    """The `stages` interface implemented with the CPU oracle (tests only)."""

    def knn(self, X, k, q_begin, q_count):
        Xn = X.numpy()
        idx, d64 = oracle.knn(Xn, k, rows=np.arange(q_begin, q_begin + q_count))
        kth, mean = oracle.scores(d64)
        dist64 = np.sqrt(d64)
        return {"idx": torch.from_numpy(idx), "dist64": torch.from_numpy(dist64),
                "score_kth": torch.from_numpy(kth), "score_mean": torch.from_numpy(mean),
                "kdist64": torch.from_numpy(dist64[:, k - 1].copy())}

    def lof_lrd(self, n, k, idx, dist64, kdist64_all):
        kd = kdist64_all.numpy()
        ii, dd = idx.numpy(), dist64.numpy()
        s = np.zeros(ii.shape[0])
        for m in range(k):
            s = s + np.maximum(kd[ii[:, m]], dd[:, m])
        lrd = np.full(ii.shape[0], np.inf)
        lrd[s > 0] = float(k) / s[s > 0]
        return torch.from_numpy(lrd)

    def lof_finish(self, n, k, q_begin, idx, lrd64_all):
        la = lrd64_all.numpy()
        ii = idx.numpy()
        lp = la[q_begin:q_begin + ii.shape[0]]
        ls = np.zeros(ii.shape[0])
        for m in range(k):
            ls = ls + la[ii[:, m]]
        lof = np.ones(ii.shape[0])
        fin = np.isfinite(lp)
        lof[fin] = ls[fin] / (float(k) * lp[fin])
        return torch.from_numpy(lof.astype(np.float32)), torch.from_numpy(lp.astype(np.float32))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, d, k, out_q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        X = torch.from_numpy(datagen.gaussian_mixture(n, d, seed=5))
        st = OracleStages()
        sc = tdist.knn_scores(X, k, st, gather_tables=True)
        lof, lrd = tdist.lof_scores(X, k, st)
        out_q.put((rank, sc["score_kth"].numpy(), sc["score_mean"].numpy(), sc["idx"].numpy(),
                   lof.numpy(), lrd.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(2, 700), (3, 1000)])
def test_sharded_knn_and_lof_equal_single_process(world, n):
    d, k = 6, 9
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, d, k, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    X = datagen.gaussian_mixture(n, d, seed=5)
    idx, d64 = oracle.knn(X, k)
    kth, mean = oracle.scores(d64)
    lrd, lof = oracle.lof_from_knn(idx, d64)
    for _, skth, smean, sidx, slof, slrd in res:   # every rank holds the full result
        assert np.array_equal(skth, kth) and np.array_equal(smean, mean)
        assert np.array_equal(sidx, idx)
        assert np.array_equal(slof, lof.astype(np.float32))
        assert np.array_equal(slrd, lrd.astype(np.float32))


def test_shard_rows_tile_aligned_and_complete():
    for n in (1, 127, 128, 1000, 100_000, 1_000_003):
        for world in (1, 2, 3, 4, 8):
            spans = [tdist.shard_rows(n, world, r) for r in range(world)]
            assert spans[0][0] == 0
            pos = 0
            for b, c in spans:
                assert b == pos and c >= 0
                assert b % tdist.ROW_ALIGN == 0 or c == 0
                pos = b + c
            assert pos == n
            counts = [c for _, c in spans]
            assert max(counts) - min(counts) <= tdist.ROW_ALIGN


def test_library_shard_rows_matches_dist_split():
    # tod_shard_rows is host-only: callable without a GPU
    from paper_2110_14007_b200 import build
    build.build()
    import paper_2110_14007_b200 as pkg
    for n in (1, 255, 256, 257, 20_077, 1_000_000, 10_000_000):
        for world in (1, 2, 3, 5, 8):
            spans = [pkg.shard_rows(n, world, r) for r in range(world)]
            assert spans == [tdist.shard_rows(n, world, r) for r in range(world)]
            off = 0
            for b, c in spans:
                assert b == off and b % 256 == 0
                off += c
            assert off == n


def test_workspace_size_estimate():
    from paper_2110_14007_b200 import build
    build.build()
    import paper_2110_14007_b200 as pkg
    a = pkg.workspace_size(1_000_000, 64, 10, 1_000_000, fmt="bf16")
    b = pkg.workspace_size(1_000_000, 64, 10, 500_000, fmt="bf16")
    assert a > b > 0
    # the reference image alone (n x (64+16) x 2 bytes) is a lower bound
    assert b > 1_000_000 * 80 * 2
    assert pkg.workspace_size(1, 64, 10, 1) == 0   # n < 2: invalid
