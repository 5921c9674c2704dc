"""SPMD multi-GPU orchestration: one process per GPU (§6.2, P:475-484:
"subtasks are split equally", one subprocess per GPU; here torch.distributed
with NCCL between B200s, gloo in CPU tests).

Two forms:

* The RING (north_star): each rank holds only its row
  block X_r; ``init_comm`` attaches the library's own NCCL communicator (id
  broadcast through the torch process group), and ``knn_ring`` / ``lof_ring``
  call tod_knn_sharded / tod_lof_sharded, where the quantized reference blocks
  circulate over NCCL send/recv with a running candidate state and the scores
  are all-gathered -- all inside libtod.so.

* The REPLICATED form below (``knn_scores`` / ``lof_scores``): every rank holds
  all of X and answers its query rows [begin_r, begin_r + count_r); the only
  exchanges are the real ones of the method:
  * kNN scores / neighbour tables -> all_gather (output assembly);
  * LOF: all_gather of the k-distances before the lrd stage, and of lrd before
    the final ratio (reach-dist and LOF of a row read its neighbours' values,
    which live on other ranks).
Results are bit-identical for every world size: each row's computation does not
depend on which rank runs it.

The per-rank compute is injected (``stages``): on GPUs it is ``CudaStages``
(libtod.so via the C ABI); the CPU tests inject the oracle.  This module holds
no arithmetic of the method.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

ROW_ALIGN = 256  # reference tile: shard edges on tile boundaries (= tod_shard_rows)


def shard_rows(n: int, world: int, rank: int, align: int = ROW_ALIGN):
    """Contiguous, tile-aligned, balanced shard [begin, begin+count) of n rows."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank/world")
    tiles = (n + align - 1) // align
    t0 = tiles * rank // world
    t1 = tiles * (rank + 1) // world
    begin = min(n, t0 * align)
    end = min(n, t1 * align)
    return begin, end - begin


def _gather_rows(local: torch.Tensor, n: int, world: int, group=None) -> torch.Tensor:
    """all_gather variable-length row shards (dim 0) into the full [n, ...] tensor."""
    counts = [shard_rows(n, world, r)[1] for r in range(world)]
    m = max(counts)
    pad = torch.zeros((m,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([b[:c] for b, c in zip(bufs, counts)], dim=0)


class CudaStages:
    """Per-rank compute through libtod.so (device tensors in, device tensors out)."""

    def __init__(self, ctx):
        self.ctx = ctx

    def knn(self, X, k, q_begin, q_count):
        r = self.ctx.knn(X, k, q_begin, q_count,
                         want=("idx", "dist64", "score_kth", "score_mean", "kdist64"))
        return {"idx": r.idx, "dist64": r.dist64, "score_kth": r.score_kth,
                "score_mean": r.score_mean, "kdist64": r.kdist64, "stats": r.stats}

    def lof_lrd(self, n, k, idx, dist64, kdist64_all):
        return self.ctx.lof_lrd(n, k, idx, dist64, kdist64_all)

    def lof_finish(self, n, k, q_begin, idx, lrd64_all):
        return self.ctx.lof_finish(n, k, q_begin, idx, lrd64_all)


def knn_scores(X, k: int, stages, group=None, gather_tables: bool = False):
    """Sharded kNN outlier scores.  Returns dict with full-length score_kth and
    score_mean on every rank (plus idx/dist64 when gather_tables)."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    n = X.shape[0]
    b, c = shard_rows(n, world, rank)
    loc = stages.knn(X, k, b, c)
    if world == 1:
        return loc
    out = {"score_kth": _gather_rows(loc["score_kth"], n, world, group),
           "score_mean": _gather_rows(loc["score_mean"], n, world, group),
           "stats": loc.get("stats")}
    if gather_tables:
        out["idx"] = _gather_rows(loc["idx"], n, world, group)
        out["dist64"] = _gather_rows(loc["dist64"], n, world, group)
    return out


def lof_scores(X, k: int, stages, group=None):
    """Sharded LOF (kNN shard -> all_gather kdist -> lrd shard -> all_gather lrd
    -> LOF shard -> all_gather LOF).  Returns (lof fp32[n], lrd fp32[n])."""
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    n = X.shape[0]
    b, c = shard_rows(n, world, rank)
    loc = stages.knn(X, k, b, c)
    kd_all = _gather_rows(loc["kdist64"], n, world, group) if world > 1 else loc["kdist64"]
    lrd_loc = stages.lof_lrd(n, k, loc["idx"], loc["dist64"], kd_all)
    lrd_all = _gather_rows(lrd_loc, n, world, group) if world > 1 else lrd_loc
    lof_loc, lrd32_loc = stages.lof_finish(n, k, b, loc["idx"], lrd_all)
    if world == 1:
        return lof_loc, lrd32_loc
    return _gather_rows(lof_loc, n, world, group), _gather_rows(lrd32_loc, n, world, group)


# ------------------------------------------------------------------ the ring
def init_comm(ctx, group=None):
    """Attach an NCCL communicator over the process group's ranks to ``ctx``
    (tod_comm_init): rank 0 creates the id, the group broadcasts it."""
    from . import tod
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    obj = [tod.comm_id_create() if rank == 0 else None]
    dist.broadcast_object_list(obj, src=0, group=group)
    ctx.comm_init(rank, world, obj[0])
    return rank, world


def local_block(X, world: int, rank: int):
    """(X_local, row_offset) of this rank's 256-row-aligned block of X."""
    b, c = shard_rows(X.shape[0], world, rank)
    return X[b:b + c], b


def knn_ring(ctx, X_local, n: int, row_offset: int, k: int, want=("idx", "dist64")):
    """Sharded kNN through the library's NCCL ring: (local KnnResult,
    score_kth[n], score_mean[n]) with the scores of all rows."""
    return ctx.knn_sharded(X_local, n, row_offset, k, want=want, gather_scores=True)


def lof_ring(ctx, X_local, n: int, row_offset: int, k: int):
    """Sharded LOF through the library's NCCL ring: (lof[n], lrd[n], stats)."""
    lof, lrd, _, st = ctx.lof_sharded(X_local, n, row_offset, k)
    return lof, lrd, st
