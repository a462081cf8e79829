"""Point-sharded multi-GPU Lloyd: one process per GPU, one NCCL allreduce per iteration.

The reference has no multi-device path.  On a B200 node the
path shards naturally: assignment is independent per point and
the update is a sum, so each rank owns a contiguous row range of every batch
element, runs assign + sort-inverse update locally, and the per-iteration
exchange is a single in-place all-reduce (sum) of one packed float64 buffer

    [ sums (B*K*d) | counts (B*K, exact as f64 below 2**53) | objective (B) | changed (1) ]

after which every rank runs the identical normalize, so the replicated
centroids never diverge.  Initial centroids follow the reference's row draws
over the GLOBAL point range (core.py:375-377); each row is contributed by the
rank that owns it through the same all-reduce primitive.
"""

from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

from .core import Assignments, Centroids, Counters, KMeansConfig, KMeansResult, init_indices
from .pipeline import LloydEngine

__all__ = ["shard_bounds", "make_allreduce", "init_centroids_sharded", "lloyd_run_sharded"]


def shard_bounds(points: int, world: int, rank: int) -> tuple[int, int]:
    """Rank r owns rows [r*N//P, (r+1)*N//P) of every batch element."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return points * rank // world, points * (rank + 1) // world


def make_allreduce(group=None):
    def allreduce(buf: torch.Tensor) -> None:
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)

    return allreduce


def init_centroids_sharded(x_shard: torch.Tensor, total_points: int, lo: int, clusters: int,
                           seed: int, method: str = "random_distinct", group=None) -> torch.Tensor:
    """Replicated initial centroids from a row-sharded dataset."""
    if method != "random_distinct":
        raise NotImplementedError("sharded k-means++ seeding is not implemented (SURVEY §8f rank 3)")
    B, n_local, d = x_shard.shape
    idx = init_indices(total_points, clusters, seed, B, method)
    buf = torch.zeros((B, clusters, d), dtype=torch.float64, device=x_shard.device)
    for b in range(B):
        sel = np.flatnonzero((idx[b] >= lo) & (idx[b] < lo + n_local))
        if sel.size:
            rows = torch.from_numpy(idx[b][sel] - lo).to(x_shard.device)
            buf[b, torch.from_numpy(sel).to(x_shard.device)] = x_shard[b].index_select(0, rows).double()
    dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    return buf


def lloyd_run_sharded(x_shard: torch.Tensor, total_points: int, lo: int, cfg: KMeansConfig,
                      update_chunk: int | None = None, group=None, backend=None,
                      counters: Counters | None = None) -> KMeansResult:
    """lloyd_run semantics (pipeline.py:110-147) over a row shard.

    Returns replicated centroids and objective history (global sums) and this
    rank's assignments (rows [lo, lo + n_local))."""
    counters = counters if counters is not None else Counters()
    eng = LloydEngine(x_shard, cfg.clusters, update_chunk or total_points,
                      allreduce=make_allreduce(group), backend=backend)
    eng.set_centroids(init_centroids_sharded(x_shard, total_points, lo, cfg.clusters, cfg.seed,
                                             cfg.init, group))
    history = torch.empty((cfg.max_iters, eng.B), dtype=torch.float64, device=x_shard.device)
    # every rank takes the same decisions: the flags are reduced in the exchange
    iterations, slot, merges = eng.run(cfg.max_iters, cfg.shift_tol, history)
    if x_shard.is_cuda:
        torch.cuda.synchronize(x_shard.device)
    # merges: each rank counted its own shard's segments; the reference count is global
    mg = torch.tensor([float(merges)], dtype=torch.float64, device=x_shard.device)
    dist.all_reduce(mg, op=dist.ReduceOp.SUM, group=group)
    counters.synchronized_merges += int(mg.item())
    return KMeansResult(Centroids(eng.centroids.clone(), check_finite=False),
                        Assignments(eng.ids[slot].clone(), validate=False),
                        history[:iterations].cpu().numpy(), iterations, counters)
