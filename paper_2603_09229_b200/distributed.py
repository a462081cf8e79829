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
from .pipeline import LloydEngine, _farthest

__all__ = ["shard_bounds", "make_allreduce", "init_centroids_sharded", "kmeanspp_indices_sharded",
           "reseed_farthest_sharded", "lloyd_run_sharded"]


def shard_bounds(points: int, world: int, rank: int) -> tuple[int, int]:
    """Rank r owns rows [r*N//P, (r+1)*N//P) of every batch element."""
    if not 0 <= rank < world:
        raise ValueError("rank out of range")
    return points * rank // world, points * (rank + 1) // world


def make_allreduce(group=None):
    def allreduce(buf: torch.Tensor) -> None:
        dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)

    return allreduce


def _center_row(x_shard: torch.Tensor, b: int, row: int, lo: int, group) -> torch.Tensor:
    """Global row `row` of batch element b, replicated on every rank (the owner
    contributes it through an all-reduce; f64 holds every data type exactly)."""
    n_local = x_shard.shape[1]
    v = torch.zeros((x_shard.shape[2],), dtype=torch.float64, device=x_shard.device)
    if lo <= row < lo + n_local:
        v.copy_(x_shard[b, row - lo].double())
    dist.all_reduce(v, op=dist.ReduceOp.SUM, group=group)
    return v.to(x_shard.dtype)


def kmeanspp_indices_sharded(x_shard: torch.Tensor, total_points: int, lo: int, clusters: int,
                             seed: int, group=None, backend=None) -> np.ndarray:
    """k-means++ seeding (core.py:342-357) over row shards, index for index equal
    to the single-process seeding.

    Every rank sweeps its own rows against the current center into its slice
    of the (N,) f64 weight table; the slices are all-gathered (one collective
    per draw), and every rank runs the identical numpy-order total and
    certified choice() on the full table.  So all ranks draw the same index
    without further communication.  The numpy substream (seed, b) is consumed
    on every rank exactly as the reference does."""
    from . import ops as _ops

    be = _ops if backend is None else backend
    B, n_local, d = x_shard.shape
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    bounds = [shard_bounds(total_points, world, r) for r in range(world)]
    if bounds[rank][0] != lo or bounds[rank][1] - bounds[rank][0] != n_local:
        raise ValueError("x_shard must be this rank's shard_bounds() rows")
    maxn = max(h - l for l, h in bounds)
    dev = x_shard.device
    out = np.empty((B, clusters), np.int64)
    for b in range(B):
        rng = np.random.default_rng((seed, b))
        idx = out[b]
        idx[0] = rng.integers(total_points)
        if clusters == 1:
            continue
        pp = be.KmeansppStream(total_points, clusters, dev)
        send = torch.zeros((maxn,), dtype=torch.float64, device=dev)
        recv = torch.empty((world * maxn,), dtype=torch.float64, device=dev)

        def sweep(row: int, first: bool, j: int) -> None:
            center = _center_row(x_shard, b, row, lo, group)
            if n_local:
                pp.sweep(x_shard[b], lo, center, first, j)
            send[:n_local].copy_(pp.m[0, lo:lo + n_local])
            dist.all_gather(list(recv.view(world, maxn).unbind(0)), send, group=group)
            for r, (l, h) in enumerate(bounds):
                if h > l and r != rank:
                    pp.m[0, l:h].copy_(recv[r * maxn:r * maxn + (h - l)])

        sweep(int(idx[0]), True, 1)
        for j in range(1, clusters):
            state = rng.bit_generator.state
            pp.select(j, float(rng.random()))
            got = int(pp.idx[0, j].item())
            if int(pp.halted[0].item()) == j:  # total == 0: rng.integers from here on
                rng.bit_generator.state = state
                for jj in range(j, clusters):
                    idx[jj] = rng.integers(total_points)
                break
            idx[j] = got
            if j + 1 < clusters:
                sweep(got, False, j + 1)
    return out


def init_centroids_sharded(x_shard: torch.Tensor, total_points: int, lo: int, clusters: int,
                           seed: int, method: str = "random_distinct", group=None,
                           backend=None) -> torch.Tensor:
    """Replicated initial centroids from a row-sharded dataset."""
    B, n_local, d = x_shard.shape
    if method == "kmeanspp":
        idx = kmeanspp_indices_sharded(x_shard, total_points, lo, clusters, seed, group, backend)
    elif method == "random_distinct":
        idx = init_indices(total_points, clusters, seed, B, method)
    else:
        raise ValueError(f"unknown init method {method!r}")
    buf = torch.zeros((B, clusters, d), dtype=torch.float64, device=x_shard.device)
    for b in range(B):
        sel = np.flatnonzero((idx[b] >= lo) & (idx[b] < lo + n_local))
        if sel.size:
            rows = torch.from_numpy(idx[b][sel] - lo).to(x_shard.device)
            buf[b, torch.from_numpy(sel).to(x_shard.device)] = x_shard[b].index_select(0, rows).double()
    dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    return buf


def reseed_farthest_sharded(eng: LloydEngine, lo: int, group=None) -> None:
    """reseed_farthest (pipeline.py:76-89) over row shards: each empty cluster, in
    id order, takes the next point by decreasing assigned distance, ties to the
    lowest GLOBAL index (pipeline._farthest: local top-E per rank, all-gathered
    in rank order); the rows come from their owners through one all-reduce.
    The empty mask is replicated (counts are all-reduced), so every rank
    reseeds alike."""
    nxt = eng.cur ^ 1
    em = eng.empty.cpu().numpy()
    if not em.any():
        return
    n_local, d, dev = eng.N, eng.d, eng.dev
    for b in range(eng.B):
        empties = np.flatnonzero(em[b])
        if empties.size == 0:
            continue
        gidx = torch.from_numpy(_farthest(eng.mind[b], int(empties.size), lo,
                                          group if group is not None else dist.group.WORLD)).to(dev)
        rows = torch.zeros((gidx.numel(), d), dtype=torch.float64, device=dev)
        mine = (gidx >= lo) & (gidx < lo + n_local)
        if bool(mine.any()):
            rows[mine] = eng.x[b, gidx[mine] - lo].double()
        dist.all_reduce(rows, op=dist.ReduceOp.SUM, group=group)
        cid = torch.from_numpy(empties[: gidx.numel()]).to(dev)
        eng.master[nxt][b, cid] = rows.to(eng.mdtype)
        if eng.operand is not eng.master:
            eng.operand[nxt][b, cid] = rows.to(eng.dtype)
    eng._refresh_bias(nxt)
    diff = eng.master[nxt].double() - eng.master[eng.cur].double()
    eng.shift2.copy_((diff * diff).sum(-1).max())


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
                                             cfg.init, group, backend))
    history = torch.empty((cfg.max_iters, eng.B), dtype=torch.float64, device=x_shard.device)
    # every rank takes the same decisions: the flags are reduced in the exchange
    if cfg.empty_cluster_policy != "reseed_farthest":
        iterations, slot, merges = eng.run(cfg.max_iters, cfg.shift_tol, history)
    else:  # stepwise: the reseed reads this iteration's min_dists before the commit
        iterations, slot = 0, 0
        for it in range(1, cfg.max_iters + 1):
            iterations = it
            slot = eng.iterate(history[it - 1])
            changed, shift = eng.poll()
            if it > 1 and not changed:
                break
            reseed_farthest_sharded(eng, lo, group)
            _, shift = eng.poll()
            eng.commit()
            if shift <= cfg.shift_tol:
                break
        merges = int(eng.merges.item())
    if x_shard.is_cuda:
        torch.cuda.synchronize(x_shard.device)
    # merges: LloydEngine.exchange re-evaluates the count on the all-reduced
    # counts, so it is already the single-process (global) figure on every rank
    counters.synchronized_merges += int(merges)
    return KMeansResult(Centroids(eng.centroids.clone(), check_finite=False),
                        Assignments(eng.ids[slot].clone(), validate=False),
                        history[:iterations].cpu().numpy(), iterations, counters)
