"""Run drivers: the in-core Lloyd loop and the chunked out-of-core variant.

Drop-in for reference pipeline.py:1-530 with the same termination semantics
(pipeline.py:110-147): stop when assignments repeat, when the largest
centroid shift falls to shift_tol, or at max_iters.  B200 design:

* ``LloydEngine`` keeps everything device-resident: X, two assignment
  buffers (ping-pong, so the repeat test is a device flag raised by the assign
  kernel), the f64/int64 statistics, a float32/float64 centroid master and the
  bf16/fp16 MMA operand, the objective history.  One iteration is four
  launches (assign, objective, update, normalize) and ONE 16-byte
  device->host read (changed flag + max shift) -- the only host sync.
* ``_streaming_pass`` streams pinned host chunks over a dedicated copy stream
  into two device buffers (event-gated ping-pong), overlapping H2D of chunk
  t+1 with assign+update of chunk t, accumulating statistics on the device
  and normalizing once per pass (pipeline.py:312-373).  Sources are either a
  host-resident array (``HostStream``, pinned once) or an FKM1 file
  (``ChunkStream``, pipeline.py:150-234): a reader thread ``readinto``s chunk
  t+2 into one of two pinned staging buffers while chunk t+1 is copied and
  chunk t computed.
"""

from __future__ import annotations

import math
import os
import threading
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np
import torch

from . import ops
from .baseline import argmin_rows, compute_distance_matrix, gather_assigned_distances, scatter_update
from .core import (INIT_METHODS, LOW_PRECISION, Assignments, Centroids, ClusterStats, Counters,
                   DataFormatError, DataMatrix, KMeansConfig, KMeansResult, device_of, init_indices,
                   master_dtype, to_device)
from .flash_assign import TilingConfig
from .tuner import CacheModel, ProblemShape, heuristic_config

__all__ = ["LloydEngine", "HostStream", "ChunkStream", "PartialStats", "DeviceAssignmentStore",
           "lloyd_run", "out_of_core_iteration", "chunked_stream_run", "stream_shard", "ENGINES"]

ENGINES = ("flash", "baseline")


def _resolve_tiling(cfg: KMeansConfig, points: int, dims: int, batch: int, elem: int,
                    workers: int) -> TilingConfig:
    if cfg.tiling is not None:
        return cfg.tiling
    shape = ProblemShape(points=points, clusters=cfg.clusters, dims=dims, batch=batch)
    return heuristic_config(shape, CacheModel(elem_bytes=elem, workers=workers))


def _workers(workers):
    from .core import worker_count

    return worker_count(workers)


class LloydEngine:
    """Device-resident Lloyd state for one (B, N, K, d) problem.

    ``x`` is a CUDA tensor (B, N, d).  ``update_chunk`` only defines the
    reference-compatible merge count.  ``allreduce`` (optional) is called
    once per iteration with a packed float64 device buffer
    [sums | counts | objective | changed] to combine point shards
    (distributed.py); it must sum in place.
    """

    def __init__(self, x: torch.Tensor, clusters: int, update_chunk: int | None = None,
                 allreduce=None, backend=None):
        # ``backend`` provides assign/objective/update/normalize with the
        # signatures of ``ops``; the product always uses ``ops`` (CUDA).  Tests
        # substitute a CPU checker to exercise the orchestration under gloo.
        self.be = ops if backend is None else backend
        if backend is None and not x.is_cuda:
            raise ValueError("LloydEngine needs the data on a CUDA device")
        self.x = x.contiguous()
        self.B, self.N, self.d = self.x.shape
        self.K = int(clusters)
        self.chunk = int(update_chunk or self.N)
        self.dev = self.x.device
        self.allreduce = allreduce
        B, N, K, d, dev = self.B, self.N, self.K, self.d, self.dev
        self.dtype = self.x.dtype
        self.mdtype = master_dtype(self.dtype)
        self.ids = [torch.empty((B, N), dtype=torch.int32, device=dev) for _ in range(2)]
        self.mind = torch.empty((B, N), dtype=torch.float32 if self.dtype in LOW_PRECISION
                                else self.dtype, device=dev)
        nred = B * K * d + B * K + B + 1
        self.red = torch.empty((nred,), dtype=torch.float64, device=dev)
        self.sums = self.red[: B * K * d].view(B, K, d)
        self.counts_f = self.red[B * K * d: B * K * d + B * K].view(B, K)
        self.obj_red = self.red[B * K * d + B * K: B * K * d + B * K + B]
        self.changed_f = self.red[-1:]
        self.counts = torch.empty((B, K), dtype=torch.int64, device=dev)
        self.master = [torch.empty((B, K, d), dtype=self.mdtype, device=dev) for _ in range(2)]
        if self.dtype in LOW_PRECISION:
            self.operand = [torch.empty((B, K, d), dtype=self.dtype, device=dev) for _ in range(2)]
        else:
            self.operand = self.master
        self.empty = torch.empty((B, K), dtype=torch.uint8, device=dev)
        # scalars: [changed(int32) | pad] and [shift2 (f64)] and merges (int64)
        self.changed = torch.zeros((), dtype=torch.int32, device=dev)
        self.shift2 = torch.zeros((), dtype=torch.float64, device=dev)
        self.merges = torch.zeros((), dtype=torch.int64, device=dev)      # committed updates
        self.merges_it = torch.zeros((), dtype=torch.int64, device=dev)   # this iteration
        self.obj = torch.empty((B,), dtype=torch.float64, device=dev)
        self.cur = 0
        self.it = 0
        # CUDA graphs of one iteration, keyed by (assignment slot, centroid slot);
        # only for the single-device CUDA path (the NCCL all-reduce stays eager)
        self.use_graphs = backend is None and allreduce is None and self.x.is_cuda
        self._graphs: dict = {}
        # single-device CUDA path: the end of an iteration is one fk_loop_tail
        # launch (objective, history row, flags, cleared accumulators), and the
        # tensor-core bias operand of the next centroids comes out of normalize
        self.fused = backend is None and allreduce is None
        self.bias = None
        # f32/f64 data: the split operand of X for the certified tensor-core
        # assign, built once (X never changes during a run)
        self.xsplit = ops.assign_xsplit(self.x) if backend is None and ops.split_auto(
            self.x, K) else None
        if self.fused:
            from .ops import OBJ_BLOCK

            # objective partials (f32 min_dists) or numpy's pairwise-tree workspace (f64)
            nb = max(int(ops.N.lib().fk_objective_workspace(B, N)), B * -(-N // OBJ_BLOCK) * 8)
            self._part = torch.empty((-(-nb // 8),), dtype=torch.float64, device=dev)
            self._flags_d = torch.zeros(3, dtype=torch.float64, device=dev)
            self._hist = None
            self._hist_row = torch.zeros((), dtype=torch.int64, device=dev)
            self._tail_ctr = torch.zeros((1,), dtype=torch.int32, device=dev)  # last-block counter
            # the update's histogram pass folded into the assign epilogue
            # (bf16/fp16, the pipelined run only; FK_HIST_FOLD=0 switches it off)
            self._fold = ops.hist_fold(self.x, K) if (
                self.xsplit is None and os.environ.get("FK_HIST_FOLD", "1") != "0") else None
            # ||x||^2 in the epilogue's own order, once per run (X is fixed):
            # the epilogue loads it instead of summing the tile row every row
            # tile -- worth its one pass over X where rows span few column
            # tiles (K <= 1024: config 2 -15 us, config 4 -6 us per iteration;
            # at config 3's 16 column tiles the gain is within noise)
            xn_env = os.environ.get("FK_ASSIGN_XNORM", "auto")
            self._xn = ops.assign_row_norms(self.x, K) if (
                self._fold is not None and xn_env != "0" and (K <= 1024 or xn_env == "1")) else None
            if self.dtype in LOW_PRECISION:
                kpad = ops.N.lib().fk_assign_bias_rows(K)
                self.bias = [torch.zeros((B, kpad, 16), dtype=torch.bfloat16, device=dev) for _ in range(2)]
                for bz in self.bias:  # padding columns: +inf bias (normalize writes rows < K only)
                    bz[:, K:, 0] = float("inf")

    # -------------------------------------------------------------- state
    def set_centroids(self, c: torch.Tensor) -> None:
        c = to_device(c, self.dev)
        self.master[self.cur].copy_(c.to(self.mdtype))
        if self.operand is not self.master:
            self.operand[self.cur].copy_(self.master[self.cur].to(self.dtype))
        self._refresh_bias(self.cur)
        self.it = 0

    def _refresh_bias(self, slot: int) -> None:
        """Recompute the bias operand of operand[slot] (after a host-side edit)."""
        if self.bias is not None:
            ops.assign_bias(self.operand[slot], out=self.bias[slot])

    def _assign_kw(self, csrc: int) -> dict:
        if self.xsplit is not None:
            return {"xsplit": self.xsplit}
        return {} if self.bias is None else {"bias": self.bias[csrc]}

    def _normalize(self, nxt: int) -> None:
        kw = {} if self.bias is None else {"bias_out": self.bias[nxt]}
        self.be.normalize(self.sums, self.counts, self.master[self.cur], out=self.master[nxt],
                          operand_out=None if self.operand is self.master else self.operand[nxt],
                          empty=self.empty, shift2=self.shift2, **kw)

    @property
    def centroids(self) -> torch.Tensor:
        return self.master[self.cur]

    @property
    def operand_centroids(self) -> torch.Tensor:
        return self.operand[self.cur]

    # -------------------------------------------------------------- phases
    def assign(self, out_slot: int, compare: bool):
        self.be.assign(self.x, self.operand[self.cur], idx_prev=self.ids[out_slot ^ 1] if compare else None,
                       changed=self.changed if compare else None, idx_out=self.ids[out_slot],
                       mind_out=self.mind, **self._assign_kw(self.cur))

    def iterate(self, history_row: torch.Tensor | None = None):
        """One Lloyd iteration, fully on the device.

        Writes: ids[slot] (this iteration's assignment), objective, the next
        master/operand into the other centroid slot, the changed flag and
        max squared shift.  Returns the assignment slot used.  From the second
        iteration on, the launch sequence is replayed from a CUDA graph (two
        graphs alternate with the ping-pong buffers)."""
        slot = self.it & 1
        if self.use_graphs and self.it > 0:
            key = (slot, self.cur)
            gr = self._graphs.get(key)
            if gr is None:
                gr = torch.cuda.CUDAGraph()
                with torch.cuda.graph(gr):
                    self._body(slot, True)
                self._graphs[key] = gr
            gr.replay()
            if history_row is not None:
                history_row.copy_(self.obj)
            self.it += 1
            return slot
        self._body(slot, self.it > 0)
        if history_row is not None:
            history_row.copy_(self.obj)
        self.it += 1
        return slot

    def _body(self, slot: int, compare: bool) -> None:
        """The device work of one iteration (eager or under graph capture)."""
        self.changed.zero_()
        self.shift2.zero_()
        self.merges_it.zero_()
        self.assign(slot, compare)
        self.be.objective(self.mind, out=self.obj)
        self.be.update(self.x, self.ids[slot], self.K, self.chunk, sums=self.sums, counts=self.counts,
                   merges=self.merges_it)
        if self.allreduce is not None:
            self.exchange()
        self._normalize(self.cur ^ 1)

    def exchange(self) -> None:
        """Combine the point shards: pack [counts | objective | changed] behind the
        sums, one in-place all-reduce of the f64 buffer, unpack (distributed.py)."""
        tail = self.red[self.B * self.K * self.d:]
        if hasattr(self.be, "stats_pack"):
            self.be.stats_pack(self.counts, self.obj, self.changed, tail)
        else:
            self.counts_f.copy_(self.counts)
            self.obj_red.copy_(self.obj)
            self.changed_f.copy_(self.changed)
        self.allreduce(self.red)
        if hasattr(self.be, "stats_pack"):
            self.be.stats_pack(self.counts, self.obj, self.changed, tail, unpack=True)
        else:
            self.counts.copy_(self.counts_f)
            self.obj.copy_(self.obj_red)
            self.changed.copy_((self.changed_f[0] > 0).to(torch.int32))
        # the reference's merge count is a function of the GLOBAL sorted order:
        # re-evaluate it on the reduced counts (each shard counted its own runs)
        self.be.merges_from_counts(self.counts, self.chunk, self.merges_it)

    # ------------------------------------------------- pipelined iteration
    # Split of one iteration into (assign) and (rest) so that the NEXT
    # iteration's assign can be queued before the host reads this one's
    # decision flags: the GPU never idles on the host's poll.  Speculation is
    # safe: the speculative assign reads the new centroid slot and writes only
    # the other assignment slot, `mind` and `changed` (zeroed after this
    # iteration's flags were copied out in stream order); if the run stops,
    # its results are simply not used.
    def _graph(self, key, fn):
        if not self.use_graphs:
            fn()
            return
        gr = self._graphs.get(key)
        if gr is None:
            fn()  # eager once (first launches set kernel attributes, outside capture)
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr):
                fn()
            self._graphs[key] = gr
            return
        gr.replay()

    def enq_assign(self, slot: int, compare: bool, csrc: int) -> None:
        """Queue iteration work part 1: assignment into ids[slot] against operand[csrc]."""
        def fn():
            if not self.fused:  # the fused tail leaves `changed` cleared
                self.changed.zero_()
            kw = self._assign_kw(csrc)
            if self.fused and self._fold is not None:
                kw["hist"] = self._fold
                if self._xn is not None:
                    kw["xnorm"] = self._xn
            self.be.assign(self.x, self.operand[csrc],
                           idx_prev=self.ids[slot ^ 1] if compare else None,
                           changed=self.changed if compare else None, idx_out=self.ids[slot],
                           mind_out=self.mind, **kw)
        self._graph(("a", slot, compare, csrc), fn)

    def enq_rest(self, slot: int, history_row: torch.Tensor | None = None, timers=None) -> None:
        """Queue part 2: objective, update, shard exchange, normalize into the
        other centroid slot, then an async copy of [changed, shift2, merges]
        to pinned host memory (read by wait_flags).  On the single-device path
        the objective, the history row (``run``'s history, row index kept on
        the device), the flags and the cleared accumulators are one
        fk_loop_tail launch."""
        if not hasattr(self, "_flags_h"):
            if not self.fused:
                self._flags_d = torch.zeros(3, dtype=torch.float64, device=self.dev)
            self._flags_h = torch.zeros(3, dtype=torch.float64).pin_memory() if self.x.is_cuda \
                else torch.zeros(3, dtype=torch.float64)
            self._flags_ev = torch.cuda.Event() if self.x.is_cuda else None
        nxt = self.cur ^ 1

        def fn_fused():
            # objective partials, normalize and the loop tail are one launch
            # (fk_normalize_loop_tail) after the update
            if timers is not None:  # bench: live per-kernel timing (eager only)
                timers[0].record()
            self.be.update(self.x, self.ids[slot], self.K, self.chunk, sums=self.sums,
                           counts=self.counts, merges=self.merges_it,
                           **({} if self._fold is None else {"hist": self._fold}))
            if timers is not None:
                timers[1].record()
            ops.normalize_loop_tail(
                self.sums, self.counts, self.master[self.cur], self.master[nxt],
                None if self.operand is self.master else self.operand[nxt], self.empty, self.shift2,
                None if self.bias is None else self.bias[nxt], self.mind, self._part, self.obj, self.changed,
                self.merges_it, self._flags_d, self._tail_ctr, self._hist,
                None if self._hist is None else self._hist_row)

        def fn():
            self.shift2.zero_()
            self.merges_it.zero_()
            self.be.objective(self.mind, out=self.obj)
            if timers is not None:
                timers[0].record()
            self.be.update(self.x, self.ids[slot], self.K, self.chunk, sums=self.sums,
                           counts=self.counts, merges=self.merges_it)
            if timers is not None:
                timers[1].record()
            if self.allreduce is not None:
                self.exchange()
            self._normalize(nxt)
            self._flags_d[0].copy_(self.changed)
            self._flags_d[1].copy_(self.shift2)
            self._flags_d[2].copy_(self.merges_it)
        body = fn_fused if self.fused else fn
        if timers is not None:
            body()
        else:
            hp = None if self._hist_ptr() is None else self._hist_ptr()
            self._graph(("r", slot, self.cur, hp), body)
        if history_row is not None:
            history_row.copy_(self.obj)
        self._flags_h.copy_(self._flags_d, non_blocking=True)
        if self._flags_ev is not None:
            self._flags_ev.record()

    def _hist_ptr(self):
        return None if not self.fused or self._hist is None else self._hist.data_ptr()

    def wait_flags(self):
        """(changed, shift, merges of this iteration) once its flags reached the host."""
        if self._flags_ev is not None:
            self._flags_ev.synchronize()
        f = self._flags_h.tolist()
        return f[0] != 0, math.sqrt(f[1]), int(f[2])

    def run(self, max_iters: int, shift_tol: float, history: torch.Tensor | None = None,
            stop_on_repeat: bool = True):
        """lloyd_run's loop (pipeline.py:128-147, policy "keep") with the next
        assign queued speculatively before each poll.  Returns (iterations,
        assignment slot of the last iteration, committed merge count)."""
        merges = 0
        slot = 0
        it = 0
        if self.fused:  # the loop tail writes history rows through a device row index
            if self._fold is not None:  # a speculative assign of an earlier run may have added
                self._fold.clear()
            self._hist = history
            self._hist_row.zero_()
            self.changed.zero_()
            self.shift2.zero_()
            self.merges_it.zero_()
        self.enq_assign(0, False, self.cur)
        while it < max_iters:
            it += 1
            slot = (it - 1) & 1
            self.enq_rest(slot, None if (history is None or self.fused) else history[it - 1])
            spec = it < max_iters
            if spec:  # assume the commit: next assign against the new centroids
                self.enq_assign(slot ^ 1, True, self.cur ^ 1)
            changed, shift, mg = self.wait_flags()
            if stop_on_repeat and it > 1 and not changed:
                break  # assignments repeated: the update reproduces c bitwise
            self.cur ^= 1
            merges += mg
            if shift <= shift_tol:
                break
        self.it = it
        if self.fused:
            self._hist = None
        return it, slot, merges

    def poll(self):
        """(changed: bool, shift: float) -- the one device->host read per iteration."""
        v = torch.stack([self.changed.to(torch.float64), self.shift2]).cpu()
        return bool(v[0] != 0), math.sqrt(float(v[1]))

    def commit(self) -> None:
        """Adopt the normalized centroids (the swap `c = new_c`); the update ran for real."""
        self.cur ^= 1
        self.merges += self.merges_it

    def reseed_farthest(self, slot: int) -> None:
        """reseed_farthest policy (pipeline.py:76-89): each empty cluster takes the
        next-farthest point (distance desc, index asc), in id order."""
        nxt = self.cur ^ 1
        em = self.empty.cpu().numpy()
        for b in range(self.B):
            empties = np.flatnonzero(em[b])
            if empties.size == 0:
                continue
            rows = torch.from_numpy(_farthest(self.mind[b], int(empties.size), 0)).to(self.dev)
            cid = torch.from_numpy(empties[: rows.numel()]).to(self.dev)
            self.master[nxt][b, cid] = self.x[b, rows].to(self.mdtype)
            if self.operand is not self.master:
                self.operand[nxt][b, cid] = self.x[b, rows]
        self._refresh_bias(nxt)
        diff = self.master[nxt].double() - self.master[self.cur].double()
        self.shift2.copy_((diff * diff).sum(-1).max())


def lloyd_run(x: DataMatrix, cfg: KMeansConfig, engine: str = "flash", workers: int | None = None,
              counters: Counters | None = None) -> KMeansResult:
    """Full in-core run (pipeline.py:110-147); device-resident, one host sync per iteration.

    objective_history[i, b] is the float64 sum of assigned squared distances
    observed by iteration i's assignment step."""
    if engine not in ENGINES:
        raise ValueError(f"engine must be one of {ENGINES}")
    counters = counters if counters is not None else Counters()
    n_workers = _workers(workers)
    tiling = _resolve_tiling(cfg, x.points, x.dims, x.batch, x.elem_bytes, n_workers)
    dev = device_of(x.data)
    xd = to_device(x.data, dev)
    if engine == "baseline":
        return _lloyd_baseline(DataMatrix(xd, check_finite=False), cfg, counters)
    idx = init_indices(x.points, cfg.clusters, cfg.seed, x.batch, cfg.init, xd)
    it_ = torch.from_numpy(idx).to(dev)
    c0 = torch.stack([xd[b].index_select(0, it_[b]) for b in range(x.batch)])
    eng = LloydEngine(xd, cfg.clusters, tiling.update_chunk)
    eng.set_centroids(c0)
    history = torch.empty((cfg.max_iters, x.batch), dtype=torch.float64, device=dev)
    if cfg.empty_cluster_policy != "reseed_farthest":
        iterations, slot, merges = eng.run(cfg.max_iters, cfg.shift_tol, history)
        torch.cuda.synchronize(dev)  # a speculative assign may still be in flight
        counters.synchronized_merges += merges
        return KMeansResult(Centroids(eng.centroids.clone(), check_finite=False),
                            Assignments(eng.ids[slot].clone(), validate=False),
                            history[:iterations].cpu().numpy(), iterations, counters)
    iterations = 0
    slot = 0
    for it in range(1, cfg.max_iters + 1):
        iterations = it
        slot = eng.iterate(history[it - 1])
        changed, shift = eng.poll()
        if it > 1 and not changed:
            break  # assignments repeated: the update reproduces c bitwise
        eng.reseed_farthest(slot)
        _, shift = eng.poll()
        eng.commit()
        if shift <= cfg.shift_tol:
            break
    counters.synchronized_merges += int(eng.merges.item())
    return KMeansResult(Centroids(eng.centroids.clone(), check_finite=False),
                        Assignments(eng.ids[slot].clone(), validate=False),
                        history[:iterations].cpu().numpy(), iterations, counters)


def _lloyd_baseline(x: DataMatrix, cfg: KMeansConfig, counters: Counters) -> KMeansResult:
    """engine="baseline": the materializing foil (baseline.py), same decisions."""
    from .baseline import normalize
    from .core import init_centroids

    c = init_centroids(x, cfg.clusters, cfg.seed, cfg.init)
    if c.data.dtype in LOW_PRECISION:
        c = Centroids(c.data.float(), check_finite=False)
    history, prev, a = [], None, None
    iterations = 0
    for it in range(1, cfg.max_iters + 1):
        iterations = it
        xc = x if c.data.dtype == x.data.dtype else DataMatrix(x.data.float(), check_finite=False)
        d = compute_distance_matrix(xc, c, counters)
        a = argmin_rows(d)
        mind = gather_assigned_distances(d, a)
        history.append(mind.double().sum(dim=1).cpu().numpy())
        if prev is not None and torch.equal(prev.values, a.values):
            break
        stats = scatter_update(xc, a, cfg.clusters, counters)
        new_c, empties = normalize(stats, c, cfg.empty_cluster_policy)
        if cfg.empty_cluster_policy == "reseed_farthest" and any(empties):
            # _reseed_in_core (pipeline.py:84-89): next-farthest point per empty cluster
            data = new_c.data.clone()
            for b, cids in enumerate(empties):
                if cids:
                    rows = torch.from_numpy(_farthest(mind[b], len(cids), 0)).to(data.device)
                    data[b, torch.tensor(cids[: rows.numel()], device=data.device)] = xc.data[b, rows].to(data.dtype)
            new_c = Centroids(data, check_finite=False)
        diff = new_c.data.double() - c.data.double()
        shift = float((diff * diff).sum(-1).max().sqrt())
        prev, c = a, new_c
        if shift <= cfg.shift_tol:
            break
    return KMeansResult(c, a, np.array(history), iterations, counters)


# ============================================================== streaming
class HostStream:
    """Chunk-granular source over a host-resident (B, N, d) array.

    Stands in for the reference's file-backed ChunkStream (pipeline.py:150-234)
    with the same surface (batch, total_points, dims, precision, chunk_points,
    n_chunks, bounds, read_rows).  The array is pinned once so every chunk is a
    true async DMA (cudaMemcpyAsync from page-locked memory).

    A rank of a sharded run may hold only its own rows: ``row_offset`` and
    ``total_points`` place ``data`` (B, n_local, d) at rows [row_offset,
    row_offset + n_local) of a ``total_points``-row dataset.  Chunk indices and
    bounds stay global (the chunk grid of the whole dataset); ``stream_shard``
    gives the rows a rank streams."""

    def __init__(self, data, chunk_points: int, pin: bool = True, row_offset: int = 0,
                 total_points: int | None = None):
        if int(chunk_points) < 1:
            raise ValueError("chunk_points must be >= 1")
        t = data.data if isinstance(data, DataMatrix) else (
            torch.from_numpy(np.ascontiguousarray(data)) if isinstance(data, np.ndarray) else data)
        if t.dim() != 3:
            raise DataFormatError("stream payload must be (batch, points, dims)")
        if t.is_cuda:
            raise ValueError("HostStream wraps host memory; use lloyd_run for device data")
        self.host = t.contiguous()
        if pin and not self.host.is_pinned():
            self.host = self.host.pin_memory()
        self.batch, n_local, self.dims = self.host.shape
        self.row_offset = int(row_offset)
        self.total_points = int(total_points) if total_points is not None else self.row_offset + n_local
        if self.row_offset < 0 or self.row_offset + n_local > self.total_points:
            raise ValueError("row_offset/total_points do not contain the local rows")
        self.row_end = self.row_offset + n_local
        self.chunk_points = min(int(chunk_points), self.total_points)
        self.path = None

    @property
    def dtype(self) -> torch.dtype:
        return self.host.dtype

    @property
    def precision(self) -> str:
        from .core import precision_for

        return precision_for(self.host.dtype)

    @property
    def elem_bytes(self) -> int:
        return self.host.element_size()

    @property
    def n_chunks(self) -> int:
        return -(-self.total_points // self.chunk_points)

    def bounds(self, t: int) -> tuple[int, int]:
        if not 0 <= t < self.n_chunks:
            raise ValueError(f"chunk index {t} out of range")
        lo = t * self.chunk_points
        return lo, min(self.total_points, lo + self.chunk_points)

    def has_rows(self, lo: int, hi: int) -> bool:
        return self.row_offset <= lo and hi <= self.row_end

    def view(self, b: int, lo: int, hi: int) -> torch.Tensor:
        if not 0 <= b < self.batch or not 0 <= lo < hi <= self.total_points:
            raise ValueError("row range outside the stream bounds")
        if not self.has_rows(lo, hi):
            raise ValueError(f"rows [{lo}, {hi}) are not held by this shard "
                             f"[{self.row_offset}, {self.row_end})")
        return self.host[b, lo - self.row_offset:hi - self.row_offset]

    def read_rows(self, b: int, lo: int, hi: int) -> torch.Tensor:
        return self.view(b, lo, hi).clone()

    def close(self) -> None:
        pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


def stream_shard(stream, world: int, rank: int) -> tuple[int, int, int, int]:
    """(chunk_lo, chunk_hi, row_lo, row_hi) a rank streams in a sharded pass:
    whole chunks of the global chunk grid, rank r taking chunks
    [r*T//P, (r+1)*T//P).  Every chunk is then processed exactly as in the
    single-process pass (same rows, same per-chunk update), so the pass
    statistics and merge count summed over ranks equal the single-process
    ones."""
    T = stream.n_chunks
    c_lo, c_hi = T * rank // world, T * (rank + 1) // world
    if c_hi <= c_lo:
        return c_lo, c_hi, 0, 0
    return c_lo, c_hi, stream.bounds(c_lo)[0], stream.bounds(c_hi - 1)[1]


class ChunkStream:
    """Chunk-granular reader over an FKM1 file that never loads it whole
    (pipeline.py:150-234): rows land directly in caller buffers (``readinto``;
    pinned staging buffers in the streaming pass), one read at a time under a
    lock.  Same surface as the reference: batch, total_points, dims,
    precision, elem_bytes, chunk_points, n_chunks, bounds, read_rows_into,
    read_rows, close."""

    def __init__(self, path: str, chunk_points: int):
        from .fileio import read_fkm1_header

        if int(chunk_points) < 1:
            raise ValueError("chunk_points must be >= 1")
        h = read_fkm1_header(path)
        self.path = path
        self.batch, self.total_points, self.dims = h.batch, h.points, h.dims
        self.precision = h.precision
        self.elem_bytes = h.elem_bytes
        self._dtype = h.dtype
        self.chunk_points = min(int(chunk_points), h.points)
        self._row_bytes = self.dims * self.elem_bytes
        self._f = None
        self._lock = threading.Lock()

    @property
    def dtype(self) -> torch.dtype:
        return self._dtype

    @property
    def n_chunks(self) -> int:
        return -(-self.total_points // self.chunk_points)

    def bounds(self, t: int) -> tuple[int, int]:
        if not 0 <= t < self.n_chunks:
            raise ValueError(f"chunk index {t} out of range")
        lo = t * self.chunk_points
        return lo, min(self.total_points, lo + self.chunk_points)

    def has_rows(self, lo: int, hi: int) -> bool:
        return True

    def _handle(self):
        if self._f is None:
            self._f = open(self.path, "rb", buffering=0)
        return self._f

    def read_rows_into(self, b: int, lo: int, hi: int, out):
        """Rows [lo, hi) of batch element b into ``out`` (a host tensor or numpy
        array of shape (>= rows, dims) and the stream's dtype); returns the view."""
        from .fileio import host_bytes_view

        rows = hi - lo
        if not 0 <= b < self.batch or not 0 <= lo < hi <= self.total_points:
            raise ValueError("row range outside the stream bounds")
        t = torch.from_numpy(out) if isinstance(out, np.ndarray) else out
        if t.dim() != 2 or t.shape[0] < rows or t.shape[1] != self.dims:
            raise ValueError("destination buffer is too small for the requested rows")
        if t.dtype != self._dtype or not t.is_contiguous() or t.is_cuda:
            raise ValueError("destination buffer must be host memory of the stream dtype, row-major")
        view = t[:rows]
        mv = host_bytes_view(view)
        nbytes = rows * self._row_bytes
        from .fileio import FKM1_HEADER_BYTES

        with self._lock:
            f = self._handle()
            f.seek(FKM1_HEADER_BYTES + (b * self.total_points + lo) * self._row_bytes)
            got = 0
            while got < nbytes:  # raw readinto may return partial counts
                n = f.readinto(mv[got:])
                if not n:
                    break
                got += n
        if got != nbytes:
            raise DataFormatError(f"short read: wanted {nbytes} bytes, got {got}")
        return out[:rows] if isinstance(out, np.ndarray) else view

    def read_rows(self, b: int, lo: int, hi: int) -> torch.Tensor:
        return self.read_rows_into(b, lo, hi, torch.empty((hi - lo, self.dims), dtype=self._dtype))

    def close(self) -> None:
        if self._f is not None:
            self._f.close()
            self._f = None

    def __enter__(self) -> "ChunkStream":
        return self

    def __exit__(self, *exc) -> None:
        self.close()


@dataclass
class PartialStats:
    """One chunk's cluster sums/counts; combined in ascending chunk order (pipeline.py:237-258)."""

    chunk_index: int
    sums: torch.Tensor
    counts: torch.Tensor

    def __post_init__(self):
        if self.sums.dim() != 2 or self.sums.dtype != torch.float64:
            raise ValueError("PartialStats.sums must be (clusters, dims) float64")
        if tuple(self.counts.shape) != tuple(self.sums.shape[:1]) or self.counts.dtype != torch.int64:
            raise ValueError("PartialStats.counts must be (clusters,) int64")

    def combine(self, other: "PartialStats") -> "PartialStats":
        if self.sums.shape != other.sums.shape:
            raise ValueError("cannot combine partials of different shapes")
        return PartialStats(min(self.chunk_index, other.chunk_index), self.sums + other.sums,
                            self.counts + other.counts)


class DeviceAssignmentStore:
    """Device-resident stand-in for the reference's FKA1 AssignmentStore
    (fileio.py:189-247): holds this pass's and the previous pass's ids and
    raises a device changed flag; starts from the 0xFFFFFFFF sentinel.  A
    sharded pass keeps only its rows [row_offset, row_offset + points)."""

    def __init__(self, batch: int, points: int, device, row_offset: int = 0):
        self.batch, self.points, self.row_offset = batch, points, int(row_offset)
        self.ids = [torch.full((batch, points), -1, dtype=torch.int32, device=device) for _ in range(2)]
        self.cur = 0
        self.changed = torch.zeros((), dtype=torch.int32, device=device)

    def begin_pass(self):
        self.cur ^= 1
        self.changed.zero_()

    @property
    def new(self) -> torch.Tensor:
        return self.ids[self.cur]

    @property
    def old(self) -> torch.Tensor:
        return self.ids[self.cur ^ 1]

    def read_all(self) -> Assignments:
        return Assignments(self.new.clone(), validate=False)

    def finalize(self) -> None:
        pass

    def abort(self) -> None:
        pass


class _StreamState:
    """Device buffers and streams for the chunk pipeline of one stream shape."""

    def __init__(self, stream, clusters: int, device, rows_local: int, keep_mind: bool = False):
        self.dev = device
        cp, d, B = stream.chunk_points, stream.dims, stream.batch
        self.buf = [torch.empty((1, cp, d), dtype=stream.dtype, device=device) for _ in range(2)]
        # file-backed sources: two pinned staging buffers filled by a reader thread
        self.staged = not isinstance(stream, HostStream)
        if self.staged:
            self.stage = [torch.empty((cp, d), dtype=stream.dtype, pin_memory=True) for _ in range(2)]
            self.copied = [torch.cuda.Event() for _ in range(2)]
            self.reader = ThreadPoolExecutor(max_workers=1)
        mdt = torch.float32 if stream.dtype in LOW_PRECISION else stream.dtype
        # reseed_farthest needs every (local) point's assigned distance of the pass
        self.mind_all = torch.empty((B, rows_local), dtype=mdt, device=device) if keep_mind else None
        self.mind = torch.empty((1, cp), dtype=mdt, device=device)
        self.copy_stream = torch.cuda.Stream(device=device)
        self.ready = [torch.cuda.Event() for _ in range(2)]
        self.free = [torch.cuda.Event() for _ in range(2)]
        BK = B * clusters
        # one packed f64 buffer [sums | counts | objective | changed | merges]: a
        # sharded pass combines its ranks with ONE all-reduce of it
        self.red = torch.zeros((BK * d + BK + B + 2,), dtype=torch.float64, device=device)
        self.sums = self.red[:BK * d].view(B, clusters, d)
        self.red_tail = self.red[BK * d:-1]
        self.counts = torch.zeros((B, clusters), dtype=torch.int64, device=device)
        self.obj = torch.zeros((B,), dtype=torch.float64, device=device)
        # per-chunk objectives, folded on the host in chunk order after the pass
        # (pipeline.py:354: obj[b] += float(np.sum(m)) chunk by chunk), so a
        # sharded pass adds them in the single-process order
        self.obj_chunks = torch.zeros((B, stream.n_chunks), dtype=torch.float64, device=device)
        self.obj_host = np.zeros((B,), np.float64)
        self.merges = torch.zeros((), dtype=torch.int64, device=device)       # all passes
        self.merges_pass = torch.zeros((), dtype=torch.int64, device=device)  # this pass


def _group_info(group):
    if group is None:
        return 1, 0
    import torch.distributed as dist

    return dist.get_world_size(group), dist.get_rank(group)


def _rows_to_device(stream, b: int, idx, device, group=None, row_lo: int = 0,
                    row_hi: int | None = None) -> torch.Tensor:
    """Rows ``idx`` (global indices) of batch element b as a (len, d) device
    tensor in the stream dtype.  In a sharded run each row comes from the rank
    whose shard holds it, through one f64 all-reduce (exact for every dtype)."""
    idx = [int(i) for i in idx]
    if group is None:
        rows = torch.stack([stream.read_rows(b, i, i + 1)[0] for i in idx]) if idx else \
            torch.empty((0, stream.dims), dtype=stream.dtype)
        return rows.to(device)
    import torch.distributed as dist

    hi = stream.total_points if row_hi is None else row_hi
    buf = torch.zeros((len(idx), stream.dims), dtype=torch.float64)
    for j, i in enumerate(idx):
        if row_lo <= i < hi:
            buf[j] = stream.read_rows(b, i, i + 1)[0].double()
    buf = buf.to(device)
    dist.all_reduce(buf, op=dist.ReduceOp.SUM, group=group)
    return buf.to(stream.dtype)


def _farthest(mind: torch.Tensor, take: int, offset: int, group=None):
    """The ``take`` points farthest from their centroid, ordered by distance
    descending then GLOBAL index ascending (reference _farthest_order,
    pipeline.py:76-81).  ``mind`` holds rows [offset, offset + len).  Sharded:
    each rank proposes its local top-``take``, the candidates are all-gathered
    in rank order (= global index order, so a stable sort keeps the lowest
    index first on ties) and every rank picks the same winners."""
    dev = mind.device
    md = mind.double()
    n = md.numel()
    k = min(take, n)
    if mind.is_cuda and k <= ops.FARTHEST_EMAX:
        order = ops.farthest(mind.reshape(1, n), k)[0]  # device radix select (fk_farthest)
    else:  # host tensors (the CPU test backend) or more than 8192 empties: a stable sort
        order = torch.sort(-md, stable=True).indices[:k]
    cand_d = torch.full((take,), float("-inf"), dtype=torch.float64, device=dev)
    cand_i = torch.full((take,), -1, dtype=torch.int64, device=dev)
    cand_d[:k] = md[order]
    cand_i[:k] = order + offset
    if group is None:
        return cand_i[:k].cpu().numpy()
    import torch.distributed as dist

    world = dist.get_world_size(group)
    all_d = torch.empty((world * take,), dtype=torch.float64, device=dev)
    all_i = torch.empty((world * take,), dtype=torch.int64, device=dev)
    dist.all_gather(list(all_d.view(world, take).unbind(0)), cand_d, group=group)
    dist.all_gather(list(all_i.view(world, take).unbind(0)), cand_i, group=group)
    win = torch.sort(-all_d, stable=True).indices[:take]
    got = all_i[win].cpu().numpy()
    return got[got >= 0]


class _StreamRunner:
    """One streamed Lloyd pass at a time over ``stream`` (pipeline.py:312-373).

    With ``group`` (torch.distributed), rank r streams whole chunks
    [r*T//P, (r+1)*T//P) of the global chunk grid (``stream_shard``), keeps
    the ids of its rows device-resident, and the pass statistics, objective,
    changed flag and merge count are summed across ranks with one packed f64
    all-reduce before the replicated normalize."""

    def __init__(self, stream, clusters: int, device, chunk: int, group=None,
                 policy: str = "keep"):
        self.group = group
        self.world, self.rank = _group_info(group)
        self.c_lo, self.c_hi, self.row_lo, self.row_hi = stream_shard(stream, self.world, self.rank)
        self.stream = stream
        self.policy = policy
        self.K = clusters
        self.chunk = chunk
        self.dev = device
        rows_local = self.row_hi - self.row_lo
        self.st = _StreamState(stream, clusters, device, rows_local,
                               keep_mind=policy == "reseed_farthest")
        B, K, d = stream.batch, clusters, stream.dims
        self.mdt = master_dtype(stream.dtype)
        self.master = [torch.empty((B, K, d), dtype=self.mdt, device=device) for _ in range(2)]
        self.lowp = stream.dtype in LOW_PRECISION
        self.operand = ([torch.empty((B, K, d), dtype=stream.dtype, device=device) for _ in range(2)]
                        if self.lowp else self.master)
        self.shift2 = torch.zeros((), dtype=torch.float64, device=device)
        self.empty = torch.empty((B, K), dtype=torch.uint8, device=device)
        self.store = DeviceAssignmentStore(B, rows_local, device, row_offset=self.row_lo)
        self.cur = 0

    def set(self, c: torch.Tensor):
        self.master[self.cur].copy_(to_device(c, self.dev).to(self.mdt))
        if self.lowp:
            self.operand[self.cur].copy_(self.master[self.cur].to(self.stream.dtype))

    def one_pass(self, counters: Counters):
        """Per-chunk assign + update with the H2D of chunk i+1 overlapping the
        compute of chunk i, then (sharded: one all-reduce) normalize into the
        other centroid slot.  Returns (changed, shift)."""
        st, stream, store = self.st, self.stream, self.store
        nxt = self.cur ^ 1
        master, operand = self.master[self.cur], self.operand[self.cur]
        st.sums.zero_()
        st.counts.zero_()
        st.obj.zero_()
        st.obj_chunks.zero_()
        st.merges_pass.zero_()
        self.shift2.zero_()
        store.begin_pass()
        compute = torch.cuda.current_stream(st.dev)
        tasks = [(b, t) for b in range(stream.batch) for t in range(self.c_lo, self.c_hi)]
        reads = {}
        r0 = self.row_lo

        def submit_read(i):  # reader thread: wait until staging buffer i&1 was copied out
            b, t = tasks[i]
            lo, hi = stream.bounds(t)
            k = i & 1
            ev = st.copied[k] if i >= 2 else None

            def job():
                if ev is not None:
                    ev.synchronize()
                stream.read_rows_into(b, lo, hi, st.stage[k])

            reads[i] = st.reader.submit(job)

        def issue_copy(i):
            b, t = tasks[i]
            lo, hi = stream.bounds(t)
            k = i & 1
            if st.staged:
                reads.pop(i).result()
                src = st.stage[k][: hi - lo]
            else:
                src = stream.view(b, lo, hi)
            with torch.cuda.stream(st.copy_stream):
                st.copy_stream.wait_event(st.free[k])
                st.buf[k][0, : hi - lo].copy_(src, non_blocking=True)
                st.ready[k].record(st.copy_stream)
                if st.staged:
                    st.copied[k].record(st.copy_stream)
            if st.staged and i + 2 < len(tasks):
                submit_read(i + 2)

        for k in range(2):  # both buffers start free
            st.free[k].record(compute)
        if st.staged:
            for i in range(min(2, len(tasks))):
                submit_read(i)
        if tasks:
            issue_copy(0)
        streamed = 0
        for i, (b, t) in enumerate(tasks):
            lo, hi = stream.bounds(t)
            rows = hi - lo
            k = i & 1
            compute.wait_event(st.ready[k])
            xb = st.buf[k][:, :rows]
            ids_new = store.new[b: b + 1, lo - r0:hi - r0]   # contiguous: one row segment of (B, n)
            ids_old = store.old[b: b + 1, lo - r0:hi - r0]
            mind = st.mind[:, :rows] if st.mind_all is None else st.mind_all[b: b + 1, lo - r0:hi - r0]
            ops.assign(xb, operand[b: b + 1], idx_prev=ids_old, changed=store.changed,
                       idx_out=ids_new, mind_out=mind)
            ops.objective(mind, out=st.obj_chunks[b, t:t + 1])
            ops.update(xb, ids_new, self.K, self.chunk, accumulate=True, sums=st.sums[b: b + 1],
                       counts=st.counts[b: b + 1], merges=st.merges_pass)
            st.free[k].record(compute)
            streamed += rows
            if i + 1 < len(tasks):  # host may block on the file read while chunk i computes
                issue_copy(i + 1)
        if self.group is not None:
            import torch.distributed as dist

            ops.stats_pack(st.counts, st.obj, store.changed, st.red_tail)
            st.red[-1:].copy_(st.merges_pass)
            dist.all_reduce(st.red, op=dist.ReduceOp.SUM, group=self.group)
            ops.stats_pack(st.counts, st.obj, store.changed, st.red_tail, unpack=True)
            st.merges_pass.copy_(st.red[-1])
            # each chunk's objective has exactly one contributor: the sum is a gather
            dist.all_reduce(st.obj_chunks, op=dist.ReduceOp.SUM, group=self.group)
            streamed = stream.batch * stream.total_points  # every rank reports the whole pass
        counters.elements_streamed += streamed
        st.merges += st.merges_pass
        ops.normalize(st.sums, st.counts, master, out=self.master[nxt],
                      operand_out=self.operand[nxt] if self.lowp else None, empty=self.empty,
                      shift2=self.shift2)
        if st.mind_all is not None:
            self._reseed(master, self.master[nxt], self.operand[nxt] if self.lowp else None)
        v = torch.stack([store.changed.to(torch.float64), self.shift2]).cpu()
        chunk_obj = st.obj_chunks.cpu().numpy()
        for b in range(stream.batch):  # chunk order, one rounding per chunk (as the reference)
            acc = 0.0
            for val in chunk_obj[b]:
                acc += float(val)
            st.obj_host[b] = acc
        return bool(v[0] != 0), math.sqrt(float(v[1]))

    def _reseed(self, master, new_master, new_operand):
        """reseed_farthest for a streamed pass (pipeline.py:283-309, 366-371): each
        empty cluster, in id order, takes the next-farthest point of the pass
        (distance desc, index asc), read back from the source; the shift is
        recomputed."""
        em = self.empty.cpu().numpy()
        if not em.any():
            return
        for b in range(self.stream.batch):
            empties = np.flatnonzero(em[b])
            if empties.size == 0:
                continue
            idx = _farthest(self.st.mind_all[b], int(empties.size), self.row_lo, self.group)
            rows = _rows_to_device(self.stream, b, idx, self.dev, self.group, self.row_lo, self.row_hi)
            cid = torch.from_numpy(empties[: len(idx)]).to(self.dev)
            new_master[b, cid] = rows.to(new_master.dtype)
            if new_operand is not None:
                new_operand[b, cid] = rows
        diff = new_master.double() - master.double()
        self.shift2.copy_((diff * diff).sum(-1).max())


def _init_from_stream(stream, clusters: int, seed: int, method: str, device=None, group=None,
                      runner: _StreamRunner | None = None) -> torch.Tensor:
    """Same row draws as the in-core initializer (pipeline.py:456-479); a
    file-backed source reads only the chosen rows (plus, for k-means++, the
    D^2 sweeps of pipeline.py:420-453, streamed through the device).  Sharded:
    every rank draws the same indices; each row comes from its owner."""
    if method not in INIT_METHODS:
        raise ValueError(f"init method must be one of {INIT_METHODS}")
    if clusters > stream.total_points:
        raise ValueError(f"cannot place {clusters} clusters with only {stream.total_points} points")
    if device is not None:
        dev = device
    elif method == "random_distinct" and group is None:
        dev = torch.device("cpu")  # rows only: stay on the host
    else:
        dev = torch.device("cuda", torch.cuda.current_device())
    r_lo, r_hi = (runner.row_lo, runner.row_hi) if runner is not None else (0, stream.total_points)
    out = torch.empty((stream.batch, clusters, stream.dims), dtype=stream.dtype, device=dev)
    for b in range(stream.batch):
        rng = np.random.default_rng((seed, b))
        if method == "random_distinct":
            idx = rng.choice(stream.total_points, size=clusters, replace=False)
        else:
            idx = _streaming_kmeanspp(stream, b, clusters, rng, dev, group, runner)
        out[b] = _rows_to_device(stream, b, idx, dev, group, r_lo, r_hi)
    return out


def _stream_rows_host(stream, b: int, lo: int, hi: int, buf: torch.Tensor | None) -> torch.Tensor:
    if isinstance(stream, HostStream):
        return stream.view(b, lo, hi)  # pinned slice: a true async DMA
    return stream.read_rows_into(b, lo, hi, buf)


def _streaming_kmeanspp(stream, b: int, k: int, rng: np.random.Generator, device, group=None,
                        runner: _StreamRunner | None = None) -> np.ndarray:
    """k-means++ over a chunk stream (pipeline.py:420-453): the (N,) f64 weight
    table is device-resident, every chunk is swept by fk_kmeanspp_sweep as it
    arrives and each choice() draw is resolved by fk_kmeanspp_select -- the
    same arithmetic as the in-core seeding, so the chosen rows match it (and
    the reference) index for index.  One host read per draw fetches the
    chosen index (its row is the next sweep's center).  Sharded: each rank
    sweeps its own chunks and the table slices are all-gathered per draw."""
    from . import ops

    n = stream.total_points
    idx = np.empty(k, np.int64)
    idx[0] = rng.integers(n)
    if k == 1:
        return idx
    world, rank = _group_info(group)
    if runner is not None:
        c_lo, c_hi, r_lo, r_hi = runner.c_lo, runner.c_hi, runner.row_lo, runner.row_hi
    else:
        c_lo, c_hi, r_lo, r_hi = 0, stream.n_chunks, 0, n
    pp = ops.KmeansppStream(n, k, device)
    buf = None
    if not isinstance(stream, HostStream):
        buf = torch.empty((stream.chunk_points, stream.dims), dtype=stream.dtype).pin_memory()
    if group is not None:
        import torch.distributed as dist

        shards = [stream_shard(stream, world, r)[2:] for r in range(world)]
        maxn = max(max(h - l for l, h in shards), 1)
        send = torch.zeros((maxn,), dtype=torch.float64, device=device)
        recv = torch.empty((world * maxn,), dtype=torch.float64, device=device)

    def sweep(row: int, first: bool, j: int) -> None:
        center = _rows_to_device(stream, b, [row], device, group, r_lo, r_hi)[0]
        for t in range(c_lo, c_hi):
            lo, hi = stream.bounds(t)
            rows = _stream_rows_host(stream, b, lo, hi, buf).to(device, non_blocking=buf is None)
            pp.sweep(rows, lo, center, first, j)
        if group is not None:
            send[: r_hi - r_lo].copy_(pp.m[0, r_lo:r_hi])
            dist.all_gather(list(recv.view(world, maxn).unbind(0)), send, group=group)
            for r, (l, h) in enumerate(shards):
                if h > l and r != rank:
                    pp.m[0, l:h].copy_(recv[r * maxn:r * maxn + (h - l)])

    sweep(int(idx[0]), True, 1)
    for j in range(1, k):
        state = rng.bit_generator.state
        pp.select(j, float(rng.random()))
        got = pp.idx[0, j].item()
        if int(pp.halted[0].item()) == j:  # total == 0: the reference draws integers from here on
            rng.bit_generator.state = state
            for jj in range(j, k):
                idx[jj] = rng.integers(n)
            return idx
        idx[j] = got
        if j + 1 < k:
            sweep(int(got), False, j + 1)
    return idx


def _check_stream_centroids(stream, c: Centroids, clusters: int) -> None:
    if c.batch != stream.batch or c.dims != stream.dims:
        raise ValueError("centroids do not match the stream shape")
    if c.clusters != clusters:
        raise ValueError("centroid count does not match the configuration")
    # the stream's precision, or (bf16/fp16 data) its f32 master -- what the pass returns
    if c.precision != stream.precision and c.dtype != master_dtype(stream.dtype):
        raise ValueError("centroid precision does not match the stream")


def _stream_device(device):
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if dev.type != "cuda":
        dev = torch.device("cuda", torch.cuda.current_device())
    elif dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    return dev


def _cached_runner(stream, clusters: int, dev, chunk: int, policy: str, group) -> _StreamRunner:
    """Per-stream cache of the pass machinery (device buffers, copy stream,
    events), so repeated out_of_core_iteration calls allocate nothing."""
    cache = stream.__dict__.setdefault("_fk_runners", {})
    key = (clusters, str(dev), chunk, policy, id(group))
    run = cache.get(key)
    if run is None:
        run = _StreamRunner(stream, clusters, dev, chunk, group=group, policy=policy)
        cache[key] = run
    return run


def out_of_core_iteration(stream, c: Centroids, cfg: KMeansConfig, counters: Counters,
                          store=None, workers: int | None = None, device=None, group=None):
    """One streaming Lloyd iteration (pipeline.py:385-417): returns (new
    centroids, assignment store, counters); the caller finalizes (or aborts)
    the store.  For an FKM1 ``ChunkStream`` a fresh store is the FKA1
    ``AssignmentStore`` at "<dataset>.fka1" (as in the reference); a
    host-array stream keeps its ids in a ``DeviceAssignmentStore``.

    ``group`` (a torch.distributed process group, e.g. ``dist.group.WORLD``)
    shards the pass: each rank streams its whole chunks (``stream_shard``)
    and the statistics are all-reduced once; the returned centroids are
    replicated and equal the single-process pass (bitwise for f32 data).  The
    store then holds this rank's rows only (device-resident)."""
    from .fileio import AssignmentStore

    _check_stream_centroids(stream, c, cfg.clusters)
    dev = _stream_device(device or device_of(c.data))
    tiling = _resolve_tiling(cfg, stream.total_points, stream.dims, stream.batch, stream.elem_bytes,
                             _workers(workers))
    own_store = store is None
    if store is None and group is None and getattr(stream, "path", None):
        store = AssignmentStore(stream.path + ".fka1", stream.batch, stream.total_points)
    try:
        run = _cached_runner(stream, cfg.clusters, dev, tiling.update_chunk, cfg.empty_cluster_policy,
                             group)
        if isinstance(store, DeviceAssignmentStore):
            if store.points != run.row_hi - run.row_lo or store.row_offset != run.row_lo:
                raise ValueError("assignment store does not cover this rank's rows")
            run.store = store
        elif store is None:  # a fresh pass: sentinel ids, so every point counts as changed
            run.store = DeviceAssignmentStore(stream.batch, run.row_hi - run.row_lo, dev, run.row_lo)
        run.cur = 0
        run.set(c.data)
        merges0 = int(run.st.merges.item())
        run.one_pass(counters)
        if isinstance(store, AssignmentStore):
            ids = run.store.new.cpu()
            for b in range(stream.batch):
                store.write_chunk(b, 0, ids[b])
    except BaseException:
        if own_store and isinstance(store, AssignmentStore):
            store.abort()
        raise
    counters.synchronized_merges += int(run.st.merges.item()) - merges0
    return (Centroids(run.master[1].clone(), check_finite=False),
            store if store is not None else run.store, counters)


def chunked_stream_run(stream, cfg: KMeansConfig, assign_path: str | None = None,
                       workers: int | None = None, counters: Counters | None = None,
                       device=None, group=None) -> KMeansResult:
    """Full out-of-core run (pipeline.py:482-530) with the in-core run's decisions.

    The final assignments are written as an FKA1 file (atomically) to
    ``assign_path``, default "<dataset>.fka1" for an FKM1 stream; a host-array
    stream without ``assign_path`` keeps them in memory only.

    ``group`` shards every pass across ranks (see ``out_of_core_iteration``):
    centroids, objective history, iteration count and counters are the
    replicated single-process values; ``assignments`` holds this rank's rows
    [row_lo, row_hi) of ``stream_shard``, and the FKA1 output is one file per
    rank, "<path>.<rank>-of-<world>"."""
    from .fileio import write_fka1

    counters = counters if counters is not None else Counters()
    if cfg.clusters > stream.total_points:
        raise ValueError("more clusters than points in the stream")
    dev = _stream_device(device)
    tiling = _resolve_tiling(cfg, stream.total_points, stream.dims, stream.batch, stream.elem_bytes,
                             _workers(workers))
    run = _StreamRunner(stream, cfg.clusters, dev, tiling.update_chunk, group=group,
                        policy=cfg.empty_cluster_policy)
    run.set(_init_from_stream(stream, cfg.clusters, cfg.seed, cfg.init, run.dev, group, run))
    history = []
    iterations = 0
    for it in range(1, cfg.max_iters + 1):
        iterations = it
        changed, shift = run.one_pass(counters)
        history.append(run.st.obj_host.copy())
        if not changed:
            break
        run.cur ^= 1
        if shift <= cfg.shift_tol:
            break
    counters.synchronized_merges += int(run.st.merges.item())
    a = run.store.read_all()
    path = assign_path or (stream.path + ".fka1" if getattr(stream, "path", None) else None)
    if path:
        if group is not None:
            path = f"{path}.{run.rank}-of-{run.world}"
        write_fka1(path, a)
    return KMeansResult(Centroids(run.master[run.cur].clone(), check_finite=False), a,
                        np.array(history), iterations, counters)
