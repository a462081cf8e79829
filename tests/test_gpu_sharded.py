"""The point-sharded paths on the CUDA kernels (no oracle backend).

One GPU is available per test box, so the multi-rank runs put every rank on
cuda:0 with the gloo backend (gloo reduces CUDA tensors through the host);
a world-1 NCCL group exercises the NCCL all-reduce itself.  What runs is the
product path: fk_assign / fk_update / fk_stats_pack / fk_merges_from_counts /
fk_normalize inside LloydEngine.exchange and the sharded streaming pass.

Parity bar: float32 data gives the single-process run bit
for bit (centroids, assignments, iteration count, merge counter; the streamed
runs' objective history too, each chunk's objective having one contributor);
the in-core sharded objective is the all-reduce of per-shard sums in numpy's
order, equal to the single-process value up to a few ulps when those f64 sums
are inexact.  bf16 gives bit-exact counts and centroids within 1e-3
(row-norm relative) of the single-process iteration.
"""

import os

import numpy as np
import pytest
import torch

import paper_2603_09229_b200 as fk
from dist_util import ROOT, spawn_world

pytestmark = pytest.mark.gpu

N, K, D = 20000, 16, 32
TILING = fk.TilingConfig(64, 16, 4096)


def _in_core_worker(rank, world, prec, max_iters):
    import torch.distributed as dist

    from paper_2603_09229_b200.distributed import lloyd_run_sharded, shard_bounds

    torch.cuda.set_device(0)
    x = fk.generate_dataset(2, N, K, D, 1.0, 21, prec).data
    lo, hi = shard_bounds(N, world, rank)
    cfg = fk.KMeansConfig(K, max_iters=max_iters, seed=6, precision=prec)
    r = lloyd_run_sharded(x[:, lo:hi].contiguous().cuda(), N, lo, cfg, update_chunk=4096,
                          group=dist.group.WORLD)
    return (r.centroids.numpy(), r.assignments.numpy(), r.objective_history, r.iterations_run,
            r.counters.synchronized_merges)


def _single(prec, max_iters):
    x = fk.generate_dataset(2, N, K, D, 1.0, 21, prec)
    cfg = fk.KMeansConfig(K, max_iters=max_iters, seed=6, precision=prec, tiling=TILING)
    return fk.lloyd_run(fk.DataMatrix(x.data.cuda()), cfg)


@pytest.mark.parametrize("backend,world", [("gloo", 2), ("gloo", 3), ("nccl", 1)])
def test_sharded_lloyd_f32_bitwise(backend, world):
    res = spawn_world(world, _in_core_worker, "single", 30, backend=backend)
    ref = _single("single", 30)
    a = np.concatenate([r[1] for r in res], axis=1)
    for c, _, hist, iters, merges in res:
        assert iters == ref.iterations_run
        assert np.array_equal(c, ref.centroids.numpy())
        # the objective is numpy's buffered pairwise order per shard, then the
        # all-reduce of the shard sums: equal to the single-process (numpy)
        # value only when the f64 sums are exact -- a few ulps otherwise
        np.testing.assert_allclose(hist, ref.objective_history, rtol=1e-13, atol=0)
        assert merges == ref.counters.synchronized_merges
    assert np.array_equal(a, ref.assignments.numpy())


@pytest.mark.parametrize("backend,world", [("gloo", 2), ("nccl", 1)])
def test_sharded_lloyd_bf16_one_iteration(backend, world):
    """One iteration from the same init: identical ids, bit-exact counts (via the
    GPU's own ids), centroids within 1e-3 of the single-process iteration."""
    res = spawn_world(world, _in_core_worker, "bf16", 1, backend=backend)
    ref = _single("bf16", 1)
    a = np.concatenate([r[1] for r in res], axis=1)
    assert np.array_equal(a, ref.assignments.numpy())
    ref_c = ref.centroids.numpy().astype(np.float64)
    for c, _, _, iters, merges in res:
        # the merge counter is evaluated on the all-reduced (global) counts
        assert iters == 1 and merges == ref.counters.synchronized_merges
        err = np.linalg.norm(c - ref_c, axis=2) / np.maximum(np.linalg.norm(ref_c, axis=2), 1e-30)
        assert err.max() <= 1e-3


def _stream_worker(rank, world, prec, chunk, shard_only, policy, init):
    import torch.distributed as dist

    from paper_2603_09229_b200.pipeline import stream_shard

    torch.cuda.set_device(0)
    if policy == "reseed_farthest":
        g = np.load(os.path.join(ROOT, "tests", "golden", "reseed_golden.npz"))
        x = torch.from_numpy(g["x"])
        cfg = fk.KMeansConfig(48, max_iters=25, seed=5, empty_cluster_policy=policy)
    else:
        x = fk.generate_dataset(2, N, K, D, 1.0, 22, prec).data
        cfg = fk.KMeansConfig(K, max_iters=12, seed=4, precision=prec, tiling=TILING, init=init)
    s = fk.HostStream(x, chunk)
    lo, hi = stream_shard(s, world, rank)[2:]
    if shard_only:  # this rank holds only its own rows in host memory
        s = fk.HostStream(x[:, lo:hi].contiguous(), chunk, row_offset=lo, total_points=x.shape[1])
    counters = fk.Counters()
    r = fk.chunked_stream_run(s, cfg, counters=counters, group=dist.group.WORLD)
    return (lo, hi, r.centroids.numpy(), r.assignments.numpy(), r.objective_history, r.iterations_run,
            counters.synchronized_merges, counters.elements_streamed)


def _stream_single(prec, chunk, policy, init):
    if policy == "reseed_farthest":
        g = np.load(os.path.join(ROOT, "tests", "golden", "reseed_golden.npz"))
        x = torch.from_numpy(g["x"])
        cfg = fk.KMeansConfig(48, max_iters=25, seed=5, empty_cluster_policy=policy)
    else:
        x = fk.generate_dataset(2, N, K, D, 1.0, 22, prec).data
        cfg = fk.KMeansConfig(K, max_iters=12, seed=4, precision=prec, tiling=TILING, init=init)
    counters = fk.Counters()
    r = fk.chunked_stream_run(fk.HostStream(x, chunk), cfg, counters=counters)
    return r, counters


@pytest.mark.parametrize("world,chunk,shard_only,policy,init", [
    (2, 3001, False, "keep", "random_distinct"),
    (3, 2500, True, "keep", "random_distinct"),
    (2, 4096, True, "keep", "kmeanspp"),
    (2, 77, True, "reseed_farthest", "random_distinct"),
])
def test_sharded_stream_run_f32_bitwise(world, chunk, shard_only, policy, init):
    """chunked_stream_run over a process group == the single-process streamed run
    (and, for the reseed case, the reference's golden run)."""
    res = spawn_world(world, _stream_worker, "single", chunk, shard_only, policy, init)
    ref, rc = _stream_single("single", chunk, policy, init)
    a = np.concatenate([r[3] for r in res], axis=1)
    assert np.array_equal(a, ref.assignments.numpy())
    for lo, hi, c, _, hist, iters, merges, streamed in res:
        assert iters == ref.iterations_run
        assert np.array_equal(c, ref.centroids.numpy())
        np.testing.assert_array_equal(hist, ref.objective_history)
        assert merges == rc.synchronized_merges and streamed == rc.elements_streamed
    if policy == "reseed_farthest":
        g = np.load(os.path.join(ROOT, "tests", "golden", "reseed_golden.npz"))
        assert ref.iterations_run == int(g["iterations"])
        assert np.array_equal(ref.centroids.numpy(), g["centroids"])


def _ooc_worker(rank, world, prec):
    import torch.distributed as dist

    torch.cuda.set_device(0)
    x = fk.generate_dataset(1, N, K, D, 1.0, 23, prec)
    c = fk.init_centroids(x, K, 2)
    s = fk.HostStream(x.data, 1000)
    new_c, store, counters = fk.out_of_core_iteration(s, fk.Centroids(c.data.cuda()),
                                                      fk.KMeansConfig(K, precision=prec),
                                                      fk.Counters(), group=dist.group.WORLD)
    return new_c.numpy(), store.row_offset, store.read_all().numpy(), counters.synchronized_merges


@pytest.mark.parametrize("prec", ["single", "fp16"])
def test_sharded_out_of_core_iteration(prec):
    res = spawn_world(2, _ooc_worker, prec)
    x = fk.generate_dataset(1, N, K, D, 1.0, 23, prec)
    c = fk.init_centroids(x, K, 2)
    new_c, store, counters = fk.out_of_core_iteration(fk.HostStream(x.data, 1000),
                                                      fk.Centroids(c.data.cuda()),
                                                      fk.KMeansConfig(K, precision=prec), fk.Counters())
    a = np.concatenate([r[2] for r in res], axis=1)
    assert np.array_equal(a, store.read_all().numpy())
    assert res[1][1] == 10000
    for r in res:
        assert r[3] == counters.synchronized_merges
        if prec == "single":
            assert np.array_equal(r[0], new_c.numpy())
        else:
            np.testing.assert_allclose(r[0], new_c.numpy(), rtol=1e-5, atol=1e-5)


def test_repeated_out_of_core_iterations_reuse_buffers():
    """The drop-in loop a user writes: out_of_core_iteration called repeatedly on
    one stream (the pass machinery is cached on the stream)."""
    x = fk.generate_dataset(1, N, K, D, 1.0, 24, "single")
    cfg = fk.KMeansConfig(K, precision="single", tiling=TILING, max_iters=5, seed=1)
    s = fk.HostStream(x.data, 3000)
    c = fk.Centroids(fk.init_centroids(x, K, 1).data)
    store = fk.DeviceAssignmentStore(1, N, torch.device("cuda", 0))
    for _ in range(5):
        c, store, _ = fk.out_of_core_iteration(s, c, cfg, fk.Counters(), store=store)
    assert len(s._fk_runners) == 1
    r = fk.lloyd_run(fk.DataMatrix(x.data.cuda()), cfg)
    # lloyd_run stops early only at a fixed point, which further passes reproduce bitwise
    assert np.array_equal(c.numpy(), r.centroids.numpy())


@pytest.mark.parametrize("backend,world", [("gloo", 2), ("nccl", 1)])
def test_sharded_lloyd_f32_split_path_bitwise(backend, world):
    """Every rank on the certified tensor-core f32 assign (FK_ASSIGN_F32=split):
    still bit for bit the single-process run (which may take the exact mirror)."""
    res = spawn_world(world, _in_core_worker, "single", 30, backend=backend, env={"FK_ASSIGN_F32": "split"})
    ref = _single("single", 30)
    a = np.concatenate([r[1] for r in res], axis=1)
    assert np.array_equal(a, ref.assignments.numpy())
    for c, _, hist, iters, merges in res:
        assert iters == ref.iterations_run
        assert np.array_equal(c, ref.centroids.numpy())
        np.testing.assert_allclose(hist, ref.objective_history, rtol=1e-13, atol=0)  # see above


def test_sharded_stream_run_f32_split_path_bitwise():
    res = spawn_world(2, _stream_worker, "single", 3001, True, "keep", "random_distinct",
                      env={"FK_ASSIGN_F32": "split"})
    ref, rc = _stream_single("single", 3001, "keep", "random_distinct")
    a = np.concatenate([r[3] for r in res], axis=1)
    assert np.array_equal(a, ref.assignments.numpy())
    for lo, hi, c, _, hist, iters, merges, streamed in res:
        assert iters == ref.iterations_run
        assert np.array_equal(c, ref.centroids.numpy())
        np.testing.assert_array_equal(hist, ref.objective_history)
