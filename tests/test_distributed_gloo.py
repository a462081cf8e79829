"""World-size > 1 gloo tests of the point-sharded Lloyd path (CPU).

Each rank owns a contiguous row range; the per-iteration exchange is the
packed float64 all-reduce of LloydEngine.  The device kernels are replaced by
the oracle (tests/oracle_backend.py) so the orchestration -- ping-pong
buffers, packed exchange, global merge count, normalize on every rank -- runs
under gloo without GPUs.  With float32 data every partial sum is exact in
float64, so the sharded run must reproduce the single-process oracle's
lloyd_run bit for bit (assignments, centroids, iteration count, merges).
The same orchestration on the CUDA kernels is tests/test_gpu_sharded.py.
"""

import os

import numpy as np
import pytest
import torch

from dist_util import ROOT, spawn_world


def _lloyd_worker(rank, world, prec, chunk):
    import oracle_backend
    from oracle import oracle as O
    from paper_2603_09229_b200 import KMeansConfig
    from paper_2603_09229_b200.distributed import lloyd_run_sharded, shard_bounds

    dt = np.float32 if prec == "single" else np.float64
    x = O.generate_dataset(2, 901, 6, 5, 1.3, 17, dt)
    lo, hi = shard_bounds(x.shape[1], world, rank)
    cfg = KMeansConfig(6, max_iters=25, seed=3, precision=prec)
    r = lloyd_run_sharded(torch.from_numpy(np.ascontiguousarray(x[:, lo:hi])), x.shape[1], lo,
                          cfg, update_chunk=chunk, backend=oracle_backend)
    return (r.centroids.data.numpy(), r.assignments.values.numpy(), r.objective_history,
            r.iterations_run, r.counters.synchronized_merges)


@pytest.mark.parametrize("prec,chunk", [("single", 901), ("double", 901), ("single", 128)])
def test_sharded_lloyd_matches_single_process(oracle, prec, chunk):
    world = 2
    res = spawn_world(world, _lloyd_worker, prec, chunk)
    dt = np.float32 if prec == "single" else np.float64
    x = oracle.generate_dataset(2, 901, 6, 5, 1.3, 17, dt)
    c_ref, a_ref, h_ref, it_ref, mg_ref = oracle.lloyd_run(x, 6, max_iters=25, seed=3, chunk=chunk)
    a = np.concatenate([r[1] for r in res], axis=1)
    assert res[0][3] == res[1][3] == it_ref
    assert np.array_equal(a, a_ref)
    np.testing.assert_allclose(res[0][2], h_ref, rtol=1e-12)
    for r in res:
        if prec == "single":
            assert np.array_equal(r[0], c_ref)
        else:
            np.testing.assert_allclose(r[0], c_ref, rtol=1e-12)
        # the merge counter is the reference's GLOBAL count (sort_inverse.py:159-165),
        # not the sum of per-shard counts
        assert r[4] == mg_ref
    assert np.array_equal(res[0][0], res[1][0])  # replicas never diverge


def _kpp_worker(rank, world):
    import oracle_backend
    from kmeanspp_cases import CASES, make_case
    from paper_2603_09229_b200.distributed import kmeanspp_indices_sharded, shard_bounds

    out = {}
    for name in ("batched_f64", "duplicates_f32", "k_eq_n_f64"):
        spec = CASES[name]
        x = make_case(spec)
        lo, hi = shard_bounds(x.shape[1], world, rank)
        out[name] = kmeanspp_indices_sharded(torch.from_numpy(np.ascontiguousarray(x[:, lo:hi])),
                                             x.shape[1], lo, spec["k"], spec["seed"],
                                             backend=oracle_backend)
    return out


def test_sharded_kmeanspp_matches_reference_golden():
    """World-3 k-means++ over row shards draws the reference's indices (golden)."""
    res = spawn_world(3, _kpp_worker)
    gold = np.load(os.path.join(ROOT, "tests", "golden", "kmeanspp_golden.npz"))
    for out in res:
        for name, idx in out.items():
            assert np.array_equal(idx, gold[name]), name


def _reseed_worker(rank, world):
    import oracle_backend
    from paper_2603_09229_b200 import KMeansConfig
    from paper_2603_09229_b200.distributed import lloyd_run_sharded, shard_bounds

    g = np.load(os.path.join(ROOT, "tests", "golden", "reseed_golden.npz"))
    x = g["x"]
    lo, hi = shard_bounds(x.shape[1], world, rank)
    cfg = KMeansConfig(48, max_iters=25, seed=5, empty_cluster_policy="reseed_farthest")
    r = lloyd_run_sharded(torch.from_numpy(np.ascontiguousarray(x[:, lo:hi])), x.shape[1], lo, cfg,
                          backend=oracle_backend)
    return r.centroids.data.numpy(), r.assignments.values.numpy(), r.objective_history, r.iterations_run


def test_sharded_reseed_farthest_matches_reference_golden():
    """World-2 lloyd_run with reseed_farthest (duplicate rows leave clusters
    empty on the first pass) reproduces the reference's golden run."""
    res = spawn_world(2, _reseed_worker)
    g = np.load(os.path.join(ROOT, "tests", "golden", "reseed_golden.npz"))
    a = np.concatenate([r[1] for r in res], axis=1)
    for r in res:
        assert r[3] == int(g["iterations"])
        assert np.array_equal(r[0], g["centroids"])
        np.testing.assert_array_equal(r[2], g["history"])
    assert np.array_equal(a, g["assignments"])


@pytest.mark.parametrize("world,n,chunk", [(2, 1000, 64), (3, 10, 4), (4, 5, 2), (8, 7, 1)])
def test_stream_shard_partitions_whole_chunks(world, n, chunk):
    """Chunk-granular sharding covers every row exactly once, in rank order."""
    from paper_2603_09229_b200.pipeline import HostStream, stream_shard

    s = HostStream(torch.zeros((1, n, 2)), chunk, pin=False)
    res = [stream_shard(s, world, r) for r in range(world)]
    rows = [(r[2], r[3]) for r in res if r[3] > r[2]]
    assert rows[0][0] == 0 and rows[-1][1] == n
    for (a0, a1), (b0, b1) in zip(rows, rows[1:]):
        assert a1 == b0
    for c_lo, c_hi, r_lo, r_hi in res:
        assert (c_hi > c_lo) == (r_hi > r_lo)
        if r_hi > r_lo:
            assert r_lo == c_lo * chunk and r_hi == min(n, c_hi * chunk)
