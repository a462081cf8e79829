"""World-size-2 gloo test of the point-sharded Lloyd path (CPU).

Each rank owns a contiguous row range; the per-iteration exchange is the
packed float64 all-reduce of LloydEngine.  With float32 data every partial
sum is exact in float64, so the sharded run must reproduce the single-process
oracle's lloyd_run bit for bit (assignments, centroids, iteration count).
"""

import os
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _worker(rank, world, port, result_q, prec):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle_backend
        from oracle import oracle as O
        from paper_2603_09229_b200 import KMeansConfig
        from paper_2603_09229_b200.distributed import lloyd_run_sharded, shard_bounds

        dt = np.float32 if prec == "single" else np.float64
        x = O.generate_dataset(2, 901, 6, 5, 1.3, 17, dt)
        lo, hi = shard_bounds(x.shape[1], world, rank)
        cfg = KMeansConfig(6, max_iters=25, seed=3, precision=prec)
        r = lloyd_run_sharded(torch.from_numpy(np.ascontiguousarray(x[:, lo:hi])), x.shape[1], lo,
                              cfg, update_chunk=x.shape[1], backend=oracle_backend)
        result_q.put((rank, lo, hi, r.centroids.data.numpy(), r.assignments.values.numpy(),
                      r.objective_history, r.iterations_run))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("prec", ["single", "double"])
def test_sharded_lloyd_matches_single_process(oracle, prec):
    world = 2
    port = 29500 + (os.getpid() % 2000)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, prec)) for r in range(world)]
    for p in procs:
        p.start()
    res = []
    import queue as _queue
    import time as _time
    deadline = _time.time() + 240
    while len(res) < world and _time.time() < deadline:
        try:
            res.append(q.get(timeout=2))
        except _queue.Empty:
            if any(p.exitcode not in (None, 0) for p in procs):
                break
    for p in procs:
        if p.exitcode is None and len(res) < world:
            p.terminate()
    assert len(res) == world, "a rank failed"
    res = sorted(res, key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    dt = np.float32 if prec == "single" else np.float64
    x = oracle.generate_dataset(2, 901, 6, 5, 1.3, 17, dt)
    c_ref, a_ref, h_ref, it_ref, _ = oracle.lloyd_run(x, 6, max_iters=25, seed=3)
    a = np.concatenate([r[4] for r in res], axis=1)
    assert res[0][6] == res[1][6] == it_ref
    assert np.array_equal(a, a_ref)
    np.testing.assert_allclose(res[0][5], h_ref, rtol=1e-12)
    for r in res:
        if prec == "single":
            assert np.array_equal(r[3], c_ref)
        else:
            np.testing.assert_allclose(r[3], c_ref, rtol=1e-12)
    assert np.array_equal(res[0][3], res[1][3])  # replicas never diverge


def _kpp_worker(rank, world, port, result_q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
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
        result_q.put((rank, out))
    finally:
        dist.destroy_process_group()


def test_sharded_kmeanspp_matches_reference_golden():
    """World-3 k-means++ over row shards draws the reference's indices (golden)."""
    world = 3
    port = 31500 + (os.getpid() % 2000)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_kpp_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    import queue as _queue
    import time as _time
    res, deadline = [], _time.time() + 240
    while len(res) < world and _time.time() < deadline:
        try:
            res.append(q.get(timeout=2))
        except _queue.Empty:
            if any(p.exitcode not in (None, 0) for p in procs):
                break
    for p in procs:
        if p.exitcode is None and len(res) < world:
            p.terminate()
    assert len(res) == world, "a rank failed"
    for p in procs:
        p.join(timeout=60)
    gold = np.load(os.path.join(ROOT, "tests", "golden", "kmeanspp_golden.npz"))
    for _, out in res:
        for name, idx in out.items():
            assert np.array_equal(idx, gold[name]), name


def _reseed_worker(rank, world, port, result_q):
    sys.path.insert(0, ROOT)
    sys.path.insert(0, os.path.join(ROOT, "tests"))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle_backend
        from paper_2603_09229_b200 import KMeansConfig
        from paper_2603_09229_b200.distributed import lloyd_run_sharded, shard_bounds

        g = np.load(os.path.join(ROOT, "tests", "golden", "reseed_golden.npz"))
        x = g["x"]
        lo, hi = shard_bounds(x.shape[1], world, rank)
        cfg = KMeansConfig(48, max_iters=25, seed=5, empty_cluster_policy="reseed_farthest")
        r = lloyd_run_sharded(torch.from_numpy(np.ascontiguousarray(x[:, lo:hi])), x.shape[1], lo, cfg,
                              backend=oracle_backend)
        result_q.put((rank, r.centroids.data.numpy(), r.assignments.values.numpy(),
                      r.objective_history, r.iterations_run))
    finally:
        dist.destroy_process_group()


def test_sharded_reseed_farthest_matches_reference_golden():
    """World-2 lloyd_run with reseed_farthest (duplicate rows leave clusters
    empty on the first pass) reproduces the reference's golden run."""
    world = 2
    port = 33500 + (os.getpid() % 2000)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_reseed_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    import queue as _queue
    import time as _time
    res, deadline = [], _time.time() + 240
    while len(res) < world and _time.time() < deadline:
        try:
            res.append(q.get(timeout=2))
        except _queue.Empty:
            if any(p.exitcode not in (None, 0) for p in procs):
                break
    for p in procs:
        if p.exitcode is None and len(res) < world:
            p.terminate()
    assert len(res) == world, "a rank failed"
    for p in procs:
        p.join(timeout=60)
    res = sorted(res, key=lambda t: t[0])
    g = np.load(os.path.join(ROOT, "tests", "golden", "reseed_golden.npz"))
    a = np.concatenate([r[2] for r in res], axis=1)
    for r in res:
        assert r[4] == int(g["iterations"])
        assert np.array_equal(r[1], g["centroids"])
        np.testing.assert_array_equal(r[3], g["history"])
    assert np.array_equal(a, g["assignments"])
