"""f64 data (the reference's default precision): the device update is bitwise
equal to the reference's sort_inverse_update, whose f64 sums depend on the
addition order (sort_inverse.py:106-149: spans of `chunk` sorted positions,
serial segment sums, in-order merges; _kernels.py:135-171), and a streamed
pass equals the reference's in-order PartialStats fold (pipeline.py:250-257,
360-365).  The oracle's restatement is pinned to the live reference in
tests/test_oracle_*.py."""

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ops():
    from paper_2603_09229_b200 import ops

    return ops


def rough_data(rng, B, N, d):
    # magnitudes spread over many binades: f64 sums round, so order matters
    return (rng.standard_normal((B, N, d)) * np.exp(rng.uniform(-20, 20, (B, N, 1)))).astype(np.float64)


@pytest.mark.parametrize("B,N,K,d,chunk", [
    (1, 1, 1, 1, 1), (1, 1000, 8, 16, 256), (2, 5000, 37, 33, 777), (1, 20000, 300, 64, 20000),
    (3, 4096, 64, 128, 1000), (1, 9000, 1, 5, 64), (1, 3000, 4000, 24, 512),
    (1, 5000, 3, 8, 2),  # > 1024 spans: the single-walk kernel
])
def test_update_f64_bitwise(ops, B, N, K, d, chunk):
    rng = np.random.default_rng(N + K + d)
    x = rough_data(rng, B, N, d)
    ids = rng.integers(0, K, (B, N)).astype(np.int32)
    if K > 3:
        ids[:, : N // 3] = 2  # one heavy cluster spanning many spans
    s_ref, c_ref, m_ref = O.sort_inverse_update(x, ids, K, chunk)
    merges = torch.zeros((), dtype=torch.int64, device="cuda")
    s, c = ops.update(torch.from_numpy(x).cuda(), torch.from_numpy(ids).cuda(), K, chunk, merges=merges)
    assert np.array_equal(c.cpu().numpy(), c_ref)
    assert np.array_equal(s.cpu().numpy().view(np.uint64), s_ref.view(np.uint64))
    assert int(merges) == m_ref


def test_update_f64_streamed_fold(ops):
    """Chunks accumulated in ascending order equal the reference's fold of
    per-chunk partials: running = running + part (pipeline.py:360-365)."""
    rng = np.random.default_rng(1)
    B, N, K, d, pts, chunk = 2, 10000, 50, 40, 3000, 700
    x = rough_data(rng, B, N, d)
    ids = rng.integers(0, K, (B, N)).astype(np.int32)
    ref = None
    xd, idd = torch.from_numpy(x).cuda(), torch.from_numpy(ids).cuda()
    sums = torch.empty((B, K, d), dtype=torch.float64, device="cuda")
    counts = torch.empty((B, K), dtype=torch.int64, device="cuda")
    for lo in range(0, N, pts):
        hi = min(lo + pts, N)
        part, _, _ = O.sort_inverse_update(x[:, lo:hi], ids[:, lo:hi], K, chunk)
        ref = part if ref is None else ref + part
        ops.update(xd[:, lo:hi].contiguous(), idd[:, lo:hi].contiguous(), K, chunk,
                   accumulate=lo > 0, sums=sums, counts=counts)
    assert np.array_equal(sums.cpu().numpy().view(np.uint64), ref.view(np.uint64))


def test_update_f64_repeatable(ops):
    rng = np.random.default_rng(2)
    x = torch.from_numpy(rough_data(rng, 1, 50000, 64)).cuda()
    ids = torch.from_numpy(rng.integers(0, 128, (1, 50000)).astype(np.int32)).cuda()
    s1, _ = ops.update(x, ids, 128, 4096)
    s1 = s1.clone()
    s2, _ = ops.update(x, ids, 128, 4096)
    assert torch.equal(s1.view(torch.int64), s2.view(torch.int64))


@pytest.mark.parametrize("N", [1, 7, 8, 129, 1000, 4097, 100000, 1 << 20])
def test_objective_f64_is_numpys_pairwise_sum(ops, N):
    """pipeline._objective_row for f64 data: np.sum(m, dtype=float64) of a float64
    row is numpy's pairwise summation -- reproduced addition for addition."""
    rng = np.random.default_rng(N)
    m = rng.random((3, N)) * np.exp(rng.uniform(-30, 30, (3, N)))
    out = ops.objective(torch.from_numpy(m).cuda()).cpu().numpy()
    ref = np.array([np.sum(m[b], dtype=np.float64) for b in range(3)])
    assert np.array_equal(out.view(np.uint64), ref.view(np.uint64))


@pytest.mark.parametrize("B,N,K,d", [(2, 30000, 24, 16), (1, 70000, 200, 32)])
def test_f64_lloyd_run_every_field_bitwise(B, N, K, d):
    """f64 data end to end (the reference's default precision): centroids,
    assignments, objective history, iteration count and merge counter equal the
    oracle's lloyd_run bit for bit (assign certified or exact mirror, update in
    the reference's serial order, objective in numpy's pairwise order)."""
    import paper_2603_09229_b200 as fk

    x = O.generate_dataset(B, N, K, d, 1.0, seed=5, dtype=np.float64)
    c0 = O.init_centroids(x, K, seed=6)
    c_ref, a_ref, h_ref, it_ref, m_ref = O.lloyd_run(x, K, max_iters=8, c0=c0, chunk=4096)
    cfg = fk.KMeansConfig(K, max_iters=8, seed=6, precision="double", tiling=fk.TilingConfig(64, 16, 4096))
    r = fk.lloyd_run(fk.DataMatrix(torch.from_numpy(x).cuda()), cfg)
    assert r.iterations_run == it_ref
    assert np.array_equal(np.asarray(r.assignments.values.cpu()), a_ref)
    assert np.array_equal(np.asarray(r.centroids.data.cpu()).view(np.uint64), c_ref.view(np.uint64))
    assert np.array_equal(np.asarray(r.objective_history).view(np.uint64), h_ref.view(np.uint64))
    assert r.counters.synchronized_merges == m_ref
