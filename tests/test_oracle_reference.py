"""Pin the CPU oracle against the LIVE reference on randomized instances.

Runs only where /root/reference exists (the build container); skipped on the
GPU box, where tests/test_oracle_golden.py carries the pinning instead.
Mirrors the reference's acceptance criteria 1-3 (test_acceptance.py:84-142):
randomized B, N, K, d; bitwise assignments/min_dists/stats.
"""

import numpy as np
import pytest


@pytest.mark.parametrize("prec,dt", [("single", np.float32), ("double", np.float64)])
def test_randomized_assign_update_normalize(reference, oracle, prec, dt):
    fm = reference
    rng = np.random.default_rng(1234 if prec == "single" else 4321)
    for trial in range(40):
        B = int(rng.integers(1, 3))
        N = int(rng.integers(1, 600))
        K = int(rng.integers(1, min(N, 40) + 1))
        d = int(rng.integers(1, 33))
        x = fm.generate_dataset(B, N, max(1, K // 2), d, float(rng.uniform(0.1, 2.0)),
                                int(rng.integers(0, 1 << 30)), prec)
        c = fm.init_centroids(x, K, int(rng.integers(0, 1 << 30)))
        t = fm.TilingConfig(int(rng.integers(1, 64)), int(rng.integers(1, 16)),
                            int(rng.integers(1, N + 1)))
        a, m, _ = fm.flash_assign(x, c, t, fm.Counters())
        ao, mo = oracle.assign(x.data, c.data)
        assert np.array_equal(a.values, ao)
        assert np.array_equal(m, mo)
        cnt = fm.Counters()
        st, _ = fm.sort_inverse_update(x, a, K, t.update_chunk, cnt)
        so, co, mg = oracle.sort_inverse_update(x.data, a.values, K, t.update_chunk)
        assert np.array_equal(st.sums, so)
        assert np.array_equal(st.counts, co)
        assert mg == cnt.synchronized_merges
        nc, empty = fm.normalize(st, c)
        no, eo = oracle.normalize(so, co, c.data)
        assert np.array_equal(nc.data, no) and empty == eo


@pytest.mark.parametrize("prec,dt", [("single", np.float32), ("double", np.float64)])
def test_lloyd_run_matches(reference, oracle, prec, dt):
    fm = reference
    x = fm.generate_dataset(2, 700, 6, 9, 1.1, 77, prec)
    t = fm.TilingConfig(64, 8, 100)
    r = fm.lloyd_run(x, fm.KMeansConfig(6, max_iters=30, seed=5, precision=prec, tiling=t))
    c, a, hist, iters, merges = oracle.lloyd_run(x.data, 6, max_iters=30, seed=5, chunk=100)
    assert iters == r.iterations_run
    assert merges == r.counters.synchronized_merges
    assert np.array_equal(c, r.centroids.data)
    assert np.array_equal(a, r.assignments.values)
    assert np.array_equal(hist, r.objective_history)


def test_generate_and_init_match(reference, oracle):
    fm = reference
    for prec, dt in (("single", np.float32), ("double", np.float64)):
        x = fm.generate_dataset(3, 257, 5, 7, 0.7, 11, prec)
        assert np.array_equal(x.data, oracle.generate_dataset(3, 257, 5, 7, 0.7, 11, dt))
        c = fm.init_centroids(x, 9, 4)
        assert np.array_equal(c.data, oracle.init_centroids(x.data, 9, 4))


def test_bf16_upcast_bridge(reference, oracle):
    """bf16 inputs reach the oracle as their exact fp32 upcast."""
    import torch

    fm = reference
    x = fm.generate_dataset(1, 300, 5, 16, 1.0, 3, "single")
    xb = torch.from_numpy(x.data).to(torch.bfloat16).float().numpy()
    c = xb[:, :7].copy()
    a, m, _ = fm.flash_assign(fm.DataMatrix(xb), fm.Centroids(c), fm.TilingConfig(64, 8, 64),
                              fm.Counters())
    ao, mo = oracle.assign(xb, c)
    assert np.array_equal(a.values, ao) and np.array_equal(m, mo)
