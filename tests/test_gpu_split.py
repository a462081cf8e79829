"""GPU parity of the certified tensor-core assign for f32/f64 data
(csrc/fk_assign_split.cu) against the reference's exact arithmetic.

The bar is the exact mode's: ids AND min_dists bitwise equal to the oracle
(oracle.assign restates dist_block + rowmin_merge, reference
_kernels.py:32-82, pinned to the live reference by tests/test_oracle_*.py),
on random data, tie-heavy data (integer grids, duplicate centroids: the
certificate must send those rows to the exact fallback), extreme magnitudes
and every batch/shape edge.  Fast mode (reference test_flash_assign.py:172-178)
is held to its reference tolerance and, on separated blobs, to exact ids.
"""

import numpy as np
import pytest
import torch

from oracle import oracle as O

pytestmark = pytest.mark.gpu

DEV = "cuda"


@pytest.fixture(scope="module")
def ops():
    from paper_2603_09229_b200 import ops

    return ops


def run(ops, x, c, **kw):
    xd = torch.from_numpy(x).to(DEV)
    cd = torch.from_numpy(c).to(DEV)
    ids, mind = ops.assign(xd, cd, **kw)
    return ids.cpu().numpy(), mind.cpu().numpy()


def assert_exact(ops, x, c, **kw):
    a_ref, m_ref = O.assign(x, c)
    a, m = run(ops, x, c, path="split", **kw)
    assert np.array_equal(a, a_ref), f"{(a != a_ref).sum()} id mismatches"
    assert np.array_equal(m.view(np.uint8), m_ref.view(np.uint8)), "min_dists differ bitwise"


SHAPES = [  # (B, N, K, d)
    (1, 1, 1, 1), (1, 7, 3, 5), (1, 1000, 8, 16), (2, 777, 300, 17), (1, 4096, 256, 64),
    (3, 2049, 513, 100), (1, 20000, 1024, 128), (1, 5000, 4096, 32), (2, 3000, 257, 128),
]


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
@pytest.mark.parametrize("shape", SHAPES)
def test_split_random_bitwise(ops, shape, dtype):
    B, N, K, d = shape
    rng = np.random.default_rng(hash(shape) & 0xffff)
    x = rng.standard_normal((B, N, d)).astype(dtype)
    c = rng.standard_normal((B, K, d)).astype(dtype)
    assert_exact(ops, x, c)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_split_blobs_bitwise(ops, dtype):
    """The reference's own generator (separated blobs, init from data rows)."""
    x = O.generate_dataset(2, 6000, 40, 48, 0.9, seed=11, dtype=dtype)
    c = O.init_centroids(x, 64, seed=12)
    assert_exact(ops, x, c)


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_split_ties_go_to_fallback(ops, dtype):
    """Integer grids (exact ties everywhere) and duplicated centroids: the
    lowest id among equal rounded distances, as the reference picks it."""
    rng = np.random.default_rng(5)
    x = rng.integers(-3, 4, (1, 6000, 24)).astype(dtype)
    c = rng.integers(-3, 4, (1, 500, 24)).astype(dtype)
    c[0, 250:] = c[0, :250]  # every centroid twice
    assert_exact(ops, x, c)
    # points sitting exactly on centroids (distance 0, clamp at 0)
    x2 = np.concatenate([c[:, :300], x[:, :700]], axis=1)
    assert_exact(ops, x2, c)


@pytest.mark.parametrize("scale", [1e-25, 1e-12, 1e12, 1e18])
def test_split_extreme_magnitudes(ops, scale):
    rng = np.random.default_rng(7)
    x = (rng.standard_normal((1, 3000, 40)) * scale).astype(np.float32)
    c = (rng.standard_normal((1, 200, 40)) * scale).astype(np.float32)
    assert_exact(ops, x, c)


def test_split_near_ties_and_mixed_scales(ops):
    """Rows equidistant up to rounding from two centroids, and rows with one
    huge component (small products far below the row's scale)."""
    rng = np.random.default_rng(9)
    c = rng.standard_normal((1, 64, 32)).astype(np.float32)
    t = rng.random((1, 4000, 1)).astype(np.float32)
    a, b = c[:, 3], c[:, 40]
    mid = (0.5 * (a + b))[:, None, :] + 1e-7 * rng.standard_normal((1, 4000, 32)).astype(np.float32)
    x = np.where(t < 0.5, mid, mid * np.float32(1.0 + 1e-6)).astype(np.float32)
    assert_exact(ops, x, c)
    x2 = rng.standard_normal((1, 2000, 32)).astype(np.float32) * 1e-3
    x2[:, :, 0] = 1e4
    assert_exact(ops, x2, c)


def test_split_nonfinite_rows(ops):
    """inf / nan / overflowing rows: the exact fallback reproduces the
    reference (ids -1 where no distance compares below +inf)."""
    rng = np.random.default_rng(3)
    x = rng.standard_normal((1, 512, 16)).astype(np.float32)
    c = rng.standard_normal((1, 300, 16)).astype(np.float32)
    x[0, 5, 3] = np.inf
    x[0, 9, 0] = np.nan
    x[0, 11] = 3e19  # squares overflow f32
    assert_exact(ops, x, c)


def test_split_changed_flag_and_preallocated_xsplit(ops):
    rng = np.random.default_rng(4)
    x = rng.standard_normal((2, 5000, 64)).astype(np.float32)
    c = rng.standard_normal((2, 700, 64)).astype(np.float32)
    xd, cd = torch.from_numpy(x).to(DEV), torch.from_numpy(c).to(DEV)
    xs = ops.assign_xsplit(xd)
    rows = ops.xsplit_rows(xs, xd)
    assert rows.shape == (2, 5000, 128) and rows.dtype == torch.bfloat16
    ids0, _ = ops.assign(xd, cd, xsplit=xs)
    changed = torch.zeros((), dtype=torch.int32, device=DEV)
    ids1, _ = ops.assign(xd, cd, xsplit=xs, idx_prev=ids0, changed=changed)
    assert int(changed) == 0 and torch.equal(ids0, ids1)
    prev = ids0.clone()
    prev[1, 17] = (prev[1, 17] + 1) % 700
    ops.assign(xd, cd, xsplit=xs, idx_prev=prev, changed=changed)
    assert int(changed) == 1
    # the split operand is exact to 2^-16 of each value
    hi, lo = rows[..., :64].double(), rows[..., 64:].double()
    err = (hi + lo - xd.double()).abs()
    assert bool((err <= xd.double().abs() * 2.0 ** -16 + 1e-300).all())


def test_fast_mode_tolerance(ops):
    """reference test_flash_assign.py:172-178: separated blobs, fast ids equal
    exact, min_dists within rtol 1e-6.  Fast mode is served by the certified
    path, so it is in fact bitwise equal to exact (also at scale)."""
    x = O.generate_dataset(1, 200, 6, 8, 0.05, seed=41, dtype=np.float64)
    c = O.init_centroids(x, 6, seed=42)
    a_ex, m_ex = run(ops, x, c, path="mirror")
    a_f, m_f = run(ops, x, c, dot_mode="fast")
    assert np.array_equal(a_ex, a_f)
    np.testing.assert_allclose(m_f, m_ex, rtol=1e-6, atol=1e-9)
    rng = np.random.default_rng(8)
    x = rng.standard_normal((1, 30000, 64))
    c = rng.standard_normal((1, 1000, 64))
    a_ex, m_ex = O.assign(x, c)
    a_f, m_f = run(ops, x, c, dot_mode="fast")
    assert np.array_equal(a_f, a_ex) and np.array_equal(m_f, m_ex)


def test_flash_assign_dot_modes(ops):
    """The drop-in operator honours dot_mode for f32 data (flash_assign.py:203-208)."""
    import paper_2603_09229_b200 as fk

    x = fk.generate_dataset(1, 30000, 12, 64, 0.5, seed=3, precision="single")
    c = fk.init_centroids(x, 500, seed=4)
    t = fk.heuristic_config(fk.ProblemShape(30000, 500, 64, 1), fk.CacheModel(elem_bytes=4, workers=8))
    a_e, m_e, _ = fk.flash_assign(x, c, t, fk.Counters())
    a_f, m_f, _ = fk.flash_assign(x, c, t, fk.Counters(), dot_mode="fast")
    a_ref, m_ref = O.assign(np.asarray(x.data.cpu()), np.asarray(c.data.cpu()))
    assert np.array_equal(np.asarray(a_e.values.cpu()), a_ref)
    assert np.array_equal(np.asarray(m_e.cpu()), m_ref)
    assert np.array_equal(np.asarray(a_f.values.cpu()), a_ref)  # separated blobs


@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_split_engine_lloyd_matches_oracle(ops, dtype):
    """A Lloyd run large enough that the engine picks the split path by itself:
    every iteration bitwise equal to the oracle's restatement of lloyd_run."""
    from paper_2603_09229_b200.pipeline import LloydEngine

    x = O.generate_dataset(1, 40000, 30, 32, 1.0, seed=21, dtype=dtype)
    K = 96
    c0 = O.init_centroids(x, K, seed=22)
    xd = torch.from_numpy(x).to(DEV)
    assert ops.split_auto(xd, K)
    eng = LloydEngine(xd, K)
    assert eng.xsplit is not None
    eng.set_centroids(torch.from_numpy(c0))
    c = c0.copy()
    for _ in range(4):
        slot = eng.iterate()
        a_ref, _ = O.assign(x, c)
        s_ref, n_ref, _ = O.sort_inverse_update(x, a_ref, K, x.shape[1])
        c, _ = O.normalize(s_ref, n_ref, c)
        assert np.array_equal(eng.ids[slot].cpu().numpy(), a_ref)
        assert np.array_equal(eng.counts.cpu().numpy(), n_ref)
        assert np.array_equal(eng.master[eng.cur ^ 1].cpu().numpy(), c)
        eng.commit()


def test_split_streamed_iteration_matches_oracle():
    """out_of_core_iteration over a HostStream with chunks large enough for the
    split path (per chunk 40000 x 64 x 32 multiply-adds): one streamed pass ==
    the oracle's iteration, bitwise (f32)."""
    import paper_2603_09229_b200 as fk

    x = O.generate_dataset(1, 120000, 50, 32, 1.0, seed=31, dtype=np.float32)
    K = 64
    c0 = O.init_centroids(x, K, seed=32)
    cfg = fk.KMeansConfig(K, max_iters=1, precision="single", tiling=fk.TilingConfig(64, 16, 120000))
    new_c, store, _ = fk.out_of_core_iteration(fk.HostStream(torch.from_numpy(x), 40000),
                                               fk.Centroids(torch.from_numpy(c0).cuda()), cfg, fk.Counters())
    a_ref, _ = O.assign(x, c0)
    s_ref, n_ref, _ = O.sort_inverse_update(x, a_ref, K, 120000)
    c_ref, _ = O.normalize(s_ref, n_ref, c0)
    assert np.array_equal(np.asarray(new_c.data.cpu()), c_ref)
