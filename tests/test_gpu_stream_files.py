"""File-backed streaming (FKM1 ChunkStream -> pinned staging -> device) and the
reseed_farthest policy, against the in-core run and the reference's goldens.

Parity bar: float32 data is bitwise equal to the reference
(assignments, centroids, iteration count); bf16 streamed == bf16 in-core.
"""

import os

import numpy as np
import pytest
import torch

import paper_2603_09229_b200 as fk

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.mark.parametrize("prec,chunk", [("single", 3001), ("single", 20000), ("bf16", 4099)])
def test_fkm1_stream_matches_in_core(tmp_path, prec, chunk):
    x = fk.generate_dataset(2, 20000, 16, 32, 1.0, 9, prec)
    p = str(tmp_path / "x.fkm1")
    fk.write_fkm1(p, x)
    cfg = fk.KMeansConfig(16, max_iters=12, seed=4, precision=prec,
                          tiling=fk.TilingConfig(64, 16, 20000))
    r_in = fk.lloyd_run(fk.DataMatrix(x.data.cuda()), cfg)
    counters = fk.Counters()
    with fk.ChunkStream(p, chunk) as s:
        r_st = fk.chunked_stream_run(s, cfg, counters=counters)
    assert counters.elements_streamed == 2 * 20000 * r_st.iterations_run
    assert r_st.iterations_run == r_in.iterations_run
    assert np.array_equal(r_st.assignments.numpy(), r_in.assignments.numpy())
    if prec == "single":
        assert np.array_equal(r_st.centroids.numpy(), r_in.centroids.numpy())
    else:
        np.testing.assert_allclose(r_st.centroids.numpy(), r_in.centroids.numpy(), rtol=1e-5, atol=1e-5)
    # the FKA1 file lands at "<dataset>.fka1" and holds the final assignments
    assert np.array_equal(fk.read_fka1(p + ".fka1").numpy(), r_st.assignments.numpy())


def test_fkm1_out_of_core_iteration_store(tmp_path):
    x = fk.generate_dataset(1, 30000, 16, 32, 1.0, 10, "single")
    p = str(tmp_path / "x.fkm1")
    fk.write_fkm1(p, x)
    c = fk.init_centroids(x, 16, 1)
    with fk.ChunkStream(p, 7000) as s:
        new_c, store, counters = fk.out_of_core_iteration(s, fk.Centroids(c.data.cuda()),
                                                          fk.KMeansConfig(16, precision="single"),
                                                          fk.Counters())
    assert isinstance(store, fk.AssignmentStore)
    a, _, _ = fk.flash_assign(x, c, fk.TilingConfig(64, 16, 30000), fk.Counters())
    st, _ = fk.sort_inverse_update(x, a, 16, 30000, fk.Counters())
    ref, _ = fk.normalize(st, fk.Centroids(c.data.cuda()))
    assert np.array_equal(new_c.numpy(), ref.numpy())
    assert np.array_equal(store.read_all().numpy(), a.numpy())
    assert not os.path.exists(p + ".fka1")      # the caller finalizes
    store.finalize()
    assert np.array_equal(fk.read_fka1(p + ".fka1").numpy(), a.numpy())


def _reseed_golden():
    g = np.load(os.path.join(GOLD, "reseed_golden.npz"))
    assert int(g["first_empties"]) > 0
    return g


@pytest.mark.parametrize("engine", ["flash", "baseline"])
def test_reseed_farthest_in_core_matches_reference(engine):
    """Both engines reseed (the reference calls _reseed_in_core for either,
    pipeline.py:84-89, 133-146)."""
    g = _reseed_golden()
    cfg = fk.KMeansConfig(48, max_iters=25, seed=5, empty_cluster_policy="reseed_farthest")
    r = fk.lloyd_run(fk.DataMatrix(torch.from_numpy(g["x"]).cuda()), cfg, engine=engine)
    assert r.iterations_run == int(g["iterations"])
    assert np.array_equal(r.centroids.numpy(), g["centroids"])
    assert np.array_equal(r.assignments.numpy(), g["assignments"])
    if engine == "flash":
        np.testing.assert_array_equal(r.objective_history, g["history"])
    else:  # the materializing foil sums its own distance matrix (not bitwise)
        np.testing.assert_allclose(r.objective_history, g["history"], rtol=1e-5)


@pytest.mark.parametrize("source", ["file", "host"])
def test_reseed_farthest_streamed_matches_reference(tmp_path, source):
    g = _reseed_golden()
    cfg = fk.KMeansConfig(48, max_iters=25, seed=5, empty_cluster_policy="reseed_farthest")
    if source == "file":
        p = str(tmp_path / "x.fkm1")
        fk.write_fkm1(p, fk.DataMatrix(torch.from_numpy(g["x"])))
        with fk.ChunkStream(p, 77) as s:
            r = fk.chunked_stream_run(s, cfg)
    else:
        r = fk.chunked_stream_run(fk.HostStream(torch.from_numpy(g["x"]), 77), cfg)
    assert r.iterations_run == int(g["iterations"])
    assert np.array_equal(r.centroids.numpy(), g["centroids"])
    assert np.array_equal(r.assignments.numpy(), g["assignments"])


def test_streaming_overlaps_copy_and_compute():
    """Acceptance criterion 6's overlap half (test_acceptance.py:193-250), on the
    device: a streamed pass from pinned host memory must take clearly less than
    copying every chunk plus computing every chunk back to back (double
    buffers + a copy stream), and at least as long as the longer of the two."""
    from paper_2603_09229_b200 import ops
    from paper_2603_09229_b200.pipeline import HostStream, _StreamRunner

    N, K, d, chunk = 1 << 22, 16384, 128, 1 << 19
    g = torch.Generator(device="cuda").manual_seed(0)
    xd = (torch.randn((1, N, d), device="cuda", generator=g) * 3).to(torch.bfloat16)
    host = xd.cpu().pin_memory()
    c0 = xd[:, :K].float()
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    # copy only: every chunk H2D
    buf = torch.empty((1, chunk, d), dtype=torch.bfloat16, device="cuda")
    a, b = ev(), ev()
    torch.cuda.synchronize()
    a.record()
    for lo in range(0, N, chunk):
        buf.copy_(host[:, lo:lo + chunk], non_blocking=True)
    b.record()
    torch.cuda.synchronize()
    t_copy = a.elapsed_time(b)
    # compute only: assign + update of every (device-resident) chunk
    ids = torch.empty((1, chunk), dtype=torch.int32, device="cuda")
    mind = torch.empty((1, chunk), dtype=torch.float32, device="cuda")
    sums = torch.empty((1, K, d), dtype=torch.float64, device="cuda")
    counts = torch.empty((1, K), dtype=torch.int64, device="cuda")
    cop = c0.to(torch.bfloat16)
    for _ in range(2):  # warm both operators (first launches load their kernels)
        ops.assign(xd[:, :chunk], cop, idx_out=ids, mind_out=mind)
        ops.update(xd[:, :chunk], ids, K, chunk, accumulate=False, sums=sums, counts=counts)
    torch.cuda.synchronize()
    a.record()
    for lo in range(0, N, chunk):
        xc = xd[:, lo:lo + chunk]
        ops.assign(xc, cop, idx_out=ids, mind_out=mind)
        ops.update(xc, ids, K, chunk, accumulate=lo > 0, sums=sums, counts=counts)
    b.record()
    torch.cuda.synchronize()
    t_compute = a.elapsed_time(b)
    # the streamed pass
    stream = HostStream(host, chunk, pin=False)
    run = _StreamRunner(stream, K, torch.device("cuda", 0), N)
    run.set(c0)
    counters = fk.Counters()
    run.one_pass(counters)
    torch.cuda.synchronize()
    a.record()
    run.one_pass(counters)
    b.record()
    torch.cuda.synchronize()
    t_pass = a.elapsed_time(b)
    assert t_pass < 0.85 * (t_copy + t_compute), (t_pass, t_copy, t_compute)
    assert t_pass > 0.9 * max(t_copy, t_compute), (t_pass, t_copy, t_compute)
