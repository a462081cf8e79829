"""The public drop-in API on a B200: reference semantics end to end.

* config 1 of BASELINE.json (N=10k, d=16, K=8 fp32, 20 Lloyd iterations, fixed
  init) reproduces the reference's golden run bit for bit (assignments,
  centroids, iteration count, merge counter);
* bf16 per-iteration parity from identical (X, C_t) under the north-star
  tolerances;
* the out-of-core streaming driver reproduces the in-core run;
* validation errors match the reference's ValueError contract.
"""

import hashlib

import numpy as np
import pytest
import torch

import paper_2603_09229_b200 as fk

pytestmark = pytest.mark.gpu


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def test_config1_lloyd_bitwise(golden):
    arr, meta = golden
    spec = meta["fixtures"]["cfg1"]
    x = fk.generate_dataset(1, spec["points"], 8, spec["dims"], spec["spread"], spec["seed"], "single")
    assert sha(x.numpy()) == spec["x_sha"]
    cfg = fk.KMeansConfig(8, max_iters=spec["max_iters"], seed=0, precision="single",
                          tiling=fk.TilingConfig(1024, 8, spec["update_chunk"]))
    r = fk.lloyd_run(fk.DataMatrix(x.data.cuda()), cfg)
    assert r.iterations_run == spec["iterations"]
    assert np.array_equal(r.assignments.numpy(), arr["cfg1_assignments"])
    assert np.array_equal(r.centroids.numpy(), arr["cfg1_centroids"])
    assert r.counters.synchronized_merges == spec["merges"]
    np.testing.assert_allclose(r.objective_history, arr["cfg1_history"], rtol=1e-13)


def test_two_blob_hand_solution(golden):
    _, meta = golden
    kat = meta["kat"]["two_blobs"]
    x = fk.DataMatrix(torch.tensor(kat["x"], dtype=torch.float64).cuda())
    for seed in range(4):
        r = fk.lloyd_run(x, fk.KMeansConfig(2, seed=seed, max_iters=50))
        np.testing.assert_allclose(sorted(r.centroids.numpy()[0, :, 0]), [0.05, 10.05], atol=1e-12)
        assert abs(r.objective_history[-1, 0] - 0.01) <= 1e-9


def test_k_equals_n_converges_to_zero():
    x = fk.DataMatrix(torch.from_numpy(np.random.default_rng(0).normal(size=(2, 12, 3))).cuda())
    r = fk.lloyd_run(x, fk.KMeansConfig(12, seed=3))
    assert r.iterations_run <= 2
    assert np.all(r.objective_history[-1] == 0.0)
    assert np.all(fk.kmeans_objective(x, r.centroids, r.assignments) == 0.0)


def test_flash_assign_dropin(golden):
    arr, meta = golden
    spec = meta["fixtures"]["assign_single"]
    x = fk.generate_dataset(spec["batch"], spec["points"], spec["k_true"], spec["dims"], spec["spread"],
                            spec["seed"], "single")
    c = fk.Centroids(torch.from_numpy(arr["assign_single_c"]))
    counters = fk.Counters()
    a, m, cnt = fk.flash_assign(x, c, fk.TilingConfig(8, 4, 64), counters)
    assert cnt is counters and counters.as_dict() == fk.Counters().as_dict()
    assert np.array_equal(a.numpy(), arr["assign_single_a"])
    assert m.dtype == torch.float32 and np.array_equal(m.cpu().numpy(), arr["assign_single_m"])
    with pytest.raises(ValueError):
        fk.flash_assign(x, c, fk.TilingConfig(4, 2, 2), counters, dot_mode="blas")
    with pytest.raises(ValueError):
        fk.flash_assign(x, fk.Centroids(torch.zeros((2, 2, 4))), fk.TilingConfig(4, 2, 2), counters)
    with pytest.raises(ValueError):
        fk.flash_assign(x, fk.Centroids(torch.zeros((2, 2, spec["dims"]), dtype=torch.float64)),
                        fk.TilingConfig(4, 2, 2), counters)


def test_tie_resolves_to_lowest_id():
    for dt in (torch.float32, torch.float64, torch.bfloat16, torch.float16):
        x = fk.DataMatrix(torch.tensor([[[1.0, 2.0] + [0.0] * 6]], dtype=dt))
        c = fk.Centroids(torch.tensor([[[0.0, 0.0] + [0.0] * 6, [2.0, 0.0] + [0.0] * 6]], dtype=dt))
        a, m, _ = fk.flash_assign(x, c, fk.TilingConfig(1, 1, 1), fk.Counters())
        assert int(a.values[0, 0]) == 0 and float(m[0, 0]) == 5.0


def test_sort_inverse_and_normalize_dropin(golden):
    arr, meta = golden
    spec = meta["fixtures"]["update_single"]
    x = fk.generate_dataset(2, 1000, 9, 6, 1.0, 7, "single")
    counters = fk.Counters()
    st, _ = fk.sort_inverse_update(x, fk.Assignments(arr["update_single_ids"]), 17, 128, counters)
    assert counters.synchronized_merges == spec["merges"]
    assert np.array_equal(st.sums.cpu().numpy(), arr["update_single_sums"])
    assert np.array_equal(st.counts.cpu().numpy(), arr["update_single_counts"])
    nc, empty = fk.normalize(st, fk.Centroids(torch.from_numpy(arr["update_single_prev"])))
    assert np.array_equal(nc.numpy(), arr["update_single_norm"]) and empty == spec["empty"]
    with pytest.raises(ValueError):
        fk.sort_inverse_update(x, fk.Assignments(np.full((2, 1000), 17, np.int32)), 17, 128, counters)


def test_normalize_empty_keeps_previous_bitwise():
    stats = fk.ClusterStats(torch.tensor([[[5.0], [0.0], [7.0]]], dtype=torch.float64),
                            torch.tensor([[1, 0, 2]], dtype=torch.int64))
    prev_row = 0.1 + 0.2
    prev = fk.Centroids(torch.tensor([[[1.0], [prev_row], [2.0]]], dtype=torch.float64))
    c, empty = fk.normalize(stats, prev)
    assert c.numpy()[0, 1, 0].tobytes() == np.float64(prev_row).tobytes()
    assert c.numpy()[0, 0, 0] == 5.0 and c.numpy()[0, 2, 0] == 3.5 and empty == [[1]]


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
def test_low_precision_iteration_parity(oracle, dtype):
    """One Lloyd iteration from identical (X, C_t): the north-star bars."""
    x = fk.generate_dataset(1, 65536, 64, 128, 1.0, 5, "bf16" if dtype == torch.bfloat16 else "fp16")
    xd = x.data.cuda()
    c0 = fk.init_centroids(fk.DataMatrix(xd, check_finite=False), 1024, 1).data
    eng = fk.LloydEngine(xd, 1024)
    eng.set_centroids(c0)
    slot = eng.iterate()
    torch.cuda.synchronize()
    ids = eng.ids[slot].cpu().numpy()
    x32 = x.data.float().numpy()
    c32 = c0.float().cpu().numpy()
    a_ref, _ = oracle.assign(x32, c32)
    mism = ids != a_ref
    if mism.any():
        d = lambda a: ((x32[0] - c32[0][a[0]]) ** 2).astype(np.float64).sum(-1)  # noqa: E731
        dg, dr = d(ids)[mism[0]], d(a_ref)[mism[0]]
        assert np.all(np.abs(dg - dr) <= 1e-3 * dr)
    assert mism.mean() < 1e-3
    # counts bit-exact and centroids within 1e-3 given the GPU's own ids
    s_ref, c_ref, _ = oracle.sort_inverse_update(x32, ids, 1024, 65536)
    assert np.array_equal(eng.counts.cpu().numpy(), c_ref)
    new_ref, _ = oracle.normalize(s_ref, c_ref, c32)
    new = eng.master[eng.cur ^ 1].cpu().numpy()
    rel = np.linalg.norm(new - new_ref, axis=-1) / np.maximum(np.linalg.norm(new_ref, axis=-1), 1e-30)
    assert rel.max() <= 1e-3


def test_bf16_lloyd_run_monotone():
    x = fk.generate_dataset(2, 20000, 32, 64, 1.2, 8, "bf16")
    r = fk.lloyd_run(fk.DataMatrix(x.data.cuda()), fk.KMeansConfig(64, max_iters=15, seed=2))
    h = r.objective_history
    assert h.shape == (r.iterations_run, 2)
    assert np.all(h[1:] <= h[:-1] * (1 + 1e-5))


@pytest.mark.parametrize("prec", ["single", "bf16"])
@pytest.mark.parametrize("chunk", [1000, 4099, 20000])
def test_streaming_matches_in_core(prec, chunk):
    x = fk.generate_dataset(2, 20000, 16, 32, 1.0, 9, prec)
    cfg = fk.KMeansConfig(16, max_iters=12, seed=4, precision=prec,
                          tiling=fk.TilingConfig(64, 16, 20000))
    r_in = fk.lloyd_run(fk.DataMatrix(x.data.cuda()), cfg)
    stream = fk.HostStream(x.data, chunk)
    counters = fk.Counters()
    r_st = fk.chunked_stream_run(stream, cfg, counters=counters)
    assert counters.elements_streamed == 2 * 20000 * r_st.iterations_run
    assert r_st.iterations_run == r_in.iterations_run
    assert np.array_equal(r_st.assignments.numpy(), r_in.assignments.numpy())
    if prec == "single":
        assert np.array_equal(r_st.centroids.numpy(), r_in.centroids.numpy())
    else:
        np.testing.assert_allclose(r_st.centroids.numpy(), r_in.centroids.numpy(), rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(r_st.objective_history, r_in.objective_history, rtol=1e-6)


def test_out_of_core_iteration_equals_in_core_step():
    x = fk.generate_dataset(1, 30000, 16, 32, 1.0, 10, "single")
    c = fk.init_centroids(x, 16, 1)
    new_c, store, counters = fk.out_of_core_iteration(fk.HostStream(x.data, 7000), fk.Centroids(c.data.cuda()),
                                                      fk.KMeansConfig(16, precision="single"), fk.Counters())
    a, _, _ = fk.flash_assign(x, c, fk.TilingConfig(64, 16, 30000), fk.Counters())
    st, _ = fk.sort_inverse_update(x, a, 16, 30000, fk.Counters())
    ref, _ = fk.normalize(st, fk.Centroids(c.data.cuda()))
    assert np.array_equal(new_c.numpy(), ref.numpy())
    assert np.array_equal(store.read_all().numpy(), a.numpy())
    assert counters.elements_streamed == 30000


def test_baseline_engine_agrees_on_separated_blobs():
    x = fk.generate_dataset(1, 3000, 5, 8, 0.05, 41, "double")
    cfg = fk.KMeansConfig(5, max_iters=30, seed=3)
    rf = fk.lloyd_run(fk.DataMatrix(x.data.cuda()), cfg)
    rb = fk.lloyd_run(fk.DataMatrix(x.data.cuda()), cfg, engine="baseline")
    assert rf.iterations_run == rb.iterations_run
    assert np.array_equal(rf.assignments.numpy(), rb.assignments.numpy())
    np.testing.assert_allclose(rf.centroids.numpy(), rb.centroids.numpy(), rtol=1e-12)


@pytest.mark.parametrize("prec", ["bf16", "fp16"])
def test_pipelined_runs_with_hist_fold_equal_stepwise(prec):
    """bf16/fp16: LloydEngine.run folds the update's histogram pass into the
    assign epilogue (fk_assign_hist / fk_update_prehist); iterate() does not.
    Two consecutive runs (the first ends with a speculative assign whose table
    the second must clear) equal the stepwise loop bit for bit."""
    from paper_2603_09229_b200 import LloydEngine

    x = fk.generate_dataset(3, 20000, 24, 32, 1.0, 7, prec).data.cuda()
    c0 = torch.stack([x[b, :48] for b in range(3)]).float()
    eng = LloydEngine(x, 48, 4096)
    assert eng._fold is not None
    eng.set_centroids(c0)
    ref = LloydEngine(x, 48, 4096)
    ref.set_centroids(c0)
    # runs stopped by the shift test after one iteration leave a speculative
    # assign behind (its histogram in the table); the next run clears it
    for n_it in (1, 1, 3, 1, 2):
        if n_it == 1:
            its, slot, _ = eng.run(10, 1e30)
        else:
            its, slot, _ = eng.run(n_it, -1.0, stop_on_repeat=False)
        assert its == n_it
        for _ in range(n_it):
            slot_b = ref.iterate()
            ref.poll()
            ref.commit()
        torch.cuda.synchronize()
        assert torch.equal(eng.centroids, ref.centroids)
        assert torch.equal(eng.ids[slot], ref.ids[slot_b])
        assert torch.equal(eng.counts, ref.counts)


@pytest.mark.parametrize("stop_iter_cap", [3, 40])
def test_pipelined_run_equals_stepwise_loop(stop_iter_cap):
    """LloydEngine.run queues the next assign before each poll (speculation);
    its decisions and results must equal the plain iterate/poll/commit loop.
    f32 data: every kernel is deterministic, so the comparison is bitwise."""
    from paper_2603_09229_b200 import LloydEngine

    x = fk.generate_dataset(2, 5000, 11, 24, 1.5, 3, "single").data.cuda()
    c0 = torch.stack([x[b, :37] for b in range(2)]).float()

    eng = LloydEngine(x, 37, 777)
    eng.set_centroids(c0)
    hist_a = torch.empty((stop_iter_cap, 2), dtype=torch.float64, device="cuda")
    its_a, slot_a, merges_a = eng.run(stop_iter_cap, 0.0, hist_a)
    torch.cuda.synchronize()
    c_a, ids_a = eng.centroids.clone(), eng.ids[slot_a].clone()

    ref = LloydEngine(x, 37, 777)
    ref.set_centroids(c0)
    hist_b = torch.empty((stop_iter_cap, 2), dtype=torch.float64, device="cuda")
    its_b, slot_b = 0, 0
    for it in range(1, stop_iter_cap + 1):
        its_b = it
        slot_b = ref.iterate(hist_b[it - 1])
        changed, shift = ref.poll()
        if it > 1 and not changed:
            break
        ref.commit()
        if shift <= 0.0:
            break
    assert its_a == its_b
    assert torch.equal(c_a, ref.centroids)
    assert torch.equal(ids_a, ref.ids[slot_b])
    assert torch.equal(hist_a[:its_a], hist_b[:its_b])
    assert merges_a == int(ref.merges.item())
