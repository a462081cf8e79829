"""Pin the CPU oracle against golden vectors produced by the live reference.

These run everywhere (no reference sources, no GPU needed): the fixtures in
tests/golden/ were written by tests/golden/make_golden.py calling
flashmeans 0.1.0 itself.
"""

import hashlib

import numpy as np
import pytest


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.mark.parametrize("prec,dt", [("single", np.float32), ("double", np.float64)])
def test_assign_matches_reference_bitwise(golden, oracle, prec, dt):
    arr, meta = golden
    spec = meta["fixtures"][f"assign_{prec}"]
    x = oracle.generate_dataset(spec["batch"], spec["points"], spec["k_true"], spec["dims"],
                                spec["spread"], spec["seed"], dt)
    assert sha(x) == spec["x_sha"], "numpy RNG drift: regenerate fixtures"
    c = arr[f"assign_{prec}_c"]
    assert np.array_equal(c, oracle.init_centroids(x, spec["clusters"], spec["init_seed"]))
    a, m = oracle.assign(x, c)
    assert np.array_equal(a, arr[f"assign_{prec}_a"])
    assert m.dtype == dt
    assert np.array_equal(m, arr[f"assign_{prec}_m"])


@pytest.mark.parametrize("name", ["grid_small", "grid_d128", "grid_d64"])
def test_integer_grid_assign(golden, oracle, name):
    arr, _ = golden
    x = arr[name + "_x"].astype(np.float32)
    c = arr[name + "_c"].astype(np.float32)
    a, m = oracle.assign(x, c)
    assert np.array_equal(a, arr[name + "_a"])
    assert np.array_equal(m, arr[name + "_m"])
    # brute-force direct-difference oracle (test_flash_assign.py:258-281)
    d = ((x[0][:, None, :].astype(np.float64) - c[0][None, :, :]) ** 2).sum(-1)
    best = np.argmin(d, axis=1)
    assert np.array_equal(a[0], best)
    assert np.array_equal(m[0], d[np.arange(d.shape[0]), best].astype(np.float32))


@pytest.mark.parametrize("prec,dt", [("single", np.float32), ("double", np.float64)])
def test_update_and_normalize(golden, oracle, prec, dt):
    arr, meta = golden
    spec = meta["fixtures"][f"update_{prec}"]
    x = oracle.generate_dataset(2, 1000, 9, 6, 1.0, 7, dt)
    assert sha(x) == spec["x_sha"]
    ids = arr[f"update_{prec}_ids"]
    sums, counts, merges = oracle.sort_inverse_update(x, ids, spec["clusters"], spec["chunk"])
    assert np.array_equal(sums, arr[f"update_{prec}_sums"])
    assert np.array_equal(counts, arr[f"update_{prec}_counts"])
    assert merges == spec["merges"]
    out, empty = oracle.normalize(sums, counts, arr[f"update_{prec}_prev"])
    assert np.array_equal(out, arr[f"update_{prec}_norm"])
    assert empty == spec["empty"]


def test_config1_lloyd_20_iterations(golden, oracle):
    arr, meta = golden
    spec = meta["fixtures"]["cfg1"]
    x = oracle.generate_dataset(1, spec["points"], 8, spec["dims"], spec["spread"], spec["seed"],
                                np.float32)
    assert sha(x) == spec["x_sha"]
    assert np.array_equal(oracle.init_centroids(x, 8, 0), arr["cfg1_init"])
    c, a, hist, iters, merges = oracle.lloyd_run(x, 8, max_iters=spec["max_iters"],
                                                 chunk=spec["update_chunk"])
    assert iters == spec["iterations"]
    assert merges == spec["merges"]
    assert np.array_equal(c, arr["cfg1_centroids"])
    assert np.array_equal(a, arr["cfg1_assignments"])
    assert np.array_equal(hist, arr["cfg1_history"])


def test_known_answers(golden, oracle):
    _, meta = golden
    kat = meta["kat"]
    t = kat["tie_lowest_id"]
    a, m = oracle.assign(np.array(t["x"]), np.array(t["c"]))
    assert a[0, 0] == t["a"] and m[0, 0] == t["m"]
    order, a_sorted = oracle.counting_sort(np.array(kat["argsort_hand"]["ids"]), 3)
    assert order.tolist() == kat["argsort_hand"]["order"]
    assert a_sorted.tolist() == kat["argsort_hand"]["a_sorted"]
    order, _ = oracle.counting_sort(np.array(kat["argsort_stable"]["ids"]), 2)
    assert order.tolist() == kat["argsort_stable"]["order"]
    s = kat["scatter_hand"]
    sums, counts = oracle.scatter_update(np.array(s["x"]), np.array([s["ids"]]), 2)
    assert sums.tolist() == s["sums"] and counts.tolist() == s["counts"]
    sums2, counts2, _ = oracle.sort_inverse_update(np.array(s["x"]), np.array([s["ids"]]), 2, 3)
    assert np.array_equal(sums, sums2) and np.array_equal(counts, counts2)
    tb = kat["two_blobs"]
    c, _, hist, _, _ = oracle.lloyd_run(np.array(tb["x"]), 2, max_iters=50, chunk=256)
    assert sorted(c[0, :, 0].tolist()) == tb["centroids"]
    assert hist[-1, 0] == tb["objective"]
    assert oracle.row_norms(np.array(kat["row_norms"]["x"])).tolist() == kat["row_norms"]["out"]
    mc = kat["merge_count"]
    _, _, merges = oracle.sort_inverse_update(np.zeros((1, 5, 1)), np.array([mc["ids"]]), 3,
                                              mc["chunk"])
    assert merges == mc["merges"]
