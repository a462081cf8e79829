"""k-means++ seeding: the oracle pinned to the reference's own draws, and the
host-side logic of the device seeding (RNG handling, integer-draw replay).

The golden indices in tests/golden/kmeanspp_golden.npz were written by the
live reference (tests/golden/make_kmeanspp_golden.py calling
core._kmeanspp_indices, core.py:342-357); the inputs are rebuilt from
tests/kmeanspp_cases.py and checked by sha256.
"""

import hashlib
import json
import os

import numpy as np
import pytest
import torch

from kmeanspp_cases import CASES, make_case

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def sha(a):
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


@pytest.fixture(scope="module")
def kpp_golden():
    arrays = np.load(os.path.join(GOLDEN, "kmeanspp_golden.npz"))
    with open(os.path.join(GOLDEN, "kmeanspp_golden.json")) as f:
        meta = json.load(f)
    return arrays, meta


@pytest.mark.parametrize("name", sorted(CASES))
def test_oracle_kmeanspp_matches_reference_golden(kpp_golden, oracle, name):
    arr, meta = kpp_golden
    spec = meta["cases"][name]
    x = make_case(CASES[name])
    assert sha(x) == spec["x_sha"], "input drift: regenerate tests/golden/kmeanspp_golden.*"
    got = np.stack([oracle.kmeanspp_indices(x[b], spec["k"], np.random.default_rng((spec["seed"], b)))
                    for b in range(x.shape[0])])
    assert np.array_equal(got, arr[name])


def test_oracle_pairwise_sum_is_numpys(oracle):
    rng = np.random.default_rng(0)
    for n in (1, 7, 8, 9, 127, 128, 129, 1000, 65537, 1 << 20):
        a = rng.random(n) * 10.0 ** rng.uniform(-6, 6, n)
        assert oracle.pairwise_sum(a) == a.sum()


def test_replay_of_integer_draws_matches_reference_tail(kpp_golden, oracle):
    """The device seeding stops at the first draw whose total is 0; the host
    replays rng.integers for the rest.  Rebuild that tail from the golden
    prefix and compare with the reference's full draw."""
    from paper_2603_09229_b200.core import _replay_integer_draws

    arr, meta = kpp_golden
    spec = meta["cases"]["duplicates_f32"]
    x = make_case(CASES["duplicates_f32"])
    hit = 0
    for b in range(x.shape[0]):
        gold = arr["duplicates_f32"][b]
        # the first draw j whose table sums to 0: the centers so far cover every distinct row
        distinct = {tuple(r) for r in x[b]}
        seen = set()
        halted = None
        for j in range(1, spec["k"]):
            seen.add(tuple(x[b][gold[j - 1]]))
            if len(seen) == len(distinct):
                halted = j
                break
        assert halted is not None
        idx = gold.copy()
        idx[halted:] = -1
        _replay_integer_draws(idx, spec["seed"], b, x.shape[1], halted)
        assert np.array_equal(idx, gold)
        hit += 1
    assert hit == 2


def test_kmeanspp_needs_device_data():
    from paper_2603_09229_b200.core import init_indices

    with pytest.raises(ValueError, match="device"):
        init_indices(100, 4, 0, 1, "kmeanspp", torch.zeros(1, 100, 3))


def test_kmeanspp_abi_validates_before_launch():
    from paper_2603_09229_b200 import _native as N

    L = N.lib()
    assert L.fk_kmeanspp_workspace(0, 10, 3, 4) == 0
    assert L.fk_kmeanspp_workspace(1, 10, 0, 0) > 0
    assert L.fk_kmeanspp_workspace(1, 10, 3, 4) > L.fk_kmeanspp_workspace(1, 10, 0, 0)
    # K > N
    assert L.fk_kmeanspp(N.FK_F32, 16, 1, 10, 4, 11, 16, 16, 16, 16, 16, 1 << 20, None) == N.FK_EINVAL
    # missing u with K > 1
    assert L.fk_kmeanspp(N.FK_F32, 16, 1, 10, 4, 3, None, 16, 16, 16, 16, 1 << 20, None) == N.FK_EINVAL
    # workspace too small
    assert L.fk_kmeanspp(N.FK_F32, 16, 1, 10, 4, 3, 16, 16, 16, 16, 16, 1, None) == N.FK_EWORKSPACE
    # draw index outside [1, K)
    assert L.fk_kmeanspp_select(16, 1, 10, 16, 3, 3, 16, 16, 16, 1 << 20, None) == N.FK_EINVAL
    assert L.fk_kmeanspp_sweep(9, 16, 1, 10, 4, 40, 16, 4, 16, 10, 1, None, 1, None) == N.FK_EINVAL
