"""Device k-means++ seeding (fk_kmeanspp) == the reference's numpy seeding.

Every case of tests/kmeanspp_cases.py is seeded on the GPU and compared index
for index with the golden draws the live reference produced
(tests/golden/kmeanspp_golden.npz) and with the oracle restatement.  The
certified-window selection and the literal serial fallback are both
exercised (FK_PP_FORCE_EXACT=1 routes every draw through the fallback).
"""

import json
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

from kmeanspp_cases import CASES, case_tensor, make_case

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


@pytest.fixture(scope="module")
def kpp_golden():
    return np.load(os.path.join(GOLDEN, "kmeanspp_golden.npz"))


@pytest.mark.parametrize("name", sorted(CASES))
def test_device_kmeanspp_matches_reference(kpp_golden, name):
    from paper_2603_09229_b200.core import kmeanspp_indices_device

    spec = CASES[name]
    x = case_tensor(spec).cuda()
    idx = kmeanspp_indices_device(x, spec["k"], spec["seed"])
    assert np.array_equal(idx, kpp_golden[name])


def test_forced_exact_fallback_matches(kpp_golden):
    """Run two cases in a child process with every draw sent through the serial
    numpy replica (k_pp_exact) -- the rarely taken branch must be exact too."""
    code = (
        "import sys, numpy as np; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
        "from kmeanspp_cases import CASES, case_tensor\n"
        "from paper_2603_09229_b200.core import kmeanspp_indices_device\n"
        "g = np.load(%r)\n"
        "for name in ('batched_f64', 'bf16_d128', 'duplicates_f32', 'large_f32'):\n"
        "    s = CASES[name]\n"
        "    idx = kmeanspp_indices_device(case_tensor(s).cuda(), s['k'], s['seed'])\n"
        "    assert np.array_equal(idx, g[name]), name\n"
        "print('ok')\n" % (ROOT, os.path.join(ROOT, "tests"), os.path.join(GOLDEN, "kmeanspp_golden.npz")))
    env = dict(os.environ, FK_PP_FORCE_EXACT="1")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, r.stderr[-3000:]


@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float32, torch.float64])
def test_device_kmeanspp_random_matches_oracle(oracle, dtype):
    from paper_2603_09229_b200.core import kmeanspp_indices_device

    g = torch.Generator().manual_seed(11)
    for (B, n, d, k) in [(3, 2053, 32, 17), (1, 20000, 128, 24), (2, 129, 9, 129), (1, 3000, 256, 12),
                         (1, 2000, 192, 10)]:
        x = (torch.randn(B, n, d, generator=g) * 4).to(dtype)
        idx = kmeanspp_indices_device(x.cuda(), k, 5)
        x64 = x.double().numpy()
        ref = np.stack([oracle.kmeanspp_indices(x64[b], k, np.random.default_rng((5, b))) for b in range(B)])
        assert np.array_equal(idx, ref), (B, n, d, k)


def test_streamed_kmeanspp_matches_in_core(kpp_golden, tmp_path):
    import paper_2603_09229_b200 as fk
    from paper_2603_09229_b200.pipeline import HostStream, _init_from_stream

    for name in ("batched_f64", "f16_d64"):
        spec = CASES[name]
        x = case_tensor(spec)
        with HostStream(x, 1000) as s:
            c = _init_from_stream(s, spec["k"], spec["seed"], "kmeanspp", torch.device("cuda", 0))
        gold = kpp_golden[name]
        ref = torch.stack([x[b][torch.from_numpy(gold[b])] for b in range(x.shape[0])])
        assert torch.equal(c.cpu(), ref)
    # file-backed stream (FKM1), f32
    spec = CASES["duplicates_f32"]
    x = fk.DataMatrix(torch.from_numpy(make_case(spec)))
    p = str(tmp_path / "x.fkm1")
    fk.write_fkm1(p, x)
    with fk.ChunkStream(p, 37) as s:
        c = _init_from_stream(s, spec["k"], spec["seed"], "kmeanspp", torch.device("cuda", 0))
    gold = kpp_golden["duplicates_f32"]
    ref = torch.stack([x.data[b][torch.from_numpy(gold[b])] for b in range(2)])
    assert torch.equal(c.cpu(), ref)


def test_lloyd_run_with_kmeanspp_init(kpp_golden):
    import paper_2603_09229_b200 as fk

    spec = CASES["blobs_f32"]
    x = fk.DataMatrix(torch.from_numpy(make_case(spec)))
    c = fk.init_centroids(x, spec["k"], spec["seed"], "kmeanspp")
    gold = kpp_golden["blobs_f32"]
    assert torch.equal(c.data.cpu(), x.data[0][torch.from_numpy(gold[0])][None])
    res = fk.lloyd_run(x, fk.KMeansConfig(spec["k"], max_iters=5, seed=spec["seed"], init="kmeanspp"))
    assert res.iterations_run >= 1


def test_sharded_kmeanspp_device_world1(kpp_golden):
    """The sharded seeding's device path (NCCL, world 1): sweep into the table
    slice, all-gather, identical select -- index for index the golden draws."""
    import torch.distributed as dist

    from paper_2603_09229_b200.distributed import kmeanspp_indices_sharded

    dist.init_process_group("nccl", init_method="tcp://127.0.0.1:29631", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        for name in ("batched_f64", "bf16_d128", "duplicates_f32"):
            spec = CASES[name]
            x = case_tensor(spec).cuda()
            idx = kmeanspp_indices_sharded(x, x.shape[1], 0, spec["k"], spec["seed"])
            assert np.array_equal(idx, kpp_golden[name]), name
    finally:
        dist.destroy_process_group()


_TIE_SCRIPT = r"""
import sys, numpy as np, torch
sys.path.insert(0, %r); sys.path.insert(0, %r)
from fractions import Fraction
from oracle import oracle as O
from paper_2603_09229_b200 import ops

def crafted(seed, n):
    # a big first weight and tiny ones whose sum makes the pairwise total exactly 1:
    # the serial cumsum then adds exact half-ulps (ties to even), whole ulps and
    # 1.5 ulps, so numpy's chain depends on the parity of S/ulp at every step
    rng = np.random.default_rng(seed)
    tiny = rng.choice([2.0**-54, 2.0**-53, 3 * 2.0**-54, 0.0], size=n - 1)
    rest = sum(Fraction(float(t)) for t in tiny)
    if (rest / Fraction(2) ** -53).denominator != 1:  # keep 1 - rest a multiple of 2^-53
        tiny[-1] += 2.0**-54
        rest += Fraction(2) ** -54
    m0 = float(1 - rest)
    assert Fraction(m0) == 1 - rest
    m = np.concatenate([[m0], tiny]).astype(np.float64)
    perm = rng.permutation(n)          # the big weight anywhere
    return m[perm]

bad = 0
for seed in range(6):
    m = crafted(seed, 6000 + 977 * seed)
    total = O.pairwise_sum(m)
    pp = ops.KmeansppStream(m.size, 2, torch.device("cuda", 0))
    pp.m[0].copy_(torch.from_numpy(m))
    rng = np.random.default_rng(100 + seed)
    for u in np.concatenate([rng.random(12), [0.0, 0.5, 1 - 2**-53]]):
        pp.halted.fill_(2)
        pp.select(1, float(u))
        got = int(pp.idx[0, 1].item())
        ref = O.choice_cdf(m, total, float(u))
        bad += got != ref
print("mismatches", bad)
"""


@pytest.mark.parametrize("forced", [False, True])
def test_cumsum_ties_and_parity(forced):
    """choice() on crafted tables whose serial cumsum resolves exact half-ulp
    ties by parity: the certified path and the parallel exact walk (forced)
    both reproduce numpy's searchsorted index."""
    code = _TIE_SCRIPT % (ROOT, os.path.join(ROOT, "tests"))
    env = dict(os.environ)
    if forced:
        env["FK_PP_FORCE_EXACT"] = "1"
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    assert "mismatches 0" in r.stdout, r.stdout + r.stderr[-2000:]
