"""Deterministic inputs of the k-means++ golden cases (tests/golden/kmeanspp_golden.*).

The data a case describes is what the reference seeds on: float32/float64
arrays, or -- for the bf16/fp16 cases -- the exact float32 upcast of the
rounded tensor (the reference rejects 16-bit data, core.py:100-101, so the
oracle sees the upcast of the very values the device kernel reads).
"""

from __future__ import annotations

import numpy as np
import torch

CASES = {
    # config-1 shape: Gaussian blobs, f32
    "blobs_f32": dict(kind="blobs", dtype="float32", B=1, N=10000, d=16, k=8, seed=0, spread=1.0),
    # batched f64, odd d (scalar tail), several dozen draws
    "batched_f64": dict(kind="normal", dtype="float64", B=2, N=1500, d=7, k=40, seed=4),
    # d > 128: numpy's recursive split inside the row sum
    "wide_f64": dict(kind="normal", dtype="float64", B=1, N=700, d=200, k=25, seed=9),
    # bf16 data (exact f32 upcast), the tensor-core path's element type
    "bf16_d128": dict(kind="blobs", dtype="bfloat16", B=1, N=4099, d=128, k=64, seed=2, spread=1.0),
    # fp16, d=64, several nodes in the pairwise tree (N > 4096)
    "f16_d64": dict(kind="normal", dtype="float16", B=1, N=9001, d=64, k=30, seed=5),
    # duplicated rows: the table sums to 0 before K draws -> rng.integers fallback
    "duplicates_f32": dict(kind="dups", dtype="float32", B=2, N=240, d=5, k=60, seed=6, distinct=37),
    # K == N, tiny d
    "k_eq_n_f64": dict(kind="normal", dtype="float64", B=1, N=50, d=1, k=50, seed=8),
    # large tree: several tiers of the pairwise sum, d=3 (unaligned rows)
    "large_f32": dict(kind="normal", dtype="float32", B=1, N=300007, d=3, k=12, seed=10),
}


def make_case(spec: dict) -> np.ndarray:
    """(B, N, d) float32/float64 numpy array the reference seeds on."""
    rng = np.random.default_rng(spec["seed"] + 1000)
    B, N, d = spec["B"], spec["N"], spec["d"]
    if spec["kind"] == "blobs":
        k_true = max(spec["k"], 4)
        out = np.empty((B, N, d), np.float64)
        for b in range(B):
            centers = rng.uniform(-10.0, 10.0, size=(k_true, d))
            labels = rng.integers(0, k_true, size=N)
            out[b] = centers[labels] + rng.standard_normal((N, d)) * spec.get("spread", 1.0)
    elif spec["kind"] == "dups":
        out = np.empty((B, N, d), np.float64)
        for b in range(B):
            base = rng.standard_normal((spec["distinct"], d)) * 3.0
            out[b] = base[rng.integers(0, spec["distinct"], size=N)]
    else:
        out = rng.standard_normal((B, N, d)) * rng.uniform(0.5, 20.0)
    dt = spec["dtype"]
    if dt in ("bfloat16", "float16"):
        t = torch.from_numpy(out.astype(np.float32)).to(getattr(torch, dt))
        return t.float().numpy()
    return np.ascontiguousarray(out.astype(dt))


def case_tensor(spec: dict) -> torch.Tensor:
    """The same data as a torch tensor in the case's element type."""
    x = make_case(spec)
    t = torch.from_numpy(x)
    if spec["dtype"] in ("bfloat16", "float16"):
        t = t.to(getattr(torch, spec["dtype"]))
    return t
