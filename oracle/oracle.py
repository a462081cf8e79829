"""CPU parity oracle for the flashmeans hot path (TEST INFRASTRUCTURE ONLY).

This module is the checker, never the thing measured or shipped.  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import it.  The product package
``paper_2603_09229_b200`` never imports anything from ``oracle/``.

It restates the reference package flashmeans 0.1.0 (read-only at
/root/reference/pkg/src/flashmeans, citations relative to that directory):

* the compiled arithmetic lives in ``fk_oracle.c`` (see its header for the
  per-function file:line map) and is loaded through ctypes;
* the Python-level drivers below restate ``lloyd_run`` (pipeline.py:110-147),
  ``init_centroids`` (core.py:360-381), ``generate_dataset`` (core.py:384-410),
  ``_objective_row`` (pipeline.py:65-68) and ``_max_shift`` (pipeline.py:71-73)
  on top of numpy, which is the reference's own third-party dependency for RNG
  and reductions (numpy>=1.24, pyproject.toml:11-14; 2.3.5 in this image).

Parity is pinned two ways (tests/test_oracle_golden.py,
tests/test_oracle_reference.py): against golden vectors produced by the live
reference (tests/golden/make_golden.py) and, when /root/reference exists,
against the reference itself on randomized instances.
"""

from __future__ import annotations

import ctypes
import os
import subprocess
import sys

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "_build", "libfk_oracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile fk_oracle.c with gcc (-O2 -fopenmp -ffp-contract=off)."""
    src = os.path.join(_HERE, "fk_oracle.c")
    if not force and os.path.exists(_LIB_PATH) and os.path.getmtime(_LIB_PATH) >= os.path.getmtime(src):
        return _LIB_PATH
    os.makedirs(os.path.dirname(_LIB_PATH), exist_ok=True)
    cmd = ["gcc", "-O2", "-fPIC", "-shared", "-fopenmp", "-ffp-contract=off",
           "-fno-fast-math", "-o", _LIB_PATH, src, "-lm"]
    subprocess.run(cmd, check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        build()
        L = ctypes.CDLL(_LIB_PATH)
        P = ctypes.c_void_p
        I64 = ctypes.c_int64
        L.orc_max_threads.restype = ctypes.c_int
        for name in ("orc_row_norms_f32", "orc_row_norms_f64"):
            getattr(L, name).argtypes = [P, I64, I64, P]
        for name in ("orc_assign_f32", "orc_assign_f64"):
            getattr(L, name).argtypes = [P, P, I64, I64, I64, P, P, ctypes.c_int]
        L.orc_counting_sort.argtypes = [P, I64, I64, P, P]
        for name in ("orc_sort_inverse_f32", "orc_sort_inverse_f64"):
            getattr(L, name).argtypes = [P, P, I64, I64, I64, I64, P, P]
            getattr(L, name).restype = I64
        for name in ("orc_scatter_f32", "orc_scatter_f64"):
            getattr(L, name).argtypes = [P, P, I64, I64, P, P]
        for name in ("orc_normalize_f32", "orc_normalize_f64"):
            getattr(L, name).argtypes = [P, P, P, I64, I64, P, P]
        L.orc_pairwise_sum.argtypes = [P, I64]
        L.orc_pairwise_sum.restype = ctypes.c_double
        L.orc_kmeanspp_sweep.argtypes = [P, I64, I64, P, P, ctypes.c_int]
        L.orc_choice_cdf.argtypes = [P, I64, ctypes.c_double, ctypes.c_double]
        L.orc_choice_cdf.restype = I64
        _lib = L
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _sfx(dt) -> str:
    dt = np.dtype(dt)
    if dt == np.float32:
        return "f32"
    if dt == np.float64:
        return "f64"
    raise ValueError(f"oracle supports float32/float64 data, got {dt}")


def max_threads() -> int:
    return int(lib().orc_max_threads())


# ----------------------------------------------------------------- kernels
def row_norms(m: np.ndarray) -> np.ndarray:
    """core.row_norms (core.py:307-318)."""
    m = np.ascontiguousarray(m)
    out = np.empty(m.shape[0], m.dtype)
    getattr(lib(), "orc_row_norms_" + _sfx(m.dtype))(_p(m), m.shape[0], m.shape[1], _p(out))
    return out


def assign(x: np.ndarray, c: np.ndarray, threads: int = 0):
    """flash_assign(dot_mode="exact") on (B,N,d)/(B,K,d): returns (a int32, m dtype)."""
    x = np.ascontiguousarray(x)
    c = np.ascontiguousarray(c)
    if x.dtype != c.dtype:
        raise ValueError("data and centroids must share one precision")
    B, N, d = x.shape
    K = c.shape[1]
    a = np.empty((B, N), np.int32)
    m = np.empty((B, N), x.dtype)
    f = getattr(lib(), "orc_assign_" + _sfx(x.dtype))
    for b in range(B):
        xb, cb = x[b], c[b]
        ab, mb = a[b], m[b]
        f(_p(xb), _p(cb), N, K, d, _p(ab), _p(mb), int(threads))
    return a, m


def counting_sort(ids: np.ndarray, k: int):
    """_kernels.counting_sort (stable): returns (order int64, a_sorted int32)."""
    ids = np.ascontiguousarray(ids, np.int32)
    order = np.empty(ids.shape[0], np.int64)
    a_sorted = np.empty(ids.shape[0], np.int32)
    lib().orc_counting_sort(_p(ids), ids.shape[0], k, _p(order), _p(a_sorted))
    return order, a_sorted


def sort_inverse_update(x: np.ndarray, a: np.ndarray, clusters: int, chunk: int):
    """sort_inverse_update: returns (sums f64 (B,K,d), counts i64 (B,K), merges)."""
    x = np.ascontiguousarray(x)
    a = np.ascontiguousarray(a, np.int32)
    B, N, d = x.shape
    sums = np.zeros((B, clusters, d), np.float64)
    counts = np.zeros((B, clusters), np.int64)
    f = getattr(lib(), "orc_sort_inverse_" + _sfx(x.dtype))
    merges = 0
    ch = max(1, min(int(chunk), N))
    for b in range(B):
        xb, ab, sb, cb = x[b], a[b], sums[b], counts[b]
        merges += int(f(_p(xb), _p(ab), N, clusters, d, ch, _p(sb), _p(cb)))
    return sums, counts, merges


def scatter_update(x: np.ndarray, a: np.ndarray, clusters: int):
    x = np.ascontiguousarray(x)
    a = np.ascontiguousarray(a, np.int32)
    B, N, d = x.shape
    sums = np.zeros((B, clusters, d), np.float64)
    counts = np.zeros((B, clusters), np.int64)
    f = getattr(lib(), "orc_scatter_" + _sfx(x.dtype))
    for b in range(B):
        xb, ab, sb, cb = x[b], a[b], sums[b], counts[b]
        f(_p(xb), _p(ab), N, d, _p(sb), _p(cb))
    return sums, counts


def normalize(sums: np.ndarray, counts: np.ndarray, prev: np.ndarray):
    """baseline.normalize(policy="keep"): returns (centroids, empty id lists)."""
    sums = np.ascontiguousarray(sums, np.float64)
    counts = np.ascontiguousarray(counts, np.int64)
    prev = np.ascontiguousarray(prev)
    B, K, d = prev.shape
    out = np.empty_like(prev)
    empty = np.zeros((B, K), np.uint8)
    f = getattr(lib(), "orc_normalize_" + _sfx(prev.dtype))
    for b in range(B):
        sb, cb, pb, ob, eb = sums[b], counts[b], prev[b], out[b], empty[b]
        f(_p(sb), _p(cb), _p(pb), K, d, _p(ob), _p(eb))
    return out, [[int(k) for k in np.flatnonzero(empty[b])] for b in range(B)]


# ----------------------------------------------------------------- drivers
def generate_dataset(batch, points, k_true, dims, spread, seed, dtype=np.float64) -> np.ndarray:
    """core.generate_dataset (core.py:384-410), numpy PCG64 substreams (seed, b)."""
    out = np.empty((batch, points, dims), np.float64)
    for b in range(batch):
        rng = np.random.default_rng((seed, b))
        centers = rng.uniform(-10.0, 10.0, size=(k_true, dims))
        labels = rng.integers(0, k_true, size=points)
        pts = centers[labels]
        if spread > 0.0:
            pts = pts + rng.standard_normal((points, dims)) * spread
        out[b] = pts
    return np.ascontiguousarray(out.astype(dtype))


def init_indices(points: int, clusters: int, seed: int, batch: int) -> np.ndarray:
    """random_distinct row choice of init_centroids (core.py:375-377)."""
    idx = np.empty((batch, clusters), np.int64)
    for b in range(batch):
        rng = np.random.default_rng((seed, b))
        idx[b] = rng.choice(points, size=clusters, replace=False)
    return idx


def pairwise_sum(a: np.ndarray) -> float:
    """numpy's pairwise summation of a 1-D f64 array (min_d2.sum())."""
    a = np.ascontiguousarray(a, np.float64)
    return float(lib().orc_pairwise_sum(_p(a), a.shape[0]))


def kmeanspp_sweep(points64: np.ndarray, center64: np.ndarray, m: np.ndarray, first: bool) -> None:
    """One D^2 sweep in numpy order into m (in place)."""
    p = np.ascontiguousarray(points64, np.float64)
    c = np.ascontiguousarray(center64, np.float64)
    lib().orc_kmeanspp_sweep(_p(p), p.shape[0], p.shape[1], _p(c), _p(m), 1 if first else 0)


def choice_cdf(m: np.ndarray, total: float, u: float) -> int:
    """searchsorted(cumsum(m/total)/cumsum[-1], u, side="right")."""
    m = np.ascontiguousarray(m, np.float64)
    return int(lib().orc_choice_cdf(_p(m), m.shape[0], float(total), float(u)))


def kmeanspp_indices(points: np.ndarray, k: int, rng: np.random.Generator) -> np.ndarray:
    """_kmeanspp_indices (core.py:342-357) with the numpy arithmetic in C.

    The generator is consumed exactly like the reference: one integers(n)
    for the first index, then per draw one random() (inside choice) when the
    total is positive, else integers(n)."""
    p64 = np.ascontiguousarray(points, np.float64)
    n, d = p64.shape
    L = lib()
    idx = np.empty(k, np.int64)
    idx[0] = rng.integers(n)
    m = np.empty(n, np.float64)
    c = np.ascontiguousarray(p64[idx[0]])
    L.orc_kmeanspp_sweep(_p(p64), n, d, _p(c), _p(m), 1)
    for j in range(1, k):
        total = float(L.orc_pairwise_sum(_p(m), n))
        if total > 0.0:
            choice = int(L.orc_choice_cdf(_p(m), n, total, float(rng.random())))
        else:
            choice = int(rng.integers(n))
        idx[j] = choice
        c = np.ascontiguousarray(p64[choice])
        L.orc_kmeanspp_sweep(_p(p64), n, d, _p(c), _p(m), 0)
    return idx


def kmeanspp_init_indices(x: np.ndarray, clusters: int, seed: int) -> np.ndarray:
    """init_centroids(method="kmeanspp") row choice per batch (core.py:373-379)."""
    out = np.empty((x.shape[0], clusters), np.int64)
    for b in range(x.shape[0]):
        out[b] = kmeanspp_indices(x[b], clusters, np.random.default_rng((seed, b)))
    return out


def init_centroids(x: np.ndarray, clusters: int, seed: int) -> np.ndarray:
    idx = init_indices(x.shape[1], clusters, seed, x.shape[0])
    return np.ascontiguousarray(np.stack([x[b][idx[b]] for b in range(x.shape[0])]))


def objective_row(m: np.ndarray) -> np.ndarray:
    """pipeline._objective_row: np.sum(m[b], dtype=float64) per batch."""
    return np.array([np.sum(m[b], dtype=np.float64) for b in range(m.shape[0])], np.float64)


def max_shift(old: np.ndarray, new: np.ndarray) -> float:
    """pipeline._max_shift."""
    diff = new.astype(np.float64) - old.astype(np.float64)
    return float(np.sqrt(np.square(diff).sum(axis=2).max()))


def lloyd_run(x: np.ndarray, clusters: int, max_iters: int = 50, shift_tol: float = 0.0,
              seed: int = 0, chunk: int | None = None, c0: np.ndarray | None = None,
              threads: int = 0):
    """lloyd_run(engine="flash", policy="keep") restated (pipeline.py:110-147).

    Returns (centroids, assignments, history (iters,B), iterations, merges)."""
    B, N, d = x.shape
    c = init_centroids(x, clusters, seed) if c0 is None else np.ascontiguousarray(c0)
    ch = N if chunk is None else chunk
    history = []
    prev = None
    a = None
    it_run = 0
    merges = 0
    for it in range(1, max_iters + 1):
        it_run = it
        a, m = assign(x, c, threads)
        history.append(objective_row(m))
        if prev is not None and np.array_equal(prev, a):
            break
        sums, counts, mg = sort_inverse_update(x, a, clusters, ch)
        merges += mg
        new_c, _ = normalize(sums, counts, c)
        shift = max_shift(c, new_c)
        prev, c = a, new_c
        if shift <= shift_tol:
            break
    return c, a, np.array(history), it_run, merges


if __name__ == "__main__":  # pragma: no cover - manual build hook
    print(build(force="--force" in sys.argv))
