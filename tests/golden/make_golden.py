"""Generate golden vectors from the LIVE reference (flashmeans 0.1.0).

Run in the build container only (the reference is not present on the GPU box):

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every array written here is produced by calling the reference's own public API
(/root/reference/pkg/src/flashmeans, file:line cited per fixture).  Inputs are
regenerated deterministically by the tests from the stored seeds; a sha256 of
each input is stored so a numpy RNG drift is detected instead of silently
changing the fixture.  Files are small (< 1 MB total).
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
if REF not in sys.path:
    sys.path.insert(0, REF)
import flashmeans as fm  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def intgrid(rng, shape, lo=-8, hi=8, dtype=np.float32):
    return rng.integers(lo, hi + 1, shape).astype(dtype)


def main() -> None:
    meta: dict = {"reference": "flashmeans " + fm.__version__, "fixtures": {}}
    arrays: dict[str, np.ndarray] = {}

    # 1. flash_assign exact (flash_assign.py:135-222), f32 and f64, batched, ragged tiles.
    for prec in ("single", "double"):
        spec = dict(batch=2, points=333, k_true=7, dims=13, spread=0.9, seed=5, clusters=11, init_seed=6)
        x = fm.generate_dataset(spec["batch"], spec["points"], spec["k_true"], spec["dims"],
                                spec["spread"], spec["seed"], prec)
        c = fm.init_centroids(x, spec["clusters"], spec["init_seed"])
        a, m, _ = fm.flash_assign(x, c, fm.TilingConfig(32, 4, 100), fm.Counters())
        key = f"assign_{prec}"
        arrays[key + "_a"] = a.values
        arrays[key + "_m"] = m
        arrays[key + "_c"] = c.data
        meta["fixtures"][key] = dict(spec, precision=prec, x_sha=sha(x.data),
                                     source="flash_assign.py:135 (dot_mode=exact)")

    # 2. integer grid: every distance exact in fp32 -> bitwise KAT for bf16/fp16 inputs too.
    rng = np.random.default_rng(2603)
    for name, (n, k, d) in {"grid_small": (97, 13, 8), "grid_d128": (515, 300, 128),
                            "grid_d64": (260, 257, 64)}.items():
        xg = intgrid(rng, (1, n, d))
        cg = intgrid(rng, (1, k, d))
        a, m, _ = fm.flash_assign(fm.DataMatrix(xg), fm.Centroids(cg), fm.TilingConfig(64, 16, 64),
                                  fm.Counters())
        arrays[name + "_x"] = xg.astype(np.int8)
        arrays[name + "_c"] = cg.astype(np.int8)
        arrays[name + "_a"] = a.values
        arrays[name + "_m"] = m
        meta["fixtures"][name] = dict(n=n, k=k, d=d, source="flash_assign.py:135 integer grid")

    # 3. sort_inverse_update (sort_inverse.py:106-149) with merges counter, f32 + f64.
    for prec in ("single", "double"):
        x = fm.generate_dataset(2, 1000, 9, 6, 1.0, 7, prec)
        ids = np.random.default_rng(8).integers(0, 17, (2, 1000)).astype(np.int32)
        ids[1, :300] = 3  # a long run crossing chunk boundaries
        cnt = fm.Counters()
        st, _ = fm.sort_inverse_update(x, fm.Assignments(ids), 17, 128, cnt)
        key = f"update_{prec}"
        arrays[key + "_ids"] = ids
        arrays[key + "_sums"] = st.sums
        arrays[key + "_counts"] = st.counts
        prev = fm.init_centroids(x, 17, 9)
        nc, empty = fm.normalize(st, prev)
        arrays[key + "_prev"] = prev.data
        arrays[key + "_norm"] = nc.data
        meta["fixtures"][key] = dict(precision=prec, x_sha=sha(x.data), chunk=128, clusters=17,
                                     merges=cnt.synchronized_merges, empty=empty,
                                     source="sort_inverse.py:106, baseline.py:127")

    # 4. config 1 of BASELINE.json: N=10k, d=16, K=8 fp32, 20 Lloyd iterations, fixed init.
    x1 = fm.generate_dataset(1, 10000, 8, 16, 1.0, 0, "single")
    t1 = fm.TilingConfig(1024, 8, 10000)
    r = fm.lloyd_run(x1, fm.KMeansConfig(8, max_iters=20, seed=0, precision="single", tiling=t1))
    arrays["cfg1_centroids"] = r.centroids.data
    arrays["cfg1_assignments"] = r.assignments.values
    arrays["cfg1_history"] = r.objective_history
    c0 = fm.init_centroids(x1, 8, 0)
    arrays["cfg1_init"] = c0.data
    meta["fixtures"]["cfg1"] = dict(points=10000, dims=16, clusters=8, spread=1.0, seed=0,
                                    max_iters=20, update_chunk=10000, x_sha=sha(x1.data),
                                    iterations=r.iterations_run,
                                    merges=r.counters.synchronized_merges,
                                    source="pipeline.py:110 lloyd_run(engine=flash)")

    # 5. known-answer cases lifted from the reference's own tests.
    kat = {}
    x = fm.DataMatrix(np.array([[[1.0, 2.0]]]))
    c = fm.Centroids(np.array([[[0.0, 0.0], [2.0, 0.0]]]))
    a, m, _ = fm.flash_assign(x, c, fm.TilingConfig(1, 1, 1), fm.Counters())
    kat["tie_lowest_id"] = dict(x=x.data.tolist(), c=c.data.tolist(), a=int(a.values[0, 0]),
                                m=float(m[0, 0]), source="tests/test_flash_assign.py:131-135")
    idx, a_sorted = fm.argsort_assignments(fm.Assignments(np.array([[2, 0, 1, 0]], np.int32)), 3)
    kat["argsort_hand"] = dict(ids=[2, 0, 1, 0], order=idx.order[0].tolist(),
                               a_sorted=a_sorted[0].tolist(), source="tests/test_sort_inverse.py:26-29")
    idx, _ = fm.argsort_assignments(fm.Assignments(np.array([[1, 1, 0, 1, 0]], np.int32)), 2)
    kat["argsort_stable"] = dict(ids=[1, 1, 0, 1, 0], order=idx.order[0].tolist(),
                                 source="tests/test_sort_inverse.py:40-42")
    xs = fm.DataMatrix(np.array([[[2.0, 0.0], [1.0, 0.0], [4.0, 0.0], [3.0, 0.0]]]))
    st = fm.scatter_update(xs, fm.Assignments(np.array([[0, 1, 0, 1]], np.int32)), 2, fm.Counters())
    kat["scatter_hand"] = dict(x=xs.data.tolist(), ids=[0, 1, 0, 1], sums=st.sums.tolist(),
                               counts=st.counts.tolist(), source="tests/test_baseline.py:136-142")
    two = fm.DataMatrix(np.array([[[0.0], [0.1], [10.0], [10.1]]]))
    r2 = fm.lloyd_run(two, fm.KMeansConfig(2, seed=0, max_iters=50))
    kat["two_blobs"] = dict(x=two.data.tolist(), centroids=sorted(r2.centroids.data[0, :, 0].tolist()),
                            objective=float(r2.objective_history[-1, 0]),
                            source="tests/test_pipeline.py:53-59")
    kat["row_norms"] = dict(x=[[3.0, 4.0]], out=fm.row_norms(np.array([[3.0, 4.0]])).tolist(),
                            source="tests/test_core.py:61-64")
    cnt = fm.Counters()
    xs5 = fm.DataMatrix(np.zeros((1, 5, 1)))
    fm.sort_inverse_update(xs5, fm.Assignments(np.array([[0, 0, 1, 2, 2]], np.int32)), 3, 2, cnt)
    kat["merge_count"] = dict(ids=[0, 0, 1, 2, 2], chunk=2, merges=cnt.synchronized_merges,
                              source="tests/test_sort_inverse.py:98-106")
    meta["kat"] = kat

    np.savez_compressed(os.path.join(OUT, "golden.npz"), **arrays)
    with open(os.path.join(OUT, "golden.json"), "w") as f:
        json.dump(meta, f, indent=1, sort_keys=True)
    print("wrote", len(arrays), "arrays")


if __name__ == "__main__":
    main()
