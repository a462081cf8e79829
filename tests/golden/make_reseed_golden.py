"""Golden runs of the reference's reseed_farthest policy (pipeline.py:76-89,
283-309): in-core lloyd_run and the FKM1 streaming run on data with duplicate
rows, so identical initial centroids leave clusters empty.

Run in the build container:  python tests/golden/make_reseed_golden.py
"""
import os
import sys
import tempfile

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
import flashmeans as fm  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
base = fm.generate_dataset(2, 300, 6, 5, 1.0, 21, "single").data
x = np.ascontiguousarray(np.concatenate([base, base[:, :200]], axis=1))  # 200 duplicated rows
X = fm.DataMatrix(x)
cfg = fm.KMeansConfig(48, max_iters=25, seed=5, empty_cluster_policy="reseed_farthest")
r = fm.lloyd_run(X, cfg)
# count the empties the run hit (re-run the first normalize)
c0 = fm.init_centroids(X, 48, 5)
a, m, _ = fm.flash_assign(X, c0, fm.TilingConfig(64, 16, 500), fm.Counters())
st, _ = fm.sort_inverse_update(X, a, 48, 500, fm.Counters())
_, empties = fm.normalize(st, c0)
assert sum(len(e) for e in empties) > 0, "no empty clusters: pick another seed"
with tempfile.TemporaryDirectory() as d:
    p = os.path.join(d, "x.fkm1")
    fm.write_fkm1(p, X)
    with fm.ChunkStream(p, 77) as s:
        rs = fm.chunked_stream_run(s, cfg)
assert np.array_equal(rs.centroids.data, r.centroids.data)
np.savez(os.path.join(HERE, "reseed_golden.npz"), x=x, centroids=r.centroids.data,
         assignments=r.assignments.values, history=r.objective_history,
         iterations=np.int64(r.iterations_run), first_empties=np.int64(sum(len(e) for e in empties)))
print("iterations", r.iterations_run, "first-pass empties", [len(e) for e in empties])
