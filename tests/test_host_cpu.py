"""Host-side logic of the drop-in package (CPU; mirrors the reference's unit tests).

Types, validation (same ValueError contract as flashmeans), the tiling
heuristic, segment detection, seeded initialization and dataset generation
(bitwise equal to the reference / oracle).
"""

import numpy as np
import pytest
import torch

import paper_2603_09229_b200 as fk


class TestTypes:
    def test_datamatrix_validation(self):
        with pytest.raises(ValueError):
            fk.DataMatrix(np.zeros((2, 3)))
        with pytest.raises(ValueError):
            fk.DataMatrix(np.zeros((1, 0, 3)))
        with pytest.raises(ValueError):
            fk.DataMatrix(np.zeros((1, 2, 3), np.int32))
        with pytest.raises(ValueError):
            fk.DataMatrix(np.full((1, 2, 3), np.nan))
        with pytest.raises(ValueError):
            fk.DataMatrix(torch.zeros((1, 4, 3)).transpose(1, 2))
        x = fk.DataMatrix(np.zeros((2, 5, 3), np.float32))
        assert (x.batch, x.points, x.dims, x.precision, x.elem_bytes) == (2, 5, 3, "single", 4)
        xb = fk.DataMatrix(torch.zeros((1, 4, 8), dtype=torch.bfloat16))
        assert xb.precision == "bf16" and xb.elem_bytes == 2

    def test_from_array(self):
        assert fk.DataMatrix.from_array([[[1, 2]]]).precision == "double"
        assert fk.DataMatrix.from_array(np.ones((1, 2, 2)), precision="bf16").data.dtype == torch.bfloat16

    def test_assignments_validation(self):
        with pytest.raises(ValueError):
            fk.Assignments(np.zeros((1, 3), np.int64))
        with pytest.raises(ValueError):
            fk.Assignments(np.array([[0, -1]], np.int32))
        with pytest.raises(ValueError):
            fk.Assignments(np.zeros(3, np.int32))
        assert fk.Assignments(np.array([[0, 2]], np.int32)).points == 2

    def test_cluster_stats(self):
        st = fk.ClusterStats.zeros(2, 3, 4)
        assert st.sums.dtype == torch.float64 and st.counts.dtype == torch.int64
        with pytest.raises(ValueError):
            fk.ClusterStats(torch.zeros((1, 2, 3)), torch.zeros((1, 2), dtype=torch.int64))
        with pytest.raises(ValueError):
            fk.ClusterStats(torch.zeros((1, 2, 3), dtype=torch.float64), torch.zeros((1, 3), dtype=torch.int64))

    def test_counters(self):
        c = fk.Counters()
        c.synchronized_merges = 5
        c.reset()
        assert c.as_dict() == {"intermediate_bytes_written": 0, "intermediate_bytes_read": 0,
                               "synchronized_merges": 0, "elements_streamed": 0}

    def test_config_validation(self):
        for bad in (dict(clusters=0), dict(clusters=2, max_iters=0), dict(clusters=2, shift_tol=-1.0),
                    dict(clusters=2, init="x"), dict(clusters=2, empty_cluster_policy="x"),
                    dict(clusters=2, precision="half")):
            with pytest.raises(ValueError):
                fk.KMeansConfig(**bad)
        assert fk.KMeansConfig(3, precision="bf16").precision == "bf16"

    def test_distances(self):
        assert fk.squared_distance((1, 2), (3, 4)) == 8.0
        assert fk.expanded_distance(5.0, 25.0, 11.0) == 8.0
        assert fk.expanded_distance(1.0, 1.0, 1.0000001) == 0.0

    def test_tiling(self):
        t = fk.TilingConfig(64, 64, 4096).clamped(points=33, clusters=7)
        assert (t.point_tile, t.centroid_tile, t.update_chunk) == (33, 7, 33)
        assert fk.TilingConfig(64, 16, 1).working_set_bytes(8, 4) == (64 * 8 + 16 * 8 + 64 * 16) * 4
        with pytest.raises(ValueError):
            fk.TilingConfig(0, 1, 1)

    def test_worker_count(self, monkeypatch):
        monkeypatch.setenv("FLASHMEANS_WORKERS", "3")
        assert fk.worker_count() == 3
        monkeypatch.setenv("FLASHMEANS_WORKERS", "x")
        with pytest.raises(ValueError):
            fk.worker_count()


class TestSegments:
    def test_detect(self):
        S = fk.Segment
        assert fk.detect_segments(np.array([0, 0, 1, 2, 2])) == [S(0, 2, 0), S(2, 3, 1), S(3, 5, 2)]
        assert fk.detect_segments(np.array([0, 0, 0, 1, 1]), chunk=2) == [
            S(0, 2, 0), S(2, 3, 0), S(3, 4, 1), S(4, 5, 1)]
        with pytest.raises(ValueError):
            fk.detect_segments(np.array([1, 0]))

    def test_argsort_validates_before_the_device(self):
        # the hand cases ([2,0,1,0] -> [1,3,2,0], stability) run on the device sort:
        # tests/test_gpu_kernels.py::test_device_argsort_*
        with pytest.raises(ValueError):
            fk.argsort_assignments(fk.Assignments(np.array([[0, 3]], np.int32)), 3)


class TestTuner:
    def test_heuristic_matches_golden_shapes(self):
        t = fk.heuristic_config(fk.ProblemShape(2000, 8, 16, 1), fk.CacheModel(elem_bytes=8, workers=8))
        assert (t.point_tile, t.centroid_tile, t.update_chunk) == (128, 8, 256)

    def test_heuristic_matches_reference(self, reference):
        rng = np.random.default_rng(0)
        for _ in range(50):
            shp = dict(points=int(rng.integers(1, 1 << 24)), clusters=int(rng.integers(1, 70000)),
                       dims=int(rng.integers(1, 600)), batch=int(rng.integers(1, 8)))
            cm = dict(elem_bytes=int(rng.choice([4, 8])), workers=int(rng.integers(1, 200)))
            ours = fk.heuristic_config(fk.ProblemShape(**shp), fk.CacheModel(**cm))
            ref = reference.heuristic_config(reference.ProblemShape(**shp), reference.CacheModel(**cm))
            assert (ours.point_tile, ours.centroid_tile, ours.update_chunk) == (
                ref.point_tile, ref.centroid_tile, ref.update_chunk)

    def test_candidates_match_reference(self, reference):
        shp = dict(points=3000, clusters=100, dims=16)
        ours = fk.enumerate_candidates(fk.ProblemShape(**shp))
        ref = reference.enumerate_candidates(reference.ProblemShape(**shp))
        assert [(c.point_tile, c.centroid_tile, c.update_chunk) for c in ours] == [
            (c.point_tile, c.centroid_tile, c.update_chunk) for c in ref]

    def test_shape_bucket(self):
        b = fk.shape_bucket(fk.ProblemShape(1 << 23, 4096, 128), torch.bfloat16)
        assert b["assign"]["kernel"].startswith("fk_assign_tc2") and b["assign"]["k_atoms"] == 2
        b256 = fk.shape_bucket(fk.ProblemShape(1 << 20, 1024, 256), torch.bfloat16)
        assert b256["assign"]["k_atoms"] == 4 and b256["assign"]["c_stages"] == 4
        assert fk.shape_bucket(fk.ProblemShape(100, 8, 16), torch.float32)["assign"]["kernel"].endswith("<exact>")
        assert fk.shape_bucket(fk.ProblemShape(100, 8, 264), torch.float16)["assign"]["kernel"].endswith("<lowp>")
        assert fk.shape_bucket(fk.ProblemShape(100, 8, 201), torch.float16)["assign"]["kernel"].endswith("<lowp>")


class TestInit:
    @pytest.mark.parametrize("prec,dt", [("single", np.float32), ("double", np.float64)])
    def test_generate_and_init_match_oracle(self, oracle, prec, dt):
        x = fk.generate_dataset(3, 257, 5, 7, 0.7, 11, prec)
        xo = oracle.generate_dataset(3, 257, 5, 7, 0.7, 11, dt)
        assert np.array_equal(x.numpy(), xo)
        c = fk.init_centroids(x, 9, 4)
        assert np.array_equal(c.numpy(), oracle.init_centroids(xo, 9, 4))

    def test_init_validation(self):
        x = fk.generate_dataset(1, 5, 2, 2, 0.5, 0)
        with pytest.raises(ValueError):
            fk.init_centroids(x, 6, 0)
        with pytest.raises(ValueError):
            fk.init_centroids(x, 2, 0, "bogus")

    def test_bf16_dataset_is_rounded_f32_draw(self, oracle):
        x = fk.generate_dataset(1, 50, 3, 8, 1.0, 2, "bf16")
        xo = oracle.generate_dataset(1, 50, 3, 8, 1.0, 2, np.float32)
        assert torch.equal(x.data, torch.from_numpy(xo).to(torch.bfloat16))


def test_partial_stats_combine():
    a = fk.PartialStats(1, torch.ones((2, 3), dtype=torch.float64), torch.ones(2, dtype=torch.int64))
    b = fk.PartialStats(0, torch.ones((2, 3), dtype=torch.float64), torch.ones(2, dtype=torch.int64))
    c = a.combine(b)
    assert c.chunk_index == 0 and float(c.sums.sum()) == 12.0 and c.counts.tolist() == [2, 2]
