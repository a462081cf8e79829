"""FKM1/FKA1 codec, AssignmentStore and the file-backed ChunkStream (CPU).

Pinned byte-for-byte against files written by the live reference
(tests/golden/make_fileio_golden.py); mirrors the reference's fileio tests
(validation errors, sentinel/changed semantics, atomic finalize/abort) and
its streaming-reader tests (bounds, short reads, dtype checks).
"""

import os

import numpy as np
import pytest
import torch

import paper_2603_09229_b200 as fk
from paper_2603_09229_b200 import fileio
from paper_2603_09229_b200.pipeline import _init_from_stream
from paper_2603_09229_b200.core import init_indices

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")


def _expected():
    return np.load(os.path.join(GOLD, "fileio_expected.npz"))


def test_reads_reference_written_files():
    e = _expected()
    x = fk.read_fkm1(os.path.join(GOLD, "ref_small_f32.fkm1"))
    assert x.data.dtype == torch.float32 and np.array_equal(x.data.numpy(), e["x32"])
    x = fk.read_fkm1(os.path.join(GOLD, "ref_small_f64.fkm1"))
    assert x.data.dtype == torch.float64 and np.array_equal(x.data.numpy(), e["x64"])
    a = fk.read_fka1(os.path.join(GOLD, "ref_small.fka1"))
    assert np.array_equal(a.values.numpy(), e["a"])
    h = fk.read_fkm1_header(os.path.join(GOLD, "ref_small_f32.fkm1"))
    assert (h.batch, h.points, h.dims, h.precision, h.elem_bytes) == (2, 5, 3, "single", 4)
    assert fk.read_fka1_header(os.path.join(GOLD, "ref_small.fka1")) == (2, 5)


def test_writes_byte_identical_files(tmp_path):
    e = _expected()
    for name, arr in (("ref_small_f32.fkm1", e["x32"]), ("ref_small_f64.fkm1", e["x64"])):
        p = tmp_path / name
        fk.write_fkm1(str(p), fk.DataMatrix(torch.from_numpy(arr)))
        assert p.read_bytes() == open(os.path.join(GOLD, name), "rb").read()
    p = tmp_path / "a.fka1"
    fk.write_fka1(str(p), fk.Assignments(torch.from_numpy(e["a"])))
    assert p.read_bytes() == open(os.path.join(GOLD, "ref_small.fka1"), "rb").read()
    st = fk.AssignmentStore(str(tmp_path / "s.fka1"), 2, 5)
    assert st.write_chunk(0, 1, np.array([4, 4], np.int32))
    assert st.write_chunk(1, 3, torch.tensor([1, 2], dtype=torch.int32))
    st.finalize()
    assert (tmp_path / "s.fka1").read_bytes() == open(os.path.join(GOLD, "ref_store.fka1"), "rb").read()


@pytest.mark.parametrize("dtype", [torch.float32, torch.float64, torch.bfloat16, torch.float16])
def test_fkm1_round_trip(tmp_path, dtype):
    x = torch.randn(3, 17, 5).to(dtype)
    p = str(tmp_path / "x.fkm1")
    fk.write_fkm1(p, fk.DataMatrix(x))
    assert os.path.getsize(p) == 32 + x.numel() * x.element_size()
    y = fk.read_fkm1(p)
    assert y.data.dtype == dtype and torch.equal(y.data, x)
    assert not [f for f in os.listdir(tmp_path) if ".tmp." in f]  # temp file renamed away


def _patch(path, off, data):
    with open(path, "r+b") as f:
        f.seek(off)
        f.write(data)


def test_fkm1_validation(tmp_path):
    p = str(tmp_path / "x.fkm1")
    fk.write_fkm1(p, fk.DataMatrix(torch.zeros(1, 4, 2)))
    good = open(p, "rb").read()
    cases = [(0, b"XKM1", "bad magic"), (4, b"\x02\x00", "version"), (6, b"\x09", "dtype code"),
             (7, b"\x01", "reserved"), (8, (0).to_bytes(8, "little"), "positive")]
    for off, data, msg in cases:
        open(p, "wb").write(good)
        _patch(p, off, data)
        with pytest.raises(fk.DataFormatError, match=msg):
            fk.read_fkm1_header(p)
    open(p, "wb").write(good[:-1])
    with pytest.raises(fk.DataFormatError, match="size mismatch"):
        fk.read_fkm1(p)
    open(p, "wb").write(good[:10])
    with pytest.raises(fk.DataFormatError, match="truncated"):
        fk.read_fkm1_header(p)
    open(p, "wb").write(good)
    _patch(p, 32, np.array([np.nan], np.float32).tobytes())
    with pytest.raises(fk.DataFormatError, match="payload invalid"):
        fk.read_fkm1(p)


def test_fka1_validation(tmp_path):
    p = str(tmp_path / "a.fka1")
    fk.write_fka1(p, fk.Assignments(torch.zeros((1, 3), dtype=torch.int32)))
    good = open(p, "rb").read()
    for off, data, msg in [(0, b"FKAX", "bad magic"), (4, (2).to_bytes(4, "little"), "version"),
                           (8, (1).to_bytes(8, "little"), "reserved")]:
        open(p, "wb").write(good)
        _patch(p, off, data)
        with pytest.raises(fk.DataFormatError, match=msg):
            fk.read_fka1(p)
    open(p, "wb").write(good + b"\0\0\0\0")
    with pytest.raises(fk.DataFormatError, match="size mismatch"):
        fk.read_fka1(p)
    open(p, "wb").write(good)
    _patch(p, 32, (0x80000000).to_bytes(4, "little"))
    with pytest.raises(fk.DataFormatError, match="range"):
        fk.read_fka1(p)


def test_assignment_store_semantics(tmp_path):
    path = str(tmp_path / "s.fka1")
    st = fk.AssignmentStore(path, 2, 6)
    assert not os.path.exists(path)  # only the working file exists until finalize
    assert st.write_chunk(0, 0, np.zeros(3, np.int32))       # sentinel -> changed
    assert not st.write_chunk(0, 0, np.zeros(3, np.int32))   # same ids -> unchanged
    assert st.write_chunk(0, 1, np.array([0, 5], np.int32))
    with pytest.raises(ValueError):
        st.write_chunk(0, 5, np.zeros(2, np.int32))
    with pytest.raises(ValueError):
        st.write_chunk(2, 0, np.zeros(1, np.int32))
    st.write_chunk(0, 3, np.ones(3, np.int32))
    st.write_chunk(1, 0, np.arange(6, dtype=np.int32))
    assert st.read_all().values.tolist() == [[0, 0, 5, 1, 1, 1], [0, 1, 2, 3, 4, 5]]
    assert st.finalize() == path
    assert fk.read_fka1(path).values.tolist() == [[0, 0, 5, 1, 1, 1], [0, 1, 2, 3, 4, 5]]
    st2 = fk.AssignmentStore(str(tmp_path / "t.fka1"), 1, 2)
    st2.abort()
    assert os.listdir(tmp_path) == ["s.fka1"]
    with pytest.raises(ValueError):
        fk.AssignmentStore(str(tmp_path / "u.fka1"), 0, 2)


def test_chunk_stream_reads(tmp_path):
    x = torch.randn(2, 23, 4)
    p = str(tmp_path / "x.fkm1")
    fk.write_fkm1(p, fk.DataMatrix(x))
    with fk.ChunkStream(p, 10) as s:
        assert (s.batch, s.total_points, s.dims, s.precision, s.n_chunks) == (2, 23, 4, "single", 3)
        assert [s.bounds(t) for t in range(3)] == [(0, 10), (10, 20), (20, 23)]
        with pytest.raises(ValueError):
            s.bounds(3)
        buf = torch.empty(10, 4).pin_memory() if torch.cuda.is_available() else torch.empty(10, 4)
        assert torch.equal(s.read_rows_into(1, 20, 23, buf), x[1, 20:23])
        npbuf = np.empty((10, 4), np.float32)
        assert np.array_equal(s.read_rows_into(0, 0, 10, npbuf), x[0, :10].numpy())
        assert torch.equal(s.read_rows(1, 5, 6), x[1, 5:6])
        with pytest.raises(ValueError, match="too small"):
            s.read_rows_into(0, 0, 11, buf)
        with pytest.raises(ValueError, match="dtype"):
            s.read_rows_into(0, 0, 2, torch.empty(10, 4, dtype=torch.float64))
        with pytest.raises(ValueError, match="bounds"):
            s.read_rows_into(0, 20, 24, buf)
    with pytest.raises(ValueError):
        fk.ChunkStream(p, 0)
    # a file truncated after the header check surfaces as a short read
    s = fk.ChunkStream(p, 10)
    with open(p, "r+b") as f:
        f.truncate(32 + 8 * 4 * 4)
    with pytest.raises(fk.DataFormatError, match="short read"):
        s.read_rows(0, 0, 10)
    s.close()


@pytest.mark.parametrize("method", ["random_distinct", pytest.param("kmeanspp", marks=pytest.mark.gpu)])
def test_stream_init_matches_in_core(tmp_path, method):
    x = fk.generate_dataset(2, 300, 5, 6, 1.0, 3, "single")
    p = str(tmp_path / "x.fkm1")
    fk.write_fkm1(p, x)
    with fk.ChunkStream(p, 37) as s:
        c_stream = _init_from_stream(s, 7, 11, method)
    idx = init_indices(300, 7, 11, 2, method, x.data.cuda() if method == "kmeanspp" else x.data)
    c_core = torch.stack([x.data[b][torch.from_numpy(idx[b])] for b in range(2)])
    assert torch.equal(c_stream.cpu(), c_core)


def test_reference_reads_our_bf16_rejecting_codes(tmp_path, reference):
    """Reference-readable for f32/f64; the bf16 extension code is rejected there."""
    p = str(tmp_path / "x.fkm1")
    x = torch.randn(1, 6, 3)
    fk.write_fkm1(p, fk.DataMatrix(x))
    assert np.array_equal(reference.read_fkm1(p).data, x.numpy())
    fk.write_fkm1(p, fk.DataMatrix(x.to(torch.bfloat16)))
    with pytest.raises(reference.DataFormatError):
        reference.read_fkm1(p)
