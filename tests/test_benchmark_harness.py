"""Bench/tune/ttfr harness (reference cli.py bench schema, cli.py:63-67, 287-336)."""

import os

import pytest

from paper_2603_09229_b200 import benchmark as bm


def test_usage_errors_exit_1(capsys):
    assert bm.main(["bench", "--n", "x,y", "--k", "4", "--d", "2", "--out", "/tmp/x.csv"]) == 1
    assert bm.main(["nosuch"]) == 1
    assert bm.main(["ttfr", "--shapes", "1:2:3", "--out", "/tmp/x.csv"]) == 1


def test_sweep_validation():
    with pytest.raises(ValueError, match="every K"):
        bm.bench_sweep([100], [200], [4])
    with pytest.raises(ValueError, match="engine"):
        bm.bench_sweep([100], [10], [4], engines=("nope",))
    with pytest.raises(ValueError, match="reps"):
        bm.bench_sweep([100], [10], [4], reps=0)


@pytest.mark.gpu
@pytest.mark.parametrize("dtype", ["single", "bf16"])
def test_bench_csv_schema(tmp_path, dtype):
    out = str(tmp_path / "b.csv")
    assert bm.main(["bench", "--n", "4096", "--k", "64", "--d", "32", "--b", "1,2", "--reps", "3",
                    "--dtype", dtype, "--out", out]) == 0
    rows = open(out).read().strip().split("\n")
    assert rows[0] == bm.BENCH_COLUMNS
    assert len(rows) == 1 + 2 * 2 * 3
    cols = bm.BENCH_COLUMNS.split(",")
    for r in rows[1:]:
        v = dict(zip(cols, r.split(",")))
        assert len(r.split(",")) == len(cols)
        assert int(v["median_latency_ns"]) > 0
        if v["engine"] == "flash":
            assert int(v["intermediate_bytes_written"]) == 0      # nothing N x K reaches HBM
            assert v["b_n"] != "" and int(v["update_chunk"]) >= 1
        elif v["stage"] in ("assign", "e2e"):
            assert int(v["intermediate_bytes_written"]) >= int(v["b"]) * 4096 * 64 * 4


@pytest.mark.gpu
def test_ttfr_and_tune(tmp_path):
    out = str(tmp_path / "t.csv")
    assert bm.main(["ttfr", "--shapes", "65536:1024:128:1,4096:64:64:4", "--out", out]) == 0
    rows = open(out).read().strip().split("\n")
    assert rows[0] == bm.TTFR_COLUMNS and len(rows) == 3
    for r in rows[1:]:
        f = r.split(",")
        assert int(f[6]) > 0 and int(f[7]) > 0
    out2 = str(tmp_path / "tune.csv")
    assert bm.main(["tune", "--n", "8192", "--k", "64", "--d", "32", "--reps", "3", "--out", out2]) == 0
    assert open(out2).readline().strip() == "b_n,b_k,update_chunk,median_latency_ns"
