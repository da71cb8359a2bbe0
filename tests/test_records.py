"""Timing-record CSV helpers (reference bench.py:55-107): schema round trip and error classes on CPU,
a short device sweep on the GPU."""

import pytest

from paper_2405_17381_b200.errors import DomainError

torch = pytest.importorskip("torch")
from paper_2405_17381_b200.kernels import TimingRecord  # noqa: E402
from paper_2405_17381_b200.records import BenchGrid, read_csv, run_bench, write_csv  # noqa: E402


def _rec(n, pass_name="fwd"):
    return TimingRecord(kernel="lightning-decay", n=n, d=16, B=16, lam=0.9, pass_name=pass_name,
                        median_ns=1000 * n, per_token_ns=1000.0, aux_bytes=2048)


def test_csv_round_trip(tmp_path):
    recs = [_rec(64), _rec(128, "bwd")]
    path = tmp_path / "sub" / "t.csv"
    write_csv(recs, path)
    rows = read_csv(path)
    assert [r["n"] for r in rows] == [64, 128] and rows[1]["pass"] == "bwd"
    assert rows[0]["lambda"] == pytest.approx(0.9) and isinstance(rows[0]["median_ns"], int)
    assert path.read_text().splitlines()[0] == TimingRecord.CSV_HEADER


def test_csv_errors(tmp_path):
    with pytest.raises(FileNotFoundError):
        read_csv(tmp_path / "missing.csv")
    (tmp_path / "cols.csv").write_text("kernel,n\nx,1\n")
    with pytest.raises(DomainError):
        read_csv(tmp_path / "cols.csv")
    (tmp_path / "empty.csv").write_text(TimingRecord.CSV_HEADER + "\n")
    with pytest.raises(DomainError):
        read_csv(tmp_path / "empty.csv")
    bad = _rec(64).csv_row().replace(",64,", ",sixty-four,", 1)
    (tmp_path / "bad.csv").write_text(TimingRecord.CSV_HEADER + "\n" + bad + "\n")
    with pytest.raises(DomainError):
        read_csv(tmp_path / "bad.csv")


def test_grid_validation():
    with pytest.raises(DomainError):
        BenchGrid(kernels=("softmax",))
    with pytest.raises(DomainError):
        BenchGrid(passes=("sideways",))
    with pytest.raises(DomainError):
        BenchGrid(ns=())


@pytest.mark.gpu
def test_run_bench_on_device(tmp_path):
    seen = []
    recs = run_bench(BenchGrid(ns=(256, 512), d=16, B=16, lam=0.9, repeats=3, kernels=("lightning-decay",)),
                     progress=seen.append)
    assert [(r.n, r.pass_name) for r in recs] == [(256, "fwd"), (256, "bwd"), (512, "fwd"), (512, "bwd")]
    assert seen == recs and all(r.median_ns > 0 for r in recs)
    write_csv(recs, tmp_path / "b.csv")
    assert len(read_csv(tmp_path / "b.csv")) == 4
