"""bench_gpu's CSV surface against CSVs written by the reference's own
emit_csv for the same rows (tests/golden/bench_*.csv)."""

import os

from conftest import GOLDEN


def _read(p):
    with open(p) as f:
        return f.read()


def test_csv_byte_identical(tmp_path):
    from paper_1803_11389_b200 import CellKind, RnnConfig, bench_gpu as B
    recs = [B.BenchRecord("qrnn", "blocked", 16, 16, 64, T, 8, r, 10.0 / T + 0.25 * r) for T in (1, 4) for r in range(3)]
    B.emit_csv(recs, tmp_path / "r.csv")
    assert _read(tmp_path / "r.csv") == _read(os.path.join(GOLDEN, "bench_records.csv"))
    rows = B.summarize(recs) + [B.SpeedupRow("LSTM", 673.667, None)]
    B.emit_csv(rows, tmp_path / "s.csv")
    assert _read(tmp_path / "s.csv") == _read(os.path.join(GOLDEN, "bench_summary.csv"))
    cfg = RnnConfig(CellKind.QRNN, 64, 64, precision="f32")
    B.emit_csv([B.estimate_traffic(cfg, 100, T) for T in (1, 8)], tmp_path / "t.csv")
    assert _read(tmp_path / "t.csv") == _read(os.path.join(GOLDEN, "bench_traffic.csv"))


def test_speedup_convention():
    import pytest
    from paper_1803_11389_b200 import bench_gpu as B
    assert B.speedup(475.43, 93.219) == 510.0
    with pytest.raises(ValueError):
        B.speedup(0, 1)
    with pytest.raises(ValueError):
        B.emit_csv([], "/tmp/x.csv")
