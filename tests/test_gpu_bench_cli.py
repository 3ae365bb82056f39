"""bench_gpu CLI end to end on the GPU: verify-before-timing, CSV outputs,
file inputs (reference-written RNNW/RNNX), exit codes (cli.py:1-11)."""

import csv
import os

import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("cell", ["qrnn", "sru", "lstm"])
def test_bench_cli(tmp_path, cell):
    from paper_1803_11389_b200 import bench_gpu as B
    out = str(tmp_path / "s.csv")
    rc = B.main(["bench", "--cell", cell, "--width", "64", "--seq-len", "100", "--blocks", "1,8,32",
                 "--repeats", "2", "--out", out])
    assert rc == 0
    rows = list(csv.reader(open(out)))
    assert rows[0] == ["label", "median_ms", "speedup_pct"] and rows[1][2] == "100.0" and len(rows) == 4
    raw = list(csv.reader(open(str(tmp_path / "s.raw.csv"))))
    assert raw[0][0] == "cell" and len(raw) == 1 + 3 * 2


def test_bench_cli_files_and_errors(tmp_path):
    from paper_1803_11389_b200 import bench_gpu as B
    rc = B.main(["verify", "--weights", os.path.join(GOLDEN, "sru2_f32.rnnw"), "--input",
                 os.path.join(GOLDEN, "seq_f32.rnnx"), "--blocks", "1,4,37"])
    assert rc == 0
    bad = tmp_path / "bad.rnnw"
    bad.write_bytes(b"XXXX" + b"\0" * 12)
    assert B.main(["verify", "--weights", str(bad)]) == 3
