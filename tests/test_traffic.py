"""The traffic model (paper_1803_11389_b200.traffic) against the reference's
own numbers (tests/golden/traffic.json, made by rnnblock.traffic), and the
model-vs-counters comparison on the committed ncu sweep."""

import json
import os

import pytest

from conftest import GOLDEN, REPO


def _rows():
    with open(os.path.join(GOLDEN, "traffic.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("row", _rows(), ids=lambda r: f"{r['kind']}{r['d_in']}x{r['d_h']}x{r['n_layers']}-L{r['L']}-T{r['T']}")
def test_traffic_model_matches_reference(row):
    from paper_1803_11389_b200 import CellKind, RnnConfig, traffic
    cfg = RnnConfig(CellKind.parse(row["kind"]), row["d_in"], row["d_h"], n_layers=row["n_layers"],
                    precision=row["precision"])
    r = traffic.estimate_traffic(cfg, row["L"], row["T"])
    assert (r.weight_bytes, r.blocks, r.est_weight_traffic) == (row["weight_bytes"], row["blocks"], row["est"])
    assert r.per_step_traffic == row["per_step"] and r.ratio_vs_t1 == row["ratio"]
    assert traffic.expected_phase_touches(cfg, row["L"], row["T"]) == row["touches"]
    if row["kind"] == "lstm":
        assert list(traffic.lstm_split_bytes(cfg)) == row["split"]


def test_measured_dram_is_weights_once():
    """profiles/traffic_vs_ncu_r1.json: for the FFMA and bf16 tcgen05 kernels
    DRAM reads equal one pass over the weights plus the input (within 1 %)
    at every T_b, while the cold-cache model grows as ceil(L/T_b)."""
    with open(os.path.join(REPO, "profiles", "traffic_vs_ncu_r1.json")) as f:
        rows = json.load(f)["rows"]
    for r in rows:
        if r["mode"] in ("f32", "bf16"):
            assert 0.99 <= r["measured_over_floor"] <= 1.02, r
    t1 = [r for r in rows if r["mode"] == "f32" and r["T_b"] == 1][0]
    assert t1["model_over_measured"] > 1000
