"""bench.py keeps the driver's JSON contract: one line with the required
keys, e2e with its byte counts, the roofline and CPU-baseline objects, the
clock sample; the reference arm's line likewise (short runs)."""

import json
import os
import subprocess
import sys

import pytest

from conftest import REPO

pytestmark = pytest.mark.gpu


def _run(args, timeout=600):
    r = subprocess.run([sys.executable, os.path.join(REPO, "bench.py")] + args, capture_output=True, text=True,
                       timeout=timeout, cwd=REPO)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    return json.loads(lines[0])


def test_bench_line_contract():
    d = _run(["--steps", "3", "--warmup", "3", "--no-sweep", "--extra-modes", "", "--cpu-seconds", "1",
              "--cpu-sample", "64", "--no-configs", "--no-partitioned"])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "e2e", "gpu_launches", "roofline",
              "cpu_baseline", "clocks"):
        assert k in d, k
    assert d["n_gpus"] == 1 and d["steps"] == 3 and d["warmup"] == 3 and d["higher_is_better"] is True
    assert d["value"] > 0 and d["unit"] == "steps/s" and d["config"]["workload"] == "cfg2"
    assert "flushed" in d["config"]["l2"]
    e = d["e2e"]
    assert e["value"] > 0 and e["unit"] == d["unit"]
    assert e["h2d_bytes_per_step"] == 2048 * 1024 * 4 and e["d2h_bytes_per_step"] == 2048 * 1024 * 4
    r = d["roofline"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in r, k
    assert 0 < r["frac"] < 1 and abs(r["frac"] - r["achieved"] / r["peak"]) < 1e-3
    c = d["cpu_baseline"]
    for k in ("value", "unit", "cores", "kind", "sample"):
        assert k in c, k
    assert c["kind"] in ("port", "reference") and c["cores"] >= 1
    assert c["cpu_model"] and c["single_thread"]["cores"] == 1 and c["single_thread"]["value"] > 0
    # fp32 at T_b = 32 runs the 3xTF32 tcgen05 layer kernel: operand conversion + layer kernel per step
    assert r["bound"] == "tensor" and "3xTF32" in r["pipe"]
    assert d["gpu_launches"] == 3 * 2
    assert 0 < r["tensor_issue"]["frac"] <= 1 and 0 < r["l2_feed"]["frac"] <= 1
    cl = d["clocks"]
    assert {"sm_mhz", "sm_max_mhz", "reasons"} <= set(cl)


def test_reference_arm_line():
    d = _run(["--impl", "reference", "--steps", "3", "--warmup", "3", "--cpu-sample", "64"])
    assert d["impl"] == "reference" and d["value"] > 0
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    assert d["cpu_baseline"]["value"] == d["value"] and d["cpu_baseline"]["cpu_model"]


def test_bench_partitioned_and_configs_objects():
    """The default line's extra objects (short run): the partitioned cfg4 /
    cfg5 paths at N = 1 and one line per other BASELINE config."""
    d = _run(["--steps", "3", "--warmup", "3", "--no-sweep", "--extra-modes", "", "--no-cpu-baseline"],
             timeout=1200)
    p = d["partitioned"]
    assert set(p) == {"pipeline", "hidden"}
    for v in p.values():
        assert v["value"] > 0 and v["scaling"] == "strong" and v["n_gpus"] == 1
    c = d["configs"]
    assert {"cfg1/f32", "cfg3/f32", "cfg3/bf16", "cfg4/f32", "cfg4/bf16", "cfg5/bf16"} <= set(c)
    for v in c.values():
        for row in v["blocks"].values():
            assert row["steps_per_s"] > 0 and 0 < row["frac"] <= 1.0, row
