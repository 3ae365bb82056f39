"""The reference's DRAM traffic model vs ncu counters of the B200 kernels
(SURVEY.md §8f rank 3).

    python tools/traffic_vs_ncu.py [profiles/ncu_sweep_r1.json] > profiles/traffic_vs_ncu_r1.json
"""
import dataclasses
import json
import os
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
from paper_1803_11389_b200 import CellKind, RnnConfig  # noqa: E402
from paper_1803_11389_b200.traffic import compare_with_counters  # noqa: E402

src = sys.argv[1] if len(sys.argv) > 1 else os.path.join(REPO, "profiles", "ncu_sweep_r1.json")
rows = json.load(open(src))["rows"]
cfg = RnnConfig(CellKind.QRNN, 1024, 1024, precision="f32")  # cfg2
out = []
for r in rows:
    # bytes per weight / input element the measured kernel reads: bf16 operands;
    # f32x3 on tcgen05 reads tf32 hi + lo planes; FFMA kernels read fp32
    tc = r["kernel"].startswith("tc_layer")
    es = {"bf16": 2, "f32x3": 8 if tc else 4}.get(r["mode"], 4)
    c = compare_with_counters(cfg, 2048, r["T_b"], r["dram_MB"] * 1e6, weight_elem_bytes=es, act_elem_bytes=es)
    d = dataclasses.asdict(c)
    d = {"mode": r["mode"], "T_b": r["T_b"], "kernel": r["kernel"], **d, "l2_MB": r.get("l2_MB")}
    out.append(d)
print(json.dumps({"what": "cfg2 (QRNN 1024, L=2048): reference cold-cache weight-traffic model "
                          "(traffic.py estimate_traffic) vs ncu dram__bytes_read of one launch",
                  "source": os.path.relpath(src, REPO), "rows": out}, indent=1))
