"""Summarise tools/ncu_sweep.sh CSVs into one JSON table.

    python tools/ncu_sweep_summary.py profiles/ncu_sweep_r1 > profiles/ncu_sweep_r1.json
"""
import csv
import json
import os
import sys

NAMES = {"gpu__time_duration.sum": ("us", 1e-3), "dram__bytes_read.sum": ("dram_MB", 1e-6),
         "lts__t_bytes.sum": ("l2_MB", 1e-6),
         "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active": ("tensor_pct", 1),
         "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active": ("fma_pct", 1),
         "smsp__issue_active.avg.pct_of_peak_sustained_active": ("issue_pct", 1),
         "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum": ("smem_wavefronts_M", 1e-6)}


def main(d):
    rows = []
    for f in sorted(os.listdir(d)):
        if not f.endswith(".csv"):
            continue
        mode, t = f[:-4].rsplit("_T", 1)
        lines = [ln for ln in open(os.path.join(d, f)) if ln.startswith('"')]
        rec = {"mode": mode, "T_b": int(t)}
        for r in csv.DictReader(lines):
            key = r["Metric Name"]
            if key in NAMES:
                name, scale = NAMES[key]
                rec[name] = round(float(r["Metric Value"].replace(",", "")) * scale, 2)
            rec["kernel"] = r["Kernel Name"].split("<")[0].replace("void rnnb::", "").replace("void ", "")
        rows.append(rec)
    rows.sort(key=lambda r: (r["mode"], r["T_b"]))
    print(json.dumps({"what": "ncu --metrics (one launch, cold caches) of the blocked-layer kernel on cfg2 "
                              "(QRNN 1024, L=2048) per mode and T_b; tools/ncu_sweep.sh", "rows": rows}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
