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


REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _peak(path, key, default):
    try:
        with open(os.path.join(REPO, path)) as f:
            return json.load(f)[key]
    except (OSError, KeyError, ValueError):
        return default


HBM_GBS = _peak("MEASURED_PEAKS.json", "hbm_gbs", 6543.7)
L2_GBS = _peak("profiles/l2_peak.json", "l2_read_gbs", 11781.8)


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
        # achieved bandwidths against the measured peaks (per launch)
        if rec.get("us"):
            sec = rec["us"] * 1e-6
            rec["dram_gbs"] = round(rec.get("dram_MB", 0) * 1e6 / sec / 1e9, 1)
            rec["l2_gbs"] = round(rec.get("l2_MB", 0) * 1e6 / sec / 1e9, 1)
            rec["dram_frac"] = round(rec["dram_gbs"] / HBM_GBS, 4)
            rec["l2_frac"] = round(rec["l2_gbs"] / L2_GBS, 4)
        rows.append(rec)
    rows.sort(key=lambda r: (r["mode"], r["T_b"]))
    print(json.dumps({"what": "ncu --metrics (one launch, cold caches) of the blocked-layer kernel on cfg2 "
                              "(QRNN 1024, L=2048) per mode and T_b; tools/ncu_sweep.sh.  dram/l2 GB/s = "
                              "measured bytes / kernel time, fractions against MEASURED_PEAKS.json hbm_gbs "
                              f"({HBM_GBS}) and profiles/l2_peak.json ({L2_GBS}); tensor_pct / fma_pct = "
                              "pipe utilisation", "rows": rows}, indent=1))


if __name__ == "__main__":
    main(sys.argv[1])
