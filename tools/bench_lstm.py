"""Time the LSTM partial-precompute path (lstm_run_precomputed) on one GPU.

    python tools/bench_lstm.py [--out gpurun_out/lstm_bench.json]

Per width: W=3 warm-ups, then `reps` forwards each bracketed by CUDA events
with a 256 MB L2 flush before it; steps/s = L / mean time.  Shapes: the
reference's presets lstm-small / lstm-large (350 / 700, model_io.py:116-118)
and 1024 / 2048 wide layers (weights U(+-1/sqrt(d)), x ~ N(0,1), seeded).
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
import paper_1803_11389_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--out", default=os.path.join(REPO, "gpurun_out", "lstm_bench.json"))
    a = ap.parse_args()
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
    rows = []
    for d, L in ((350, 1024), (700, 1024), (1024, 2048), (2048, 1024)):
        rng = np.random.default_rng(d)
        s = 1.0 / np.sqrt(d)
        mats = [rng.uniform(-s, s, (d, d)).astype(np.float32) for _ in range(8)] + \
               [np.zeros(d, np.float32) for _ in range(4)]
        X = torch.from_numpy(rng.standard_normal((L, d)).astype(np.float32)).cuda()
        dev = P.DeviceLstm(mats)
        out = torch.empty((L, d), device="cuda")
        for _ in range(3):
            dev.forward(X, 32, out=out)
        torch.cuda.synchronize()
        ts = []
        for i in range(a.reps):
            flush.fill_(float(i))
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            dev.forward(X, 32, out=out)
            e1.record()
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1))
        ms = sum(ts) / len(ts)
        flops = 2.0 * 4 * d * (d + d) * L
        row = {"d_in": d, "d_h": d, "L": L, "ms": round(ms, 4), "steps_per_s": round(L / ms * 1e3, 1),
               "us_per_step": round(ms * 1e3 / L, 3), "tflops": round(flops / ms / 1e9, 2),
               "u_resident_smem": bool(dev.query(3)), "units_per_cta": dev.query(2), "grid": dev.query(4),
               "cluster_ctas": dev.query(5)}
        rows.append(row)
        print(row, flush=True)
        dev.close()
    os.makedirs(os.path.dirname(a.out), exist_ok=True)
    with open(a.out, "w") as f:
        json.dump({"what": "lstm_run_precomputed on one B200 (f32), L2 flushed, CUDA events", "rows": rows}, f,
                  indent=1)


if __name__ == "__main__":
    main()
