"""Error of the 3xTF32 tensor-core mode vs K (f64 oracle), to see whether the
tensor-core fp32 accumulation error grows with the reduction length."""
import os
import sys

import numpy as np
import torch

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "oracle"))
import oracle as O  # noqa: E402
import paper_1803_11389_b200 as P  # noqa: E402

for kind in ("qrnn", "sru"):
    for d in (128, 256, 512, 1024, 2048):
        layers = O.generate_layers(kind, d, d, 1, 3, np.float32)
        s = 1.0 / np.sqrt(d) / 0.058  # rescale U(+-0.1) to ~U(+-1/sqrt(d)) * const
        layers = [[(m * s).astype(np.float32) if m.ndim == 2 else m for m in l] for l in layers]
        X = np.random.default_rng(1).standard_normal((256, d)).astype(np.float32)
        ref = O.run_blocked(kind, [[m.astype(np.float64) for m in l] for l in layers], X.astype(np.float64), 32)
        out = {}
        for mode in ("f32", "f32x3"):
            st = P.DeviceStack(kind, layers, mode=mode)
            H = st.forward(torch.from_numpy(X).cuda(), 32).cpu().numpy()
            out[mode] = float(np.max(np.abs(H - ref)) / np.max(np.abs(ref)))
            st.close()
        print(kind, "K =", d * (2 if kind == "qrnn" else 1), {k: f"{v:.2e}" for k, v in out.items()}, flush=True)
