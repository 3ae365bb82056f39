"""Quick device timing of one workload forward per T_b (CUDA events, no L2
flush) for kernel iteration; not the bench."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1803_11389_b200 as P  # noqa: E402
from paper_1803_11389_b200 import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg2")
ap.add_argument("--blocks", default="1,2,4,8,16,32")
ap.add_argument("--mode", default="f32")
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--scale", type=float, default=1.0)
a = ap.parse_args()
w = workloads.make(a.workload, scale=a.scale)
st = P.DeviceStack(w.kind, w.layers, mode=a.mode)
Xn = w.X if w.X.shape[1] == st.d_in[0] else \
    __import__("numpy").random.default_rng(0).standard_normal((w.seq_len, st.d_in[0])).astype("float32")
X = torch.from_numpy(Xn.astype(st.np_dtype)).cuda()
L = w.seq_len
fl = workloads.flops_per_step(w)
for T in [int(b) for b in a.blocks.split(",")]:
    for _ in range(3):
        st.forward(X, T)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.reps):
        st.forward(X, T)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / a.reps
    print(f"{a.workload} {a.mode} T_b={T:3d}: {ms:8.4f} ms  {L / ms * 1e3 / 1e6:7.3f} M steps/s  "
          f"{fl * L / ms / 1e9:7.2f} TFLOP/s  ws={st.query(6)} nt={st.query(7)} kc={st.query(8)} "
          f"smem={st.query(5)} grid={st.query(4)} reg={st.query(10)} tc={st.query(9)}", flush=True)
