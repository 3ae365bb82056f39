"""Run one workload forward a few times with no timing: the command the
ncu captures in profiles/ are taken on."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1803_11389_b200 as P  # noqa: E402
from paper_1803_11389_b200 import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg2")
ap.add_argument("--block", type=int, default=32)
ap.add_argument("--mode", default="f32")
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--scale", type=float, default=1.0)
a = ap.parse_args()
w = workloads.make(a.workload, scale=a.scale)
st = P.DeviceStack(w.kind, w.layers, mode=a.mode)
X = torch.from_numpy(w.X.astype(st.np_dtype)).cuda()
for _ in range(a.reps):
    H = st.forward(X, a.block)
torch.cuda.synchronize()
print("ok", a.workload, a.block, a.mode, float(H.float().abs().sum()))
