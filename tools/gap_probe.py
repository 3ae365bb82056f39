"""Where a forward's time goes: CUDA-event time of st.forward (as bench.py
times it, after an L2 flush) vs the device time of each kernel it launched
(torch.profiler / CUPTI).  The difference is launch gaps on the stream."""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1803_11389_b200 as P  # noqa: E402
from paper_1803_11389_b200 import workloads  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg2")
ap.add_argument("--mode", default="bf16")
ap.add_argument("--blocks", default="16,32,64")
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
w = workloads.make(a.workload)
st = P.DeviceStack(w.kind, w.layers, mode=a.mode)
X = torch.from_numpy(w.X.astype(st.np_dtype)).cuda()
out = torch.empty((w.seq_len, st.d_h[-1]), dtype=st.dtype, device="cuda")
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
for T in [int(b) for b in a.blocks.split(",")]:
    for _ in range(3):
        st.forward(X, T, out=out)
    ts = []
    for i in range(a.reps):
        flush.fill_(float(i))
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        st.forward(X, T, out=out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
        for i in range(5):
            flush.fill_(float(i))
            st.forward(X, T, out=out)
        torch.cuda.synchronize()
    per = {}
    for e in prof.events():
        if e.device_type == torch.autograd.DeviceType.CUDA and "fill" not in e.name.lower():
            per.setdefault(e.name[:70], []).append(e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total)
    ts.sort()
    print(f"{a.workload} {a.mode} T_b={T}: event median {ts[len(ts) // 2]:.1f} us, min {ts[0]:.1f} us")
    tot = 0.0
    for k, v in per.items():
        m = sum(v) / 5
        tot += m
        print(f"   {m:8.1f} us/forward  x{len(v) / 5:.0f}  {k}")
    print(f"   kernels+copies total {tot:.1f} us -> gaps {ts[len(ts) // 2] - tot:.1f} us")
