"""SM clock / power / throttle reasons sampled (NVML, 5 ms) while one
workload's forward runs back to back for a few seconds: tells a power-capped
kernel (clocks drop under the full pipeline) from a pipeline stall."""
import argparse
import os
import sys
import threading
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1803_11389_b200 as P  # noqa: E402
from paper_1803_11389_b200 import workloads  # noqa: E402
import pynvml  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg4")
ap.add_argument("--block", type=int, default=32)
ap.add_argument("--mode", default="bf16")
ap.add_argument("--seconds", type=float, default=3.0)
a = ap.parse_args()
w = workloads.make(a.workload)
st = P.DeviceStack(w.kind, w.layers, mode=a.mode)
X = torch.from_numpy(w.X.astype(st.np_dtype)).cuda()
for _ in range(2):
    st.forward(X, a.block)
torch.cuda.synchronize()
pynvml.nvmlInit()
h = pynvml.nvmlDeviceGetHandleByIndex(0)
sm, pw, rs = [], [], set()
stop = threading.Event()


def loop():
    while not stop.is_set():
        sm.append(pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM))
        pw.append(pynvml.nvmlDeviceGetPowerUsage(h) / 1000.0)
        rs.add(pynvml.nvmlDeviceGetCurrentClocksEventReasons(h))
        time.sleep(0.005)


t = threading.Thread(target=loop, daemon=True)
t.start()
t0 = time.time()
n = 0
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
while time.time() - t0 < a.seconds:
    st.forward(X, a.block)
    torch.cuda.synchronize()
    n += 1
e1.record()
torch.cuda.synchronize()
stop.set()
t.join()
sm.sort()
print(f"{a.workload} {a.mode} T_b={a.block} dbg={os.environ.get('RNNB_DEBUG', '0')}: {e0.elapsed_time(e1) / n:.3f} ms/forward, "
      f"sm MHz min/median/max {sm[0]}/{sm[len(sm) // 2]}/{sm[-1]}, power max {max(pw):.0f} W, reasons {sorted(rs)}")
