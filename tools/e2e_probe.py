"""Wall-clock timing of the host-buffer entry point (rnnb_forward_host) for
one workload, as bench.py's e2e leg measures it; for tuning the streaming
path (RNNB_STREAM_CHUNK, RNNB_NT32, RNNB_HOST_STREAM).  Not the bench."""
import argparse
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1803_11389_b200 as P  # noqa: E402
from paper_1803_11389_b200 import workloads  # noqa: E402

def bind_to_gpu_numa_node(index=0):
    """Pin this process to the CPU cores NVML reports as local to the GPU, so
    pinned host buffers are first-touched on the GPU's NUMA node."""
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(index)
        n = os.cpu_count() or 1
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (n + 63) // 64)
        cpus = [64 * i + b for i, wd in enumerate(words) for b in range(64) if (wd >> b) & 1 and 64 * i + b < n]
        if cpus:
            os.sched_setaffinity(0, cpus)
        return cpus
    except Exception as e:  # noqa: BLE001
        return f"unavailable: {e}"


ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg2")
ap.add_argument("--block", type=int, default=32)
ap.add_argument("--mode", default="f32")
ap.add_argument("--reps", type=int, default=50)
ap.add_argument("--tag", default="")
a = ap.parse_args()
if os.environ.get("E2E_BIND"):
    print("bound to cpus", bind_to_gpu_numa_node(), flush=True)
print("affinity", sorted(os.sched_getaffinity(0))[:4], "...", len(os.sched_getaffinity(0)), "cpus", flush=True)
w = workloads.make(a.workload)
st = P.DeviceStack(w.kind, w.layers, mode=a.mode)
Xh = torch.from_numpy(w.X.astype(st.np_dtype)).pin_memory()
Hh = torch.empty((w.seq_len, st.d_h[-1]), dtype=st.dtype).pin_memory()
Xn, Hn = Xh.numpy(), Hh.numpy()
for _ in range(5):
    st.forward_host(Xn, a.block, out=Hn)
torch.cuda.synchronize()
ts = []
for _ in range(a.reps):
    t0 = time.perf_counter()
    st.forward_host(Xn, a.block, out=Hn)
    ts.append(time.perf_counter() - t0)
ts = np.array(ts) * 1e3
L = w.seq_len
print(f"{a.tag} {a.workload} {a.mode} T_b={a.block}: mean {ts.mean():.4f} ms ({L / ts.mean() * 1e-3:.3f} M steps/s) "
      f"median {np.median(ts):.4f} min {ts.min():.4f} max {ts.max():.4f}", flush=True)

if os.environ.get("E2E_TIMELINE"):
    # CUPTI timeline of one call: start/end of every copy and kernel relative to the first activity
    with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA, torch.profiler.ProfilerActivity.CPU]) as prof:
        t0 = time.perf_counter()
        st.forward_host(Xn, a.block, out=Hn)
        t1 = time.perf_counter()
    evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    base = min(e.time_range.start for e in evs)
    print(f"wall {(t1 - t0) * 1e6:.1f} us; device span {max(e.time_range.end for e in evs) - base:.1f} us")
    for e in sorted(evs, key=lambda e: e.time_range.start):
        print(f"  {e.time_range.start - base:9.1f} .. {e.time_range.end - base:9.1f}  {e.name[:60]}")

if os.environ.get("E2E_TRACE"):
    # device-side event trace of the streaming path (RNNB_STREAM_TRACE, rnnb_api.cu)
    os.environ["RNNB_STREAM_TRACE"] = "1"
    for _ in range(2):
        t0 = time.perf_counter()
        st.forward_host(Xn, a.block, out=Hn)
        print(f"traced call wall {(time.perf_counter() - t0) * 1e6:.1f} us", flush=True)
