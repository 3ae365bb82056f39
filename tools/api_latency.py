"""Host-side cost of the CUDA calls the streaming host path issues (per call,
microseconds): tells a slow host (VM steal, CPU clocks) from a slow GPU path."""
import time
import torch
s = torch.cuda.Stream()
x = torch.empty(1024, device="cuda")
h = torch.empty(1024).pin_memory()
ev = torch.cuda.Event()
torch.cuda.synchronize()
def per_call(fn, n=2000):
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    dt = time.perf_counter() - t0
    torch.cuda.synchronize()
    return dt / n * 1e6
with torch.cuda.stream(s):
    print(f"memcpyAsync H2D 4 KB: {per_call(lambda: x.copy_(h, non_blocking=True)):.2f} us/call")
    print(f"event record: {per_call(lambda: ev.record(s)):.2f} us/call")
    print(f"tiny kernel launch: {per_call(lambda: x.add_(1.0)):.2f} us/call")
t0 = time.perf_counter(); n = 0
while time.perf_counter() - t0 < 0.2:
    n += 1
print(f"python loop iterations in 0.2 s: {n}")
