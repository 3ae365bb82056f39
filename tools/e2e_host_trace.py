"""Host-side time stamps of rnnb_forward_host's streaming call (RNNB_STREAM_TRACE=3)."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1803_11389_b200 as P
from paper_1803_11389_b200 import workloads
w = workloads.make("cfg2")
st = P.DeviceStack(w.kind, w.layers, mode="f32")
Xh = torch.from_numpy(w.X.astype(st.np_dtype)).pin_memory()
Hh = torch.empty((w.seq_len, st.d_h[-1]), dtype=st.dtype).pin_memory()
Xn, Hn = Xh.numpy(), Hh.numpy()
for _ in range(5):
    st.forward_host(Xn, 32, out=Hn)
ts = []
for _ in range(30):
    t0 = time.perf_counter(); st.forward_host(Xn, 32, out=Hn); ts.append(time.perf_counter() - t0)
print(f"median {np.median(ts) * 1e3:.4f} ms")
os.environ["RNNB_STREAM_TRACE"] = "3"
for _ in range(3):
    t0 = time.perf_counter(); st.forward_host(Xn, 32, out=Hn)
    print(f"call {(time.perf_counter() - t0) * 1e6:.1f} us", flush=True)
