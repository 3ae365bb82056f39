"""First rnnb_forward_host call on a fresh handle with the stream trace on
(debugging the streaming path)."""
import os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1803_11389_b200 as P
from paper_1803_11389_b200 import workloads
os.environ["RNNB_STREAM_TRACE"] = "1"
os.environ["RNNB_STREAM_DEBUG"] = "1"
w = workloads.make("cfg2")
st = P.DeviceStack(w.kind, w.layers, mode="f32")
Xh = torch.from_numpy(w.X.astype(st.np_dtype)).pin_memory()
Hh = torch.empty((w.seq_len, st.d_h[-1]), dtype=st.dtype).pin_memory()
Xn, Hn = Xh.numpy(), Hh.numpy()
ref = st.forward(Xh.cuda(), 32).cpu().numpy()
for i in range(3):
    t0 = time.perf_counter()
    st.forward_host(Xn, 32, out=Hn)
    print(f"call {i}: {(time.perf_counter() - t0) * 1e3:.3f} ms, bitwise equal to device call: {Hn.tobytes() == ref.tobytes()}", flush=True)
