import sys, os, numpy as np, torch
sys.path.insert(0, '/root/repo'); sys.path.insert(0, '/root/repo/oracle')
import oracle as O
import paper_1803_11389_b200 as P
from paper_1803_11389_b200 import workloads
for wl in ("cfg2",):
    w = workloads.make(wl)
    st = P.DeviceStack(w.kind, w.layers, mode="f32")
    ref = O.run_blocked("qrnn", [l.mats() for l in w.layers], w.X, 32)
    H = st.forward(torch.from_numpy(w.X).cuda(), 32).cpu().numpy()
    print(wl, "err", float(np.max(np.abs(H - ref)) / np.max(np.abs(ref))))
w = workloads.make("cfg4")
xp = np.ascontiguousarray(w.X[:8192])
mats = [l.mats() for l in w.layers]
ref = O.run_blocked("qrnn", mats, xp, 32)
st = P.DeviceStack(w.kind, w.layers, mode="f32")
H = st.forward(torch.from_numpy(xp).cuda(), 32).cpu().numpy()
print("cfg4 prefix err", float(np.max(np.abs(H - ref)) / np.max(np.abs(ref))))
