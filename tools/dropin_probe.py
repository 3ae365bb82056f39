"""Where the reference-signature run_blocked call spends its time (weights are
uploaded and repacked per call, as the reference re-stacks them)."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1803_11389_b200 as P
from paper_1803_11389_b200 import workloads
w = workloads.make(sys.argv[1] if len(sys.argv) > 1 else "cfg2")
T = 32
for rep in range(4):
    t0 = time.perf_counter()
    st = P.DeviceStack(w.kind, w.layers, mode="f32")
    t1 = time.perf_counter()
    H = st.forward_host(w.X, T)
    t2 = time.perf_counter()
    st.close()
    t3 = time.perf_counter()
    print(f"create {1e3 * (t1 - t0):.2f} ms, forward_host (pageable) {1e3 * (t2 - t1):.2f} ms, close {1e3 * (t3 - t2):.2f} ms")
cfg_ = P.RnnConfig(w.kind, int(w.X.shape[1]), int(w.layers[-1].d_h), n_layers=len(w.layers), precision="f32")
ws_ = P.WeightSet(w.kind, "f32", w.layers)
Xf = np.ascontiguousarray(w.X, np.float32)
for rep in range(3):
    t0 = time.perf_counter()
    H2 = P.run_blocked(cfg_, ws_, Xf, T)
    print(f"run_blocked {1e3 * (time.perf_counter() - t0):.2f} ms")
