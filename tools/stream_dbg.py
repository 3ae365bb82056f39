import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "oracle"))
import oracle
import paper_1803_11389_b200 as P
kind, mode, d, L, T = sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4]), int(sys.argv[5])
layers = oracle.generate_layers(kind, d, d, 1, 73, np.float32)
X = np.random.default_rng(20).standard_normal((L, d)).astype(np.float32)
st = P.DeviceStack(kind, layers, mode=mode)
c0 = np.random.default_rng(21).standard_normal(d).astype(np.float32)
x0 = np.random.default_rng(22).standard_normal(d).astype(np.float32)
cd, xd = torch.from_numpy(c0.copy()).cuda(), torch.from_numpy(x0.copy()).cuda()
ref = st.forward(torch.from_numpy(X).cuda(), T, c_state=cd, x_carry=xd if kind == "qrnn" else None).cpu().numpy()
import time
if os.environ.get("PIN"):
    X = torch.from_numpy(X).pin_memory().numpy()
for rep in range(3):
    c, x = c0.copy(), x0.copy()
    t0 = time.perf_counter()
    H = st.forward_host(X, T, c_state=c, x_carry=x if kind == "qrnn" else None)
    print(f"call {time.perf_counter() - t0:.4f} s")
    bad = np.argwhere(H != ref)
    print(f"rep {rep}: {len(bad)} differing of {H.size}; max abs diff {np.abs(H - ref).max():.3e}; "
          f"rows {sorted(set(bad[:, 0]))[:12]} cols {sorted(set(bad[:, 1]))[:12]} ncols {len(set(bad[:,1]))}")
