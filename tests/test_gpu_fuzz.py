"""Seeded randomized parity sweep: random (cell, widths, layers, L, T_b, mode,
entry point) combinations through the CUDA path vs the oracle (the C
restatement pinned to the reference's goldens), with the bounds of
tests/test_gpu_parity.py:

* f32 / f32x3: normwise <= 1e-5 and max-abs <= 1e-4 vs the fp32 oracle;
* f64: max-abs <= 1e-12;
* tf32 / bf16: normwise <= 2e-3 / 2e-2 vs the fp32 oracle.

Shapes cover every kernel family: unaligned widths (generic FFMA kernel),
aligned (warp-specialised kernel, register kernel at T_b = 1), tcgen05 (bf16
/ tf32 / f32x3), partial blocks, T_b > L; entry points `DeviceStack.forward`
(device buffers), `forward_host` (the streaming / chunked host path) and the
reference-shaped `run_blocked`."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

N_CASES = 160


def _cases():
    rng = np.random.default_rng(20261020)
    out = []
    for i in range(N_CASES):
        kind = ("sru", "qrnn")[int(rng.integers(2))]
        mode = ("f32", "f32", "f64", "bf16", "tf32", "f32x3")[int(rng.integers(6))]
        aligned = rng.random() < 0.7
        d = int(rng.integers(2, 40)) * 8 if aligned else int(rng.integers(3, 300))
        n_layers = int(rng.integers(1, 4))
        L = int(rng.integers(1, 400))
        T = int(rng.choice([1, 2, 3, 4, 7, 8, 16, 24, 32, 33, 64, 100, 500]))
        entry = ("forward", "forward", "host", "run_blocked")[int(rng.integers(4))]
        if entry == "run_blocked" and mode not in ("f32", "f64"):
            entry = "forward"
        out.append((i, kind, mode, d, n_layers, L, T, entry))
    return out


def _normwise(a, ref):
    ref = np.asarray(ref, np.float64)
    return float(np.max(np.abs(np.asarray(a, np.float64) - ref)) / max(np.max(np.abs(ref)), 1e-30))


@pytest.mark.parametrize("case", _cases(), ids=lambda c: f"{c[0]}-{c[1]}-{c[2]}-d{c[3]}-n{c[4]}-L{c[5]}-T{c[6]}-{c[7]}")
def test_random_case_matches_oracle(oracle, case):
    import torch
    import paper_1803_11389_b200 as P
    i, kind, mode, d, n_layers, L, T, entry = case
    dt = np.float64 if mode == "f64" else np.float32
    layers = oracle.generate_layers(kind, d, d, n_layers, 1000 + i, dt)
    X = np.random.default_rng(2000 + i).standard_normal((L, d)).astype(dt)
    ref = oracle.run_blocked(kind, layers, X if mode != "f64" else X, T)
    if entry == "run_blocked":
        k = P.CellKind.parse(kind)
        cls = P.SruWeights if k is P.CellKind.SRU else P.QrnnWeights
        ws = P.WeightSet(k, "f64" if mode == "f64" else "f32", [cls(*[np.ascontiguousarray(m) for m in lay])
                                                               for lay in layers])
        cfg = P.RnnConfig(k, d, d, n_layers=n_layers, precision="f64" if mode == "f64" else "f32")
        H = P.run_blocked(cfg, ws, X, T)
    else:
        st = P.DeviceStack(kind, layers, mode=mode)
        if entry == "host":
            H = st.forward_host(X, T)
        else:
            H = st.forward(torch.from_numpy(X).cuda(), T).cpu().numpy()
        st.close()
    assert H.shape == (L, d) and H.dtype == dt
    if mode == "f64":
        assert float(np.max(np.abs(H - ref))) <= 1e-12
    elif mode in ("f32", "f32x3"):
        assert _normwise(H, ref) <= 1e-5 and float(np.max(np.abs(H.astype(np.float64) - ref))) <= 1e-4, \
            _normwise(H, ref)
    else:
        assert _normwise(H, ref) <= (2e-3 if mode == "tf32" else 2e-2), _normwise(H, ref)
