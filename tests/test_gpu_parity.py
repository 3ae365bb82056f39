"""GPU parity: the CUDA path (through librnnb.so) against the oracle and the
reference's own golden outputs.

Tolerances (written per test):
* fp32: normwise max|d|/max|ref| <= 1e-5 AND max|d| <= 1e-4
  (the reference's ORACLE_TOLERANCE, bench.py:25);
* f64: max|d| <= 1e-12;
* TF32: <= 2e-3 normwise vs the fp32 oracle, <= 1e-5 vs the oracle on
  tf32-rounded operands;
* BF16: <= 2e-2 normwise vs the fp32 oracle, <= 1e-3 vs the oracle on
  bf16-rounded weights and inputs.
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def normwise(a, ref):
    ref = np.asarray(ref, np.float64)
    return float(np.max(np.abs(np.asarray(a, np.float64) - ref)) / max(np.max(np.abs(ref)), 1e-30))


def assert_f32(a, ref):
    d = float(np.max(np.abs(np.asarray(a, np.float64) - np.asarray(ref, np.float64))))
    assert normwise(a, ref) <= 1e-5 and d <= 1e-4, (normwise(a, ref), d)


@pytest.fixture(scope="module")
def P():
    import paper_1803_11389_b200 as P
    return P


def _ws(P, kind, layers, precision):
    kind = P.CellKind.parse(kind)
    cls = P.SruWeights if kind is P.CellKind.SRU else P.QrnnWeights
    return P.WeightSet(kind, precision, [cls(*[np.ascontiguousarray(m) for m in lay]) for lay in layers])


def _cfg(P, kind, d, n_layers, precision):
    return P.RnnConfig(P.CellKind.parse(kind), d, d, n_layers=n_layers, precision=precision)


def _cases():
    with open(os.path.join(GOLDEN, "blocked_cases.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("case", _cases(), ids=lambda c: f"{c['kind']}-{c['precision']}-d{c['d']}-L{c['L']}-n{c['n_layers']}")
def test_run_blocked_matches_reference_fixtures(P, oracle, case):
    g = np.load(os.path.join(GOLDEN, "blocked_cases.npz"))
    prec = case["precision"]
    dt = np.float32 if prec == "f32" else np.float64
    layers = oracle.generate_layers(case["kind"], case["d"], case["d"], case["n_layers"], case["wseed"], dt)
    X = oracle.generate_sequence(case["L"], case["d"], case["xseed"], dt)
    cfg = _cfg(P, case["kind"], case["d"], case["n_layers"], prec)
    ws = _ws(P, case["kind"], layers, prec)
    n = case["case"]
    for T in case["T_b"]:
        H, cs, xcs = P.run_blocked(cfg, ws, X, T, return_state=True)
        assert H.dtype == dt and H.shape == (case["L"], case["d"])
        ref = g[f"c{n}_T{T}_H"]
        if prec == "f32":
            assert_f32(H, ref)
            assert_f32(np.stack(cs), g[f"c{n}_T{T}_c"])
        else:
            assert np.max(np.abs(H - ref)) <= 1e-12
            assert np.max(np.abs(np.stack(cs) - g[f"c{n}_T{T}_c"])) <= 1e-12
        # and against the stepwise oracle of the reference (bench.verify)
        step = g[f"c{n}_stepwise"]
        assert np.max(np.abs(H - step)) <= (1e-4 if prec == "f32" else 1e-9)


@pytest.mark.parametrize("kind", ["sru", "qrnn"])
def test_d2_golden_vectors_on_gpu(P, kind):
    with open(os.path.join(GOLDEN, "cells_d2.json")) as f:
        g = json.load(f)[kind]
    fields = ("w_cand", "w_forget", "w_highway", "b_forget", "b_highway") if kind == "sru" else \
        ("w_cand", "w_cand_prev", "w_forget", "w_forget_prev", "w_out", "w_out_prev")
    layer = [np.array(g["weights"][f], np.float64) for f in fields]
    X = np.array(g["X"], np.float64)
    cfg = _cfg(P, kind, 2, 1, "f64")
    for T in (1, 2, 3):
        H, cs, _ = P.run_blocked(cfg, _ws(P, kind, [layer], "f64"), X, T, return_state=True)
        assert np.max(np.abs(H - np.array(g["H"]))) < 1e-12
        assert np.max(np.abs(cs[0] - np.array(g["C"][-1]))) < 1e-12


@pytest.mark.parametrize("kind", ["sru", "qrnn"])
@pytest.mark.parametrize("d", [3, 40, 256])
def test_block_size_sweep_vs_oracle(P, oracle, kind, d):
    """Every T_b incl. remainders, T_b > L and non-power-of-2 widths."""
    L = 150
    layers = oracle.generate_layers(kind, d, d, 1, 100 + d, np.float32)
    X = np.random.default_rng(d).standard_normal((L, d)).astype(np.float32)
    cfg = _cfg(P, kind, d, 1, "f32")
    ws = _ws(P, kind, layers, "f32")
    for T in (1, 2, 3, 4, 5, 8, 13, 16, 17, 32, 64, 128, 200):
        ref, cref, _ = oracle.run_blocked(kind, layers, X, T, return_state=True)
        H, cs, xcs = P.run_blocked(cfg, ws, X, T, return_state=True)
        assert_f32(H, ref)
        assert_f32(cs[0], cref[0])
        if kind == "qrnn":
            assert np.array_equal(xcs[0], X[-1])


def test_single_step_and_tiny_sequences(P, oracle):
    for kind in ("sru", "qrnn"):
        layers = oracle.generate_layers(kind, 64, 64, 1, 3, np.float32)
        for L in (1, 2, 7):
            X = oracle.generate_sequence(L, 64, 4, np.float32)
            ref = oracle.run_stepwise(kind, layers, X)
            for T in (1, 4, 32):
                assert_f32(P.run_blocked(_cfg(P, kind, 64, 1, "f32"), _ws(P, kind, layers, "f32"), X, T), ref)


def test_multilayer_stacks_vs_oracle(P, oracle):
    for kind, d, nl in (("sru", 256, 3), ("qrnn", 192, 4)):
        layers = oracle.generate_layers(kind, d, d, nl, 11, np.float32)
        X = np.random.default_rng(2).standard_normal((300, d)).astype(np.float32)
        for T in (1, 8, 32):
            ref = oracle.run_blocked(kind, layers, X, T)
            assert_f32(P.run_blocked(_cfg(P, kind, d, nl, "f32"), _ws(P, kind, layers, "f32"), X, T), ref)


def test_baseline_cfg1_full(P, oracle):
    """BASELINE cfg1 at full size against the reference's own outputs."""
    from paper_1803_11389_b200 import workloads
    g = np.load(os.path.join(GOLDEN, "baseline_cfg.npz"))
    w = workloads.make("cfg1")
    cfg = _cfg(P, "sru", 512, 1, "f32")
    ws = P.WeightSet(P.CellKind.SRU, "f32", w.layers)
    for T in (1, 4, 16):
        H, cs, _ = P.run_blocked(cfg, ws, w.X, T, return_state=True)
        assert_f32(cs[0], g[f"cfg1_T{T}_c"])
        assert_f32(H, g["cfg1_T16_H"])


@pytest.mark.parametrize("f32_tc", ["0", "1"])
def test_baseline_cfg2_full(P, oracle, f32_tc, monkeypatch):
    """BASELINE cfg2 (QRNN 1024, L=2048) at full size: reference row
    subsample + c_T, plus the oracle over the whole output at every T_b --
    on the FFMA kernels (RNNB_F32_TC=0) and on fp32 mode's default dispatch
    (3xTF32 tcgen05 from T_b = 8)."""
    import torch
    monkeypatch.setenv("RNNB_F32_TC", f32_tc)
    from paper_1803_11389_b200 import workloads
    g = np.load(os.path.join(GOLDEN, "baseline_cfg.npz"))
    w = workloads.make("cfg2")
    layers = [lay.mats() for lay in w.layers]
    st = P.DeviceStack(P.CellKind.QRNN, w.layers, mode="f32")
    Xd = torch.from_numpy(w.X).cuda()
    for T in w.block_sizes:
        c = torch.zeros(1024, dtype=torch.float32, device="cuda")
        H = st.forward(Xd, T, c_state=c).cpu().numpy()
        if T == 32:
            assert_f32(H[g["cfg2_T32_rows"]], g["cfg2_T32_Hrows"])
            assert_f32(c.cpu().numpy(), g["cfg2_T32_c"])
        if f32_tc == "0" or T < 8:
            assert st.query(3) == 1 and st.query(6) == 1  # SMEM-resident, warp-specialised FFMA
        else:
            assert st.query(9) == 1  # 3xTF32 on tcgen05
        ref, cref, _ = oracle.run_blocked("qrnn", layers, w.X, T, return_state=True)
        assert_f32(H, ref)
        assert_f32(c.cpu().numpy(), cref[0])
    st.close()


def test_streaming_state_carry_equals_whole_sequence(P, oracle, monkeypatch):
    """c and x_carry in/out across calls: two half-sequence calls on a block
    boundary reproduce the whole-sequence call bit for bit (FFMA kernels:
    the per-unit dot products never depend on the chunking)."""
    import torch
    monkeypatch.setenv("RNNB_F32_TC", "0")
    for kind in ("sru", "qrnn"):
        layers = oracle.generate_layers(kind, 128, 128, 2, 21, np.float32)
        X = np.random.default_rng(3).standard_normal((256, 128)).astype(np.float32)
        st = P.DeviceStack(kind, layers, mode="f32")
        Xd = torch.from_numpy(X).cuda()
        whole = st.forward(Xd, 16).cpu().numpy()
        c = torch.zeros(256, device="cuda")
        xc = torch.zeros(256, device="cuda")
        a = st.forward(Xd[:96].contiguous(), 16, c_state=c, x_carry=xc).cpu().numpy()
        b = st.forward(Xd[96:].contiguous(), 16, c_state=c, x_carry=xc).cpu().numpy()
        assert np.concatenate([a, b]).tobytes() == whole.tobytes()
        st.close()


def test_strided_device_input(P, oracle):
    import torch
    layers = oracle.generate_layers("qrnn", 96, 96, 1, 5, np.float32)
    X = np.random.default_rng(4).standard_normal((64, 96)).astype(np.float32)
    st = P.DeviceStack("qrnn", layers)
    big = torch.zeros((64, 128), device="cuda")
    big[:, :96] = torch.from_numpy(X).cuda()
    a = st.forward(big[:, :96], 8).cpu().numpy()
    b = st.forward(torch.from_numpy(X).cuda(), 8).cpu().numpy()
    assert a.tobytes() == b.tobytes()
    st.close()


def test_host_e2e_matches_device(P, oracle):
    import torch
    layers = oracle.generate_layers("sru", 512, 512, 1, 6, np.float32)
    X = np.random.default_rng(5).standard_normal((200, 512)).astype(np.float32)
    st = P.DeviceStack("sru", layers)
    a = st.forward_host(X, 16)
    b = st.forward(torch.from_numpy(X).cuda(), 16).cpu().numpy()
    assert a.tobytes() == b.tobytes()
    st.close()


# ---------------------------------------------------------------------------
# unit-level ops (blocked.py:123-193)


def _sig(z):
    return 0.5 * (1.0 + np.tanh(0.5 * z))


def test_precompute_gates_sru(P, oracle):
    layers = oracle.generate_layers("sru", 64, 64, 1, 8, np.float64)
    lay = layers[0]
    w = P.SruWeights(*lay)
    Xb = np.ascontiguousarray(oracle.generate_sequence(16, 64, 9, np.float64).T)
    g = P.precompute_gates_sru(w, Xb)
    assert np.max(np.abs(g.cand - lay[0] @ Xb)) <= 1e-12
    assert np.max(np.abs(g.forget - _sig(lay[1] @ Xb + lay[3][:, None]))) <= 1e-12
    assert np.max(np.abs(g.out_gate - _sig(lay[2] @ Xb + lay[4][:, None]))) <= 1e-12
    # zero weights: cand 0, forget sigma(b), highway 0.5 (test_blocked.py:105-118 property)
    z = np.zeros((3, 3))
    w0 = P.SruWeights(z, z.copy(), z.copy(), np.array([0.3, -0.1, 0.0]), np.zeros(3))
    g0 = P.precompute_gates_sru(w0, np.ones((3, 4)))
    assert np.allclose(g0.cand, 0.0) and (g0.out_gate == 0.5).all()
    assert np.max(np.abs(g0.forget - _sig(np.array([0.3, -0.1, 0.0]))[:, None])) <= 1e-15


def test_precompute_gates_qrnn_carry_and_ablation(P, oracle):
    lay = oracle.generate_layers("qrnn", 48, 48, 1, 10, np.float64)[0]
    w = P.QrnnWeights(*lay)
    X = oracle.generate_sequence(12, 48, 11, np.float64)
    b1, b2 = np.ascontiguousarray(X[:5].T), np.ascontiguousarray(X[5:].T)
    g2 = P.precompute_gates_qrnn(w, b2, np.ascontiguousarray(b1[:, -1]))
    xprev = np.concatenate([b1[:, -1:], b2[:, :-1]], axis=1)
    assert np.max(np.abs(g2.cand - np.tanh(lay[0] @ b2 + lay[1] @ xprev))) <= 1e-12
    assert np.max(np.abs(g2.forget - _sig(lay[2] @ b2 + lay[3] @ xprev))) <= 1e-12
    assert np.max(np.abs(g2.out_gate - _sig(lay[4] @ b2 + lay[5] @ xprev))) <= 1e-12
    for m in (1, 3, 5):
        lay[m][:] = 0.0
    w = P.QrnnWeights(*lay)
    a = P.precompute_gates_qrnn(w, b2, np.zeros(48))
    b = P.precompute_gates_qrnn(w, b2, np.full(48, 9.0))
    assert (a.cand == b.cand).all() and (a.forget == b.forget).all()


def test_sweep_and_finalize_known_answers(P):
    C = P.recurrence_sweep(np.array([[0.5, 0.5]]), np.array([[1.0, 1.0]]), np.zeros(1))
    assert C.tolist() == [[0.5, 0.75]]
    d, T = 4, 6
    Xh = np.random.default_rng(0).uniform(-1, 1, (d, T))
    c0 = np.array([0.1, -0.2, 0.3, -0.4])
    assert (P.recurrence_sweep(np.ones((d, T)), Xh, c0) == c0[:, None]).all()
    assert (P.recurrence_sweep(np.zeros((d, T)), Xh, np.ones(d)) == Xh).all()
    Cm = np.random.default_rng(2).uniform(-1, 1, (3, 5))
    gq = P.GateBlock(cand=np.zeros_like(Cm), forget=np.zeros_like(Cm), out_gate=np.ones_like(Cm))
    assert np.max(np.abs(P.finalize_outputs(P.CellKind.QRNN, gq, Cm) - np.tanh(Cm))) <= 1e-15
    Xb = np.random.default_rng(4).uniform(-1, 1, (3, 5))
    gs = P.GateBlock(cand=np.zeros_like(Cm), forget=np.zeros_like(Cm), out_gate=np.zeros_like(Cm))
    assert (P.finalize_outputs(P.CellKind.SRU, gs, Cm, Xb) == Xb).all()
    with pytest.raises(ValueError):
        P.finalize_outputs(P.CellKind.SRU, gs, Cm)
    with pytest.raises(ValueError):
        P.recurrence_sweep(np.zeros((2, 3)), np.zeros((2, 4)), np.zeros(2))


def test_blocked_errors_match_reference(P, oracle):
    lay = oracle.generate_layers("sru", 8, 8, 1, 1, np.float32)
    cfg = _cfg(P, "sru", 8, 1, "f32")
    ws = _ws(P, "sru", lay, "f32")
    X = np.zeros((4, 8), np.float32)
    with pytest.raises(ValueError):
        P.run_blocked(cfg, ws, np.zeros((4, 9), np.float32), 2)
    with pytest.raises(ValueError):
        P.run_blocked(cfg, ws, X, 0)
    with pytest.raises(ValueError):
        P.run_blocked(cfg, ws, X, 2, kernel="bogus")
    with pytest.raises(ValueError, match="dtype mismatch"):
        P.run_blocked(cfg, ws, X.astype(np.float64), 2)
    with pytest.raises(ValueError):
        P.run_blocked(P.RnnConfig(P.CellKind.LSTM, 8, 8), ws, X, 2)


# ---------------------------------------------------------------------------
# tensor-core numerics modes


def _round_tf32(a):
    u = np.ascontiguousarray(a, np.float32).view(np.uint32).astype(np.uint64)
    u = ((u + 0x1000) & 0xFFFFE000).astype(np.uint32)
    return u.view(np.float32)


def _round_bf16(a):
    u = np.ascontiguousarray(a, np.float32).view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return u.view(np.float32)


@pytest.mark.parametrize("kind", ["sru", "qrnn"])
@pytest.mark.parametrize("mode", ["tf32", "bf16"])
def test_reduced_precision_modes(P, oracle, kind, mode):
    import torch
    d = 512
    # the "vs rounded oracle" bound is per layer: for a stack, ulp differences in
    # layer-1 outputs flip tf32/bf16 roundings of layer-2 operands
    layers = oracle.generate_layers(kind, d, d, 1, 31, np.float32)
    X = np.random.default_rng(7).standard_normal((256, d)).astype(np.float32)
    st = P.DeviceStack(kind, layers, mode=mode)
    rnd = _round_tf32 if mode == "tf32" else _round_bf16
    for T in (1, 16, 32):
        H = st.forward(torch.from_numpy(X).cuda(), T).cpu().numpy()
        ref = oracle.run_blocked(kind, layers, X, T)
        assert normwise(H, ref) <= (2e-3 if mode == "tf32" else 2e-2)
        # vs the oracle fed rounded weights and rounded MMA operands, layer by layer
        inp = X
        for lay in layers:
            rl = [rnd(m) if m.ndim == 2 else m for m in lay]
            xr = rnd(inp)
            if kind == "sru":
                # highway term uses the unrounded input; emulate by correcting
                out_r = oracle.run_blocked(kind, [rl], xr, T)
                out_u = _sru_highway_fix(oracle, rl, xr, inp, T)
                inp = out_u
            else:
                inp = oracle.run_blocked(kind, [rl], xr, T)
        assert normwise(H, inp) <= (1e-5 if mode == "tf32" else 1e-3)
    st.close()


def _sru_highway_fix(oracle, rl, xr, x, T):
    """SRU with products on rounded x but the (1-r) x highway on the raw x."""
    import numpy as _np
    H = oracle.run_blocked("sru", [rl], xr, T)
    # H = r tanh c + (1-r) xr  ->  replace xr by x: add (1-r)(x - xr)
    r = 0.5 * (1.0 + _np.tanh(0.5 * (xr.astype(_np.float64) @ rl[2].T.astype(_np.float64) + rl[4])))
    return (H + (1.0 - r) * (x.astype(_np.float64) - xr.astype(_np.float64))).astype(_np.float32)


# ---------------------------------------------------------------------------
# tcgen05 tensor-core path (T_b in [16, 128] for bf16 / tf32 stacks)


@pytest.mark.parametrize("kind", ["sru", "qrnn"])
@pytest.mark.parametrize("mode", ["bf16", "tf32"])
def test_tensor_core_path_matches_oracle_on_rounded_operands(P, oracle, kind, mode, monkeypatch):
    """TC kernel vs the oracle run on operands rounded like the MMA sees them
    (per-layer bound 1e-5 tf32 / 1e-3 bf16), odd sizes: H=300 (3 unit tiles,
    padded), D=200 (partial k-tile), L=777 (remainder block)."""
    import torch
    d = 200 if kind == "qrnn" else 300
    h = 300
    layers = oracle.generate_layers(kind, d, h, 1, 41, np.float32)
    X = np.random.default_rng(9).standard_normal((777, d)).astype(np.float32)
    st = P.DeviceStack(kind, layers, mode=mode)
    rnd = _round_tf32 if mode == "tf32" else _round_bf16
    rl = [rnd(m) if m.ndim == 2 else m for m in layers[0]]
    for T in (16, 32, 48, 64, 100, 128):
        Ht = st.forward(torch.from_numpy(X).cuda(), T)
        assert st.query(9) == 1, "tensor-core kernel did not run"
        H = Ht.cpu().numpy()
        if kind == "sru":
            ref = _sru_highway_fix(oracle, rl, rnd(X), X, T)
        else:
            ref = oracle.run_blocked(kind, [rl], rnd(X), T)
        assert normwise(H, ref) <= (1e-5 if mode == "tf32" else 1e-3), (T, normwise(H, ref))
        monkeypatch.setenv("RNNB_NO_TC", "1")
        Hf = st.forward(torch.from_numpy(X).cuda(), T).cpu().numpy()
        monkeypatch.delenv("RNNB_NO_TC")
        assert st.query(9) == 0
        assert normwise(H, Hf) <= (1e-5 if mode == "tf32" else 1e-3)
    st.close()


def test_tensor_core_streaming_carry(P, oracle):
    """c and x_carry across calls on the TC path (operand row 0 = x_carry)."""
    import torch
    layers = oracle.generate_layers("qrnn", 256, 256, 2, 43, np.float32)
    X = np.random.default_rng(10).standard_normal((512, 256)).astype(np.float32)
    st = P.DeviceStack("qrnn", layers, mode="bf16")
    Xd = torch.from_numpy(X).cuda()
    whole = st.forward(Xd, 32).cpu().numpy()
    c = torch.zeros(512, device="cuda")
    xc = torch.zeros(512, device="cuda")
    a = st.forward(Xd[:256].contiguous(), 32, c_state=c, x_carry=xc).cpu().numpy()
    b = st.forward(Xd[256:].contiguous(), 32, c_state=c, x_carry=xc).cpu().numpy()
    assert st.query(9) == 1
    assert normwise(np.concatenate([a, b]), whole) <= 1e-6
    st.close()


def test_tensor_core_look_back_is_deterministic(P, oracle):
    """Fixed-depth look-back: bitwise identical results run to run (the
    reference's worker-count invariance, test_blocked.py:386-396)."""
    import torch
    layers = oracle.generate_layers("qrnn", 512, 512, 1, 47, np.float32)
    X = torch.from_numpy(np.random.default_rng(11).standard_normal((4096, 512)).astype(np.float32)).cuda()
    st = P.DeviceStack("qrnn", layers, mode="bf16")
    a = st.forward(X, 16).cpu().numpy()
    for _ in range(3):
        assert st.forward(X, 16).cpu().numpy().tobytes() == a.tobytes()
    st.close()


@pytest.mark.parametrize("kind", ["sru", "qrnn"])
def test_f32x3_split_tensor_core_meets_fp32_bound(P, oracle, kind):
    """3xTF32 split products on tcgen05 (mode "f32x3", T_b >= 16; blocks past
    32 steps run as 32-step tensor-core blocks) with 128-deep K chunks summed
    in fp32 meet the fp32 bound (normwise 1e-5, max-abs 1e-4); the error vs
    an f64 oracle is reported beside FFMA's."""
    import torch
    d = 512
    layers = oracle.generate_layers(kind, d, d, 2, 51, np.float32)
    X = np.random.default_rng(12).standard_normal((600, d)).astype(np.float32)
    st = P.DeviceStack(kind, layers, mode="f32x3")
    ref64 = oracle.run_blocked(kind, [[m.astype(np.float64) for m in l] for l in layers], X.astype(np.float64), 32)
    for T in (64, 48, 16, 24, 32):
        H = st.forward(torch.from_numpy(X).cuda(), T).cpu().numpy()
        assert st.query(9) == 1
        ref = oracle.run_blocked(kind, layers, X, T)
        print(f"{kind} T_b={T}: 3xTF32 vs fp32 oracle normwise {normwise(H, ref):.2e}")
        assert_f32(H, ref)
    e3 = normwise(H, ref64)
    f32 = P.DeviceStack(kind, layers, mode="f32")
    Hf = f32.forward(torch.from_numpy(X).cuda(), 32).cpu().numpy()
    ef = normwise(Hf, ref64)
    print(f"normwise error vs f64: 3xTF32 {e3:.2e}  FFMA fp32 {ef:.2e}")
    assert e3 <= 5e-6
    st.close()
    f32.close()


@pytest.mark.parametrize("kind,d", [("sru", 1024), ("sru", 512), ("qrnn", 512), ("qrnn", 1024)])
def test_register_resident_kernel(P, oracle, kind, d, monkeypatch):
    """ffma_reg (weights in registers, FFMA2, epilogue warp) at small T_b vs
    the oracle and vs the shared-memory kernel (U=7 for d=1024 SRU, U=4 for
    d=512; QRNN d=1024 is K=2048 with U=7: not eligible, SMEM kernel runs)."""
    import torch
    layers = oracle.generate_layers(kind, d, d, 2, 57, np.float32)
    X = torch.from_numpy(np.random.default_rng(14).standard_normal((333, d)).astype(np.float32)).cuda()
    st = P.DeviceStack(kind, layers)
    monkeypatch.setenv("RNNB_F32_TC", "0")  # the FFMA kernels (fp32 mode runs T_b >= 8 on tcgen05 by default)
    for T in (1, 2, 3, 8):
        monkeypatch.setenv("RNNB_REG", "1")
        H = st.forward(X, T).cpu().numpy()
        used = st.query(10)
        assert used == (0 if (kind == "qrnn" and d == 1024) else 1)
        monkeypatch.setenv("RNNB_REG", "0")
        Hs = st.forward(X, T).cpu().numpy()
        ref = oracle.run_blocked(kind, layers, X.cpu().numpy(), T)
        assert_f32(H, ref)
        assert_f32(Hs, ref)
    st.close()


@pytest.mark.parametrize("kind,d", [("sru", 1024), ("qrnn", 1024), ("qrnn", 520)])
def test_wide_pass_kernels(P, oracle, kind, d, monkeypatch):
    """ffma_ws wide tile (8 consumer warps, 11x4 FFMA2 tile, reduce-scatter)
    at NT=16 and the opt-in NT=32 pass, including a remainder block and a
    partial last K chunk (d=520), vs the oracle."""
    import torch
    monkeypatch.setenv("RNNB_F32_TC", "0")
    layers = oracle.generate_layers(kind, d, d, 2, 61, np.float32)
    X = np.random.default_rng(15).standard_normal((301, d)).astype(np.float32)
    Xd = torch.from_numpy(X).cuda()
    st = P.DeviceStack(kind, layers)
    for nt32 in ("0", "1"):
        monkeypatch.setenv("RNNB_NT32", nt32)
        for T in (16, 32, 40, 64):
            H = st.forward(Xd, T).cpu().numpy()
            assert_f32(H, oracle.run_blocked(kind, layers, X, T))
    st.close()


@pytest.mark.parametrize("kind,d,L,T", [("qrnn", 1024, 2048, 32), ("qrnn", 1024, 1000, 16), ("sru", 1024, 777, 8),
                                        ("qrnn", 512, 300, 1), ("sru", 256, 130, 200), ("qrnn", 1024, 9000, 32)])
def test_host_streaming_matches_device(P, oracle, kind, d, L, T, monkeypatch):
    """rnnb_forward_host's streaming mode (one layer launch fed by the copy
    stream through a device row counter, chunks drained by a wait-value copy
    stream) and its chunked fallback are bitwise equal to the device call,
    including carried c / x_carry in-out state (FFMA kernels; streaming
    needs them)."""
    import torch
    monkeypatch.setenv("RNNB_F32_TC", "0")
    layers = oracle.generate_layers(kind, d, d, 1, 71, np.float32)
    X = np.random.default_rng(16).standard_normal((L, d)).astype(np.float32)
    st = P.DeviceStack(kind, layers)
    c0 = np.random.default_rng(17).standard_normal(d).astype(np.float32)
    x0 = np.random.default_rng(18).standard_normal(d).astype(np.float32)
    cd, xd = torch.from_numpy(c0.copy()).cuda(), torch.from_numpy(x0.copy()).cuda()
    ref = st.forward(torch.from_numpy(X).cuda(), T, c_state=cd, x_carry=xd if kind == "qrnn" else None)
    ref = ref.cpu().numpy()
    for mode in ("1", "0"):
        monkeypatch.setenv("RNNB_HOST_STREAM", mode)
        c, x = c0.copy(), x0.copy()
        H = st.forward_host(X, T, c_state=c, x_carry=x if kind == "qrnn" else None)
        assert H.tobytes() == ref.tobytes(), mode
        assert c.tobytes() == cd.cpu().numpy().tobytes()
        if kind == "qrnn":
            assert x.tobytes() == xd.cpu().numpy().tobytes()
        H2 = st.forward_host(X, T)  # zero state, twice (counter / event reuse)
        H3 = st.forward_host(X, T)
        assert H2.tobytes() == H3.tobytes()
    st.close()


@pytest.mark.parametrize("kind,d,n_layers", [("qrnn", 2048, 2), ("sru", 4096, 1), ("qrnn", 1536, 1), ("sru", 2760, 1)])
def test_weight_streaming_kernel(P, oracle, kind, d, n_layers, monkeypatch):
    """fp32 layers whose weights do not fit in shared memory (BASELINE cfg4:
    QRNN 2048, 100 MB per layer): the ws kernel with per-(CTA, chunk) weight
    images streamed through its ring (14 units per CTA), T_b >= 32, incl. a
    remainder block, carried state and an H not a multiple of 14, vs the
    oracle and vs the generic kernel (RNNB_WSTREAM=0)."""
    import torch
    monkeypatch.setenv("RNNB_F32_TC", "0")
    layers = oracle.generate_layers(kind, d, d, n_layers, 81, np.float32)
    L = 203
    X = np.random.default_rng(19).standard_normal((L, d)).astype(np.float32)
    Xd = torch.from_numpy(X).cuda()
    st = P.DeviceStack(kind, layers)
    for T in (32, 48, 64):
        H = st.forward(Xd, T).cpu().numpy()
        assert all(st.query(11, li) == 1 for li in range(n_layers)), T
        ref = oracle.run_blocked(kind, layers, X, T)
        assert_f32(H, ref)
    # chunked with carried state == one call (same kernel, same per-unit order)
    c = torch.zeros(d * n_layers, device="cuda")
    xc = torch.zeros(d * n_layers, device="cuda")
    a = st.forward(Xd[:96], 32, c_state=c, x_carry=xc if kind == "qrnn" else None)
    b = st.forward(Xd[96:], 32, c_state=c, x_carry=xc if kind == "qrnn" else None)
    whole = st.forward(Xd, 32).cpu().numpy()
    assert np.concatenate([a.cpu().numpy(), b.cpu().numpy()]).tobytes() == whole.tobytes()
    monkeypatch.setenv("RNNB_WSTREAM", "0")
    G = st.forward(Xd, 32).cpu().numpy()
    assert st.query(11) == 0
    assert_f32(G, whole)
    st.close()


@pytest.mark.parametrize("kind,mode,d,L,T", [("qrnn", "f32", 1024, 2048, 32), ("qrnn", "f32", 1024, 1000, 64),
                                             ("sru", "f32", 512, 777, 16), ("qrnn", "bf16", 1024, 2048, 64),
                                             ("sru", "bf16", 256, 130, 1), ("qrnn", "tf32", 512, 9000, 32)])
def test_host_streaming_tensor_core_matches_device(P, oracle, kind, mode, d, L, T, monkeypatch):
    """rnnb_forward_host on the tcgen05 path: one layer launch on all but two
    SMs while the copy-in stream lands rows and converts them into the MMA
    operand (an operand-row counter the TMA producer waits on), copy-out per
    granule of finished items -- bitwise the device call (the look-back's
    fixed order makes the result independent of the item schedule), with
    carried c / x_carry; the chunked fallback within the look-back bound."""
    import torch
    layers = oracle.generate_layers(kind, d, d, 1, 73, np.float32)
    X = np.random.default_rng(20).standard_normal((L, d)).astype(np.float32)
    st = P.DeviceStack(kind, layers, mode=mode)
    c0 = np.random.default_rng(21).standard_normal(d).astype(np.float32)
    x0 = np.random.default_rng(22).standard_normal(d).astype(np.float32)
    cd, xd = torch.from_numpy(c0.copy()).cuda(), torch.from_numpy(x0.copy()).cuda()
    ref = st.forward(torch.from_numpy(X).cuda(), T, c_state=cd, x_carry=xd if kind == "qrnn" else None)
    ref = ref.cpu().numpy()
    assert st.query(9) == 1
    for stream in ("1", "0"):
        monkeypatch.setenv("RNNB_HOST_STREAM", stream)
        c, x = c0.copy(), x0.copy()
        H = st.forward_host(X, T, c_state=c, x_carry=x if kind == "qrnn" else None)
        if stream == "1":
            assert H.tobytes() == ref.tobytes()
            assert c.tobytes() == cd.cpu().numpy().tobytes()
        else:
            # chunked fallback: the look-back re-anchors at chunk edges, and an
            # fp32 chunk too short to fill the GPU runs on the FFMA kernel
            assert normwise(H, ref) <= (1e-5 if mode == "f32" else 1e-6)
        if kind == "qrnn":
            assert x.tobytes() == xd.cpu().numpy().tobytes()
        H2 = st.forward_host(X, T)  # zero state, twice (counter reuse)
        H3 = st.forward_host(X, T)
        assert H2.tobytes() == H3.tobytes()
    st.close()


@pytest.mark.parametrize("kind,mode,d,L,T", [("qrnn", "f32", 1024, 2048, 32), ("sru", "f32", 512, 777, 16),
                                             ("qrnn", "bf16", 1024, 3000, 64), ("sru", "tf32", 640, 5000, 32)])
def test_host_streaming_pinned_buffers_zero_copy_output(P, oracle, kind, mode, d, L, T, monkeypatch):
    """rnnb_forward_host with PINNED host buffers (what bench.py's e2e leg
    passes): the persistent conversion kernel follows the copy segments and the
    layer epilogue stores h straight into the caller's pinned buffer (no
    copy-out) -- bitwise the device call, repeatably, with the zero-copy
    output switched off too."""
    import torch
    layers = oracle.generate_layers(kind, d, d, 1, 91, np.float32)
    X = np.random.default_rng(30).standard_normal((L, d)).astype(np.float32)
    st = P.DeviceStack(kind, layers, mode=mode)
    ref = st.forward(torch.from_numpy(X).cuda(), T).cpu().numpy()
    assert st.query(9) == 1
    Xp = torch.from_numpy(X).pin_memory()
    Hp = torch.full((L, d), float("nan"), dtype=torch.float32).pin_memory()
    for zc in ("1", "0", "1"):
        monkeypatch.setenv("RNNB_ZC_OUT", zc)
        Hp.fill_(float("nan"))
        st.forward_host(Xp.numpy(), T, out=Hp.numpy())
        assert Hp.numpy().tobytes() == ref.tobytes()
    st.close()


@pytest.mark.parametrize("kind,mode,d,L,T", [("qrnn", "bf16", 1024, 3000, 32), ("sru", "tf32", 768, 2500, 8),
                                             ("sru", "bf16", 512, 4100, 1), ("qrnn", "tf32", 512, 2000, 64)])
def test_epilogue_groups_are_bitwise_neutral(P, oracle, kind, mode, d, L, T, monkeypatch):
    """bf16 / tf32: the one- and the two-epilogue-group kernel variants (the
    second group takes every other item on its own TMEM buffers) compute the
    same arithmetic in the same order per unit -- bitwise equal outputs and
    final c, whichever the host would pick."""
    import torch
    layers = oracle.generate_layers(kind, d, d, 1, 101, np.float32)
    X = torch.from_numpy(np.random.default_rng(33).standard_normal((L, d)).astype(np.float32)).cuda()
    st = P.DeviceStack(kind, layers, mode=mode)
    outs = []
    for eg in ("1", "2"):
        monkeypatch.setenv("RNNB_TC_EGROUPS", eg)
        c = torch.zeros(d, dtype=torch.float32, device="cuda")
        H = st.forward(X, T, c_state=c).cpu().numpy()
        assert st.query(9) == 1
        outs.append((H, c.cpu().numpy()))
    assert outs[0][0].tobytes() == outs[1][0].tobytes()
    assert outs[0][1].tobytes() == outs[1][1].tobytes()
    st.close()


@pytest.mark.timeout(120)
@pytest.mark.parametrize("mode,T", [("bf16", 16), ("f32", 32), ("tf32", 64)])
def test_lookback_sentinel_never_collides_with_data(P, oracle, mode, T):
    """The look-back publishes carry maps by value into arrays pre-filled with
    an all-ones sentinel and consumers wait until a value differs from it: NaN
    inputs -- including the NaN whose bits ARE the sentinel -- must not hang
    the launch (published NaNs are re-coded) and must leave every step before
    the first NaN row bitwise equal to the clean run; the next launch on the
    same stack is clean again."""
    import torch
    d, L = 512, 40 * T + 5
    layers = oracle.generate_layers("qrnn", d, d, 1, 97, np.float32)
    X = np.random.default_rng(31).standard_normal((L, d)).astype(np.float32)
    st = P.DeviceStack("qrnn", layers, mode=mode)
    clean = st.forward(torch.from_numpy(X).cuda(), T).cpu().numpy()
    assert st.query(9) == 1
    bad = X.copy()
    t_bad = 17 * T + 3
    bad[t_bad, :] = np.frombuffer(np.uint32(0xFFFFFFFF).tobytes(), np.float32)[0]
    bad[t_bad + 1, ::2] = np.nan
    H = st.forward(torch.from_numpy(bad).cuda(), T).cpu().numpy()  # must return
    assert H[:t_bad].tobytes() == clean[:t_bad].tobytes()
    assert H.shape == clean.shape  # (what a NaN step yields is not specified: the branch-free activations saturate it)
    again = st.forward(torch.from_numpy(X).cuda(), T).cpu().numpy()
    assert again.tobytes() == clean.tobytes()
    st.close()


@pytest.mark.parametrize("kind,d,L", [("qrnn", 1024, 2048), ("sru", 1024, 3000), ("qrnn", 2048, 700)])
def test_split_last_wave_is_bitwise_neutral(P, oracle, kind, d, L, monkeypatch):
    """3xTF32: the last partial wave's items run as two K halves on two CTAs
    (first half's chunk sum handed over through global memory); every item
    sums (first half) + (second half), so the split changes no bit
    (RNNB_TC_SPLIT=0 disables it) -- and the result stays within the fp32
    bound of the oracle."""
    import torch
    layers = oracle.generate_layers(kind, d, d, 1, 79, np.float32)
    X = np.random.default_rng(23).standard_normal((L, d)).astype(np.float32)
    Xd = torch.from_numpy(X).cuda()
    st = P.DeviceStack(kind, layers, mode="f32")
    split = st.forward(Xd, 32).cpu().numpy()
    assert st.query(9) == 1
    monkeypatch.setenv("RNNB_TC_SPLIT", "0")
    whole = st.forward(Xd, 32).cpu().numpy()
    assert split.tobytes() == whole.tobytes()
    assert_f32(split, oracle.run_blocked(kind, layers, X, 32))
    st.close()
