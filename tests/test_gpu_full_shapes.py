"""GPU parity at the BASELINE.json configurations' real shapes (VERDICT r1
"next" #1), against the CPU oracle (oracle/, pinned to the reference).

* cfg2 (QRNN 1024, L=2048): every tensor-core mode at every T_b.
* cfg3 (projection 120->1024, 6 x SRU-1024, logits 1024->2000, L=4096):
  f32 / bf16 / tf32 at T_b in {1, 8, 32}; the projection and the logits
  against the oracle's gemm; per-layer rounded-operand bounds.
* cfg4 (8 x QRNN-2048, L=65536, T_b=32): all 8 layers on an 8192-step
  prefix in f32 (weight-streaming FFMA), bf16 and f32x3 with every layer's
  c_T; the full 65536-step sequence through a split-at-a-block-boundary
  window whose last 1024 steps are re-run on the oracle from the GPU's
  carried state (c, x_carry) of every layer.
* cfg5 (bidirectional wide SRU, H=4096/dir, L=8192, bf16, T_b in {16, 64}):
  layer 1 of each direction vs the oracle's run_blocked(X) /
  run_blocked(X[::-1])[::-1] (the reference's SRU is square,
  cells.py:89), layers 2-4 vs a float64 restatement of the cell on a
  256-step prefix (forward) / suffix (backward) of the GPU's own layer
  input, and the fused sharded product path (p2p.P2PBidirSRU) vs that
  per-layer composition.

The oracle is computed once per configuration at T_b=32 (its values do not
depend on the block size beyond rounding: blocked.py's "one weight fetch
per block" never reorders a dot product) and every GPU T_b is compared with
it.  Reference call sites: /root/reference/pkg/src/rnnblock/blocked.py:221-268.
"""

import numpy as np
import pytest

from parity_util import (BOUND_VS_F32, BOUND_VS_ROUNDED, ROUND, assert_f32, normwise, rounded_layer,
                         sru_wide_f64)

pytestmark = pytest.mark.gpu

ERRORS = {}  # measured errors, printed at the end (pytest -s) for DESIGN.md


def _record(key, v):
    ERRORS[key] = v
    print(f"[parity] {key}: {v:.3e}")


@pytest.fixture(scope="module")
def P():
    import paper_1803_11389_b200 as P
    return P


def _cuda(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


# ---------------------------------------------------------------------------
# cfg2


@pytest.fixture(scope="module")
def cfg2(oracle):
    from paper_1803_11389_b200 import workloads
    w = workloads.make("cfg2")
    mats = w.layers[0].mats()
    ref = oracle.run_blocked("qrnn", [mats], w.X, 32)
    return w, mats, ref


@pytest.mark.parametrize("mode", ["bf16", "tf32", "f32x3"])
def test_cfg2_tensor_modes_full_size_every_block_size(P, oracle, cfg2, mode):
    w, mats, ref = cfg2
    st = P.DeviceStack("qrnn", w.layers, mode=mode)
    Xd = _cuda(w.X)
    rref = None if mode == "f32x3" else rounded_layer(oracle, "qrnn", mats, w.X, 32, mode)[0]
    for T in w.block_sizes:
        H = st.forward(Xd, T).cpu().numpy()
        if mode == "f32x3":
            _record(f"cfg2 f32x3 T_b={T} vs fp32 oracle", assert_f32(H, ref, T))
            if T >= 16:
                assert st.query(9) == 1, "3xTF32 tensor-core kernel did not run"
            continue
        e32, er = normwise(H, ref), normwise(H, rref)
        _record(f"cfg2 {mode} T_b={T} vs fp32 oracle", e32)
        _record(f"cfg2 {mode} T_b={T} vs rounded-operand oracle", er)
        assert e32 <= BOUND_VS_F32[mode], (T, e32)
        assert er <= BOUND_VS_ROUNDED[mode], (T, er)
    st.close()


# ---------------------------------------------------------------------------
# cfg3


@pytest.fixture(scope="module")
def cfg3(oracle):
    from paper_1803_11389_b200 import workloads
    w = workloads.make("cfg3")
    mats = [lay.mats() for lay in w.layers]
    # oracle: projection gemm, 6 blocked SRU layers, logits gemm (kernels.py:203-225)
    h0 = oracle.gemm(w.proj, np.ascontiguousarray(w.X.T), kernel="fast").T.copy()
    hs = [h0]
    for m in mats:
        hs.append(oracle.layer_blocked("sru", m, hs[-1], 32)[0])
    logits = oracle.gemm(w.logits, np.ascontiguousarray(hs[-1].T), kernel="fast").T.copy()
    return w, mats, hs, logits


@pytest.mark.parametrize("mode", ["f32", "bf16", "tf32"])
def test_cfg3_acoustic_full_length(P, oracle, cfg3, mode):
    """Whole model at L=4096, T_b in {1, 8, 32} vs the fp32 oracle chain; the
    projection and logits kernels vs the oracle gemm on the same inputs."""
    from paper_1803_11389_b200.acoustic import AcousticSRU
    w, mats, hs, logits = cfg3
    m = AcousticSRU(w.proj, w.layers, w.logits, mode=mode)
    frames = _cuda(w.X)
    # projection alone (on the same frames as the oracle)
    h0 = m.project(frames).cpu().numpy()
    e = normwise(h0, hs[0])
    _record(f"cfg3 {mode} projection vs oracle gemm", e)
    if mode == "f32":
        assert_f32(h0, hs[0])
    else:
        rnd = ROUND[mode]
        assert normwise(h0, rnd(w.X).astype(np.float64) @ rnd(w.proj).T.astype(np.float64)) <= 1e-5
        assert e <= BOUND_VS_F32[mode]
    # logits alone, fed the oracle's final hidden state
    lg = m.classify(_cuda(hs[-1])).cpu().numpy()
    e = normwise(lg, logits)
    _record(f"cfg3 {mode} logits vs oracle gemm", e)
    if mode == "f32":
        assert_f32(lg, logits)
    else:
        rnd = ROUND[mode]
        assert normwise(lg, rnd(hs[-1]).astype(np.float64) @ rnd(w.logits).T.astype(np.float64)) <= 1e-5
        assert e <= BOUND_VS_F32[mode]
    for T in w.block_sizes:
        got = m.forward(frames, T).cpu().numpy()
        assert got.shape == (4096, 2000)
        e = normwise(got, logits)
        _record(f"cfg3 {mode} T_b={T} logits vs fp32 oracle", e)
        if mode == "f32":
            assert_f32(got, logits, T)
        else:
            assert e <= BOUND_VS_F32[mode], (T, e)
    m.close()


@pytest.mark.parametrize("mode", ["bf16", "tf32"])
def test_cfg3_per_layer_rounded_operands(P, oracle, cfg3, mode):
    """Each of the 6 SRU layers at L=4096, T_b=32 on the GPU's own layer
    input vs the oracle on rounded operands (the per-layer bound), c_T too."""
    import torch
    w, mats, hs, _ = cfg3
    x = hs[0]
    for li, lay in enumerate(w.layers):
        st = P.DeviceStack("sru", [lay], mode=mode)
        c = torch.zeros(1024, device="cuda")
        H = st.forward(_cuda(x), 32, c_state=c).cpu().numpy()
        assert st.query(9) == 1
        ref, cref = rounded_layer(oracle, "sru", mats[li], x, 32, mode)
        e = normwise(H, ref)
        _record(f"cfg3 {mode} layer {li + 1} vs rounded-operand oracle", e)
        assert e <= BOUND_VS_ROUNDED[mode], (li, e)
        assert normwise(c.cpu().numpy(), cref) <= BOUND_VS_ROUNDED[mode]
        st.close()
        x = H


# ---------------------------------------------------------------------------
# cfg4

PREFIX4 = 8192
WINDOW4 = 1024


@pytest.fixture(scope="module")
def cfg4(oracle):
    from paper_1803_11389_b200 import workloads
    w = workloads.make("cfg4")
    mats = [lay.mats() for lay in w.layers]
    xp = np.ascontiguousarray(w.X[:PREFIX4])
    ref, cref, _ = oracle.run_blocked("qrnn", mats, xp, 32, return_state=True)
    return w, mats, xp, ref, cref


@pytest.mark.parametrize("mode", ["f32_ffma", "f32", "bf16", "tf32", "f32x3"])
def test_cfg4_all_layers_prefix(P, oracle, cfg4, mode, monkeypatch):
    """8 x QRNN-2048 on an 8192-step prefix, T_b=32: output and every
    layer's c_T vs the fp32 oracle (fp32 bound for the fp32 modes: the
    weight-streaming FFMA kernel, fp32 mode's default 3xTF32 tcgen05, f32x3)."""
    import torch
    w, mats, xp, ref, cref = cfg4
    if mode == "f32_ffma":
        monkeypatch.setenv("RNNB_F32_TC", "0")
        mode = "f32"
        ffma = True
    else:
        ffma = False
    st = P.DeviceStack("qrnn", w.layers, mode=mode)
    c = torch.zeros(8 * 2048, device="cuda")
    H = st.forward(_cuda(xp), 32, c_state=c).cpu().numpy()
    if ffma:
        assert all(st.query(11, li) == 1 for li in range(8)), "weight-streaming FFMA kernel did not run"
        mode = "f32_ffma"
    else:
        assert all(st.query(9, li) == 1 for li in range(8)), "tcgen05 kernel did not run"
    cs = c.cpu().numpy().reshape(8, 2048)
    e = normwise(H, ref)
    _record(f"cfg4 {mode} 8 layers L={PREFIX4} vs fp32 oracle", e)
    for li in range(8):
        _record(f"cfg4 {mode} layer {li + 1} c_T vs fp32 oracle", normwise(cs[li], cref[li]))
    if mode in ("bf16", "tf32"):
        assert e <= BOUND_VS_F32[mode]
        for li in range(8):
            assert normwise(cs[li], cref[li]) <= BOUND_VS_F32[mode]
    else:
        assert_f32(H, ref, mode)
        for li in range(8):
            assert_f32(cs[li], cref[li], (mode, li))
    st.close()


def test_cfg4_bf16_per_layer_rounded_operands(P, oracle, cfg4):
    """bf16 per layer on the GPU's own layer input (rounded-operand bound)
    with c_T; the chain of one-layer stacks equals the 8-layer stack."""
    import torch
    w, mats, xp, _, _ = cfg4
    x = xp
    for li, lay in enumerate(w.layers):
        st = P.DeviceStack("qrnn", [lay], mode="bf16")
        c = torch.zeros(2048, device="cuda")
        H = st.forward(_cuda(x), 32, c_state=c).cpu().numpy()
        ref, cref = rounded_layer(oracle, "qrnn", mats[li], x, 32, "bf16")
        e = normwise(H, ref)
        _record(f"cfg4 bf16 layer {li + 1} vs rounded-operand oracle", e)
        assert e <= BOUND_VS_ROUNDED["bf16"], (li, e)
        assert normwise(c.cpu().numpy(), cref) <= BOUND_VS_ROUNDED["bf16"], li
        st.close()
        x = H
    whole = P.DeviceStack("qrnn", w.layers, mode="bf16")
    Hw = whole.forward(_cuda(xp), 32).cpu().numpy()
    assert normwise(Hw, x) <= 1e-6
    whole.close()


@pytest.mark.parametrize("mode", ["f32", "bf16"])
def test_cfg4_full_sequence_window(P, oracle, cfg4, mode, monkeypatch):
    """The full 65536-step sequence (2048 blocks x 8 layers through the
    look-back / the streamed FFMA passes): one call == the same sequence in
    two calls split at L-1024 with carried (c, x_carry) (bitwise for the
    FFMA kernel, look-back re-anchored at the split for tcgen05), and the
    last 1024 steps == the oracle restarted from the GPU's state there."""
    import torch
    monkeypatch.setenv("RNNB_F32_TC", "0")  # f32 here = the FFMA kernels (bitwise split invariance)
    w, mats, _, _, _ = cfg4
    L = w.X.shape[0]
    s = L - WINDOW4
    st = P.DeviceStack("qrnn", w.layers, mode=mode)
    Xd = _cuda(w.X)
    whole = st.forward(Xd, 32)
    c = torch.zeros(8 * 2048, device="cuda")
    xc = torch.zeros(8 * 2048, device="cuda")
    a = st.forward(Xd[:s], 32, c_state=c, x_carry=xc)
    c_s, xc_s = c.cpu().numpy().reshape(8, 2048).copy(), xc.cpu().numpy().reshape(8, 2048).copy()
    b = st.forward(Xd[s:], 32, c_state=c, x_carry=xc).cpu().numpy()
    tail = whole[s:].cpu().numpy()
    if mode == "f32":
        assert a.cpu().numpy().tobytes() == whole[:s].cpu().numpy().tobytes()
        assert b.tobytes() == tail.tobytes()
    else:
        assert normwise(a.cpu().numpy(), whole[:s].cpu().numpy()) <= 1e-6
        assert normwise(b, tail) <= 1e-6
    del whole, a
    x = np.ascontiguousarray(w.X[s:])
    for li in range(8):
        x, _, _ = oracle.layer_blocked("qrnn", mats[li], x, 32, c=c_s[li], xc=xc_s[li])
    e = normwise(b, x)
    _record(f"cfg4 {mode} steps {s}..{L} (restarted oracle) vs fp32 oracle", e)
    if mode == "f32":
        assert_f32(b, x)
    else:
        assert e <= BOUND_VS_F32["bf16"]
    st.close()


# ---------------------------------------------------------------------------
# cfg5

EDGE5 = 256


@pytest.fixture(scope="module")
def cfg5():
    from paper_1803_11389_b200 import workloads
    return workloads.make("cfg5")


def _bidir_layers(P, w, mode, T):
    """The unsharded per-layer composition (one-direction DeviceStacks, the
    backward one on the time-reversed input): returns every layer's input
    and output as CUDA tensors."""
    import torch
    x = _cuda(w.X)
    H = w.layers[0].mats()[0].shape[0]
    ins, outs = [], []
    for lf, lb in zip(w.layers, w.layers_bwd):
        ys = []
        for d, lay in enumerate((lf, lb)):
            m = lay.mats()
            hw = 0 if m[0].shape[1] == H else d * H
            st = P.DeviceStack("sru", [tuple(m[:5])], mode=mode, wide=True, highway_offsets=[hw])
            xin = x if d == 0 else torch.flip(x, dims=[0]).contiguous()
            y = st.forward(xin, T)
            assert st.query(9) == 1
            ys.append(y if d == 0 else torch.flip(y, dims=[0]))
            st.close()
        ins.append(x)
        x = torch.cat(ys, dim=1).contiguous()
        outs.append(x)
    return ins, outs


@pytest.mark.parametrize("T", [16, 64])
def test_cfg5_bidirectional_wide_sru(P, oracle, cfg5, T):
    import torch
    from paper_1803_11389_b200 import p2p
    w = cfg5
    Hd = 4096
    ins, outs = _bidir_layers(P, w, "bf16", T)
    rnd = ROUND["bf16"]
    # layer 1, both directions: the oracle's square SRU on rounded operands
    X = w.X
    y1 = outs[0].cpu().numpy()
    mf = w.layers[0].mats()
    mb = w.layers_bwd[0].mats()
    if T == 64:  # the oracle is independent of T_b: run it once
        ref_f, _ = rounded_layer(oracle, "sru", list(mf), X, 32, "bf16")
        ref_b, _ = rounded_layer(oracle, "sru", list(mb), np.ascontiguousarray(X[::-1]), 32, "bf16")
        ef, eb = normwise(y1[:, :Hd], ref_f), normwise(y1[:, Hd:], ref_b[::-1])
        _record(f"cfg5 bf16 T_b={T} layer 1 fwd vs rounded-operand oracle", ef)
        _record(f"cfg5 bf16 T_b={T} layer 1 bwd vs rounded-operand oracle", eb)
        assert ef <= BOUND_VS_ROUNDED["bf16"] and eb <= BOUND_VS_ROUNDED["bf16"]
    # layers 2-4 (d_in 8192): float64 cell on the GPU's own layer input,
    # forward direction on a prefix, backward on a suffix (its scan starts at t = L-1)
    L = X.shape[0]
    for li in range(1, 4):
        x = ins[li].cpu().numpy()
        y = outs[li].cpu().numpy()
        xr = rnd(x)
        mf = [rnd(m) if m.ndim == 2 else m for m in w.layers[li].mats()]
        mb = [rnd(m) if m.ndim == 2 else m for m in w.layers_bwd[li].mats()]
        rf = sru_wide_f64(mf, xr, x[:, :Hd], rows=EDGE5)
        xrb = np.ascontiguousarray(xr[::-1][:EDGE5])
        rb = sru_wide_f64(mb, xrb, x[::-1][:EDGE5, Hd:])[::-1]
        ef = normwise(y[:EDGE5, :Hd], rf)
        eb = normwise(y[L - EDGE5:, Hd:], rb)
        _record(f"cfg5 bf16 T_b={T} layer {li + 1} fwd prefix vs f64 cell", ef)
        _record(f"cfg5 bf16 T_b={T} layer {li + 1} bwd suffix vs f64 cell", eb)
        assert ef <= BOUND_VS_ROUNDED["bf16"] and eb <= BOUND_VS_ROUNDED["bf16"], (li, ef, eb)
    # the product path: fused, sharded (world 1 and 2 emulated on this GPU)
    want = outs[-1]
    del ins, outs
    for world in (1, 2):
        ranks = [p2p.P2PBidirSRU(w.layers, w.layers_bwd, g, world, T, "bf16", L) for g in range(world)]
        for r in ranks:
            r.connect_local(ranks)
        got = p2p.run_local_bidir(ranks, _cuda(X))
        torch.cuda.synchronize()
        e = normwise(got[0].cpu().numpy(), want.cpu().numpy())
        _record(f"cfg5 bf16 T_b={T} fused sharded G={world} vs per-layer composition", e)
        assert e <= 1e-6, (world, e)
        for r in ranks:
            r.close()
        del got, ranks
        torch.cuda.empty_cache()


def test_cfg5_fp32_mode_wide_layers(P, oracle, cfg5):
    """cfg5's shape in fp32 mode (3xTF32 tcgen05 at T_b = 64): layer 1 of each
    direction vs the fp32 oracle, layer 2 (d_in 8192) vs the float64 cell on
    a prefix / suffix of the GPU's own layer input, all at the fp32 bound."""
    import torch
    w = cfg5
    Hd, L = 4096, w.X.shape[0]
    ins, outs = _bidir_layers(P, type(w)(w.name, w.kind, w.layers[:2], w.X, w.block_sizes,
                                         bidirectional=True, layers_bwd=w.layers_bwd[:2]), "f32", 64)
    y1 = outs[0].cpu().numpy()
    ref_f = oracle.layer_blocked("sru", list(w.layers[0].mats()), w.X, 32)[0]
    ref_b = oracle.layer_blocked("sru", list(w.layers_bwd[0].mats()), np.ascontiguousarray(w.X[::-1]), 32)[0]
    _record("cfg5 f32 layer 1 fwd vs fp32 oracle", assert_f32(y1[:, :Hd], ref_f))
    _record("cfg5 f32 layer 1 bwd vs fp32 oracle", assert_f32(y1[:, Hd:], ref_b[::-1]))
    x = ins[1].cpu().numpy()
    y = outs[1].cpu().numpy()
    rf = sru_wide_f64(list(w.layers[1].mats()), x, x[:, :Hd], rows=EDGE5)
    rb = sru_wide_f64(list(w.layers_bwd[1].mats()), np.ascontiguousarray(x[::-1][:EDGE5]), x[::-1][:EDGE5, Hd:])[::-1]
    _record("cfg5 f32 layer 2 fwd prefix vs f64 cell", assert_f32(y[:EDGE5, :Hd], rf))
    _record("cfg5 f32 layer 2 bwd suffix vs f64 cell", assert_f32(y[L - EDGE5:, Hd:], rb))
    del ins, outs
    torch.cuda.empty_cache()
