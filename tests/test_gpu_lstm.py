"""GPU parity of the LSTM partial-precompute path:
``lstm_run_precomputed`` (blocked.py:271-305) through librnnb.so against the
reference's own outputs (tests/golden/lstm_cases.npz) and the C oracle.

Tolerances: fp32 normwise <= 1e-5 AND max-abs <= 1e-4 (ORACLE_TOLERANCE,
bench.py:25); f64 <= 1e-12 max-abs.
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import paper_1803_11389_b200 as P
    return P


def assert_close(a, ref, dtype):
    a = np.asarray(a, np.float64)
    ref = np.asarray(ref, np.float64)
    d = float(np.max(np.abs(a - ref)))
    if dtype == np.float64:
        assert d <= 1e-12, d
    else:
        nw = d / max(float(np.max(np.abs(ref))), 1e-30)
        assert nw <= 1e-5 and d <= 1e-4, (nw, d)


def _cases():
    with open(os.path.join(GOLDEN, "lstm_cases.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("case", _cases(), ids=lambda c: f"{c['precision']}-{c['d_in']}x{c['d_h']}-L{c['L']}")
def test_lstm_matches_reference_fixtures(P, oracle, case):
    z = np.load(os.path.join(GOLDEN, "lstm_cases.npz"))
    n = case["case"]
    dt = np.float32 if case["precision"] == "f32" else np.float64
    w = P.LstmWeights(*oracle.generate_layers("lstm", case["d_in"], case["d_h"], 1, case["wseed"], dt)[0])
    X = z[f"l{n}_X"]
    for T in case["T_b"]:
        H = P.lstm_run_precomputed(w, X, T)
        assert H.dtype == X.dtype and H.shape == (case["L"], case["d_h"])
        assert_close(H, z[f"l{n}_T{T}_H"], dt)
        assert_close(H, z[f"l{n}_stepwise"], dt)


@pytest.mark.parametrize("din,dh,L", [(1024, 1024, 300), (512, 700, 129), (256, 2048, 64), (3, 5, 40)])
def test_lstm_sizes_vs_oracle(P, oracle, din, dh, L):
    """Resident U (d_h <= 1024 fp32), U read from L2 (d_h = 2048), odd widths."""
    import torch
    w = oracle.generate_layers("lstm", din, dh, 1, 91, np.float32)[0]
    X = np.random.default_rng(3).standard_normal((L, din)).astype(np.float32)
    dev = P.DeviceLstm(w)
    H = dev.forward(torch.from_numpy(X).cuda(), 16).cpu().numpy()
    assert dev.query(3) == (1 if dh <= 1024 else 0)
    assert dev.query(4) * dev.query(2) >= dh
    assert_close(H, oracle.lstm_blocked(w, X, 16), np.float32)
    dev.close()


def test_lstm_f64_and_state_in_out(P, oracle):
    import torch
    w = oracle.generate_layers("lstm", 96, 160, 1, 17, np.float64)[0]
    X = np.random.default_rng(4).standard_normal((90, 96))
    c0 = np.random.default_rng(5).standard_normal(160) * 0.5
    h0 = np.random.default_rng(6).standard_normal(160) * 0.5
    ref, cT, hT = oracle.lstm_blocked(w, X, 8, c=c0, h=h0, return_state=True)
    dev = P.DeviceLstm(w, mode="f64")
    c = torch.from_numpy(c0.copy()).cuda()
    h = torch.from_numpy(h0.copy()).cuda()
    H = dev.forward(torch.from_numpy(X).cuda(), 8, c_state=c, h_state=h).cpu().numpy()
    assert_close(H, ref, np.float64)
    assert_close(c.cpu().numpy(), cT, np.float64)
    assert_close(h.cpu().numpy(), hT, np.float64)
    # streaming: two halves with carried (c, h) equal one call, bitwise
    c2 = torch.from_numpy(c0.copy()).cuda()
    h2 = torch.from_numpy(h0.copy()).cuda()
    Xd = torch.from_numpy(X).cuda()
    A = dev.forward(Xd[:40].contiguous(), 8, c_state=c2, h_state=h2).cpu().numpy()
    B = dev.forward(Xd[40:].contiguous(), 8, c_state=c2, h_state=h2).cpu().numpy()
    assert np.concatenate([A, B]).tobytes() == H.tobytes()
    # host entry point: bitwise the device result
    ch, hh = c0.copy(), h0.copy()
    Hh = dev.forward_host(X, 8, c_state=ch, h_state=hh)
    assert Hh.tobytes() == H.tobytes() and ch.tobytes() == c.cpu().numpy().tobytes()
    dev.close()


def test_lstm_block_size_independent_and_deterministic(P, oracle):
    w = P.LstmWeights(*oracle.generate_layers("lstm", 128, 128, 1, 23, np.float32)[0])
    X = oracle.generate_sequence(200, 128, 24, np.float32)
    outs = [P.lstm_run_precomputed(w, X, T) for T in (1, 7, 32, 200, 1000)]
    for o in outs[1:]:
        assert o.tobytes() == outs[0].tobytes()


def test_lstm_recurrent_ablation(P, oracle):
    """test_blocked.py:346-359: with U = 0 the computation is feed-forward."""
    w = P.LstmWeights(*oracle.generate_layers("lstm", 8, 8, 1, 5, np.float64)[0])
    for f in ("u_forget", "u_input", "u_output", "u_cand"):
        getattr(w, f)[:] = 0.0
    X = oracle.generate_sequence(32, 8, 6, np.float64)
    ref = oracle.lstm_stepwise(w.mats(), X)
    for T in (1, 8, 32):
        assert np.max(np.abs(P.lstm_run_precomputed(w, X, T) - ref)) <= 1e-12


def test_lstm_call_counts_and_errors(P, oracle):
    """test_blocked.py:362-376."""
    w = P.LstmWeights(*oracle.generate_layers("lstm", 8, 8, 1, 7, np.float32)[0])
    X = oracle.generate_sequence(64, 8, 8, np.float32)
    trace = P.KernelTrace()
    P.lstm_run_precomputed(w, X, 16, trace=trace)
    assert trace.count(P.PHASE_GEMM) == 4 * 4
    assert trace.count(P.PHASE_GEMV) == 4 * 64
    with pytest.raises(ValueError):
        P.lstm_run_precomputed(w, np.zeros((4, 9), np.float32), 2)
    with pytest.raises(ValueError):
        P.lstm_run_precomputed(w, X, 0)
    with pytest.raises(ValueError):
        P.lstm_run_precomputed(w, X.astype(np.float64), 4)
    with pytest.raises(ValueError):
        P.lstm_run_precomputed(w, X, 4, kernel="cuda")


@pytest.mark.parametrize("din,dh,L", [(350, 350, 257), (64, 64, 100), (7, 5, 33), (512, 470, 65), (96, 17, 40)])
def test_lstm_cluster_recurrence_vs_oracle(P, oracle, din, dh, L, monkeypatch):
    """Small fp32 layers run the recurrence inside one 16-CTA cluster (h
    exchanged through distributed shared memory, one cluster barrier per
    step); the grid kernel (RNNB_LSTM_CLUSTER=0) must agree with the oracle
    on the same inputs, and both are deterministic."""
    import torch
    w = oracle.generate_layers("lstm", din, dh, 1, 17, np.float32)[0]
    X = np.random.default_rng(5).standard_normal((L, din)).astype(np.float32)
    ref = oracle.lstm_blocked(w, X, 8)
    dev = P.DeviceLstm(w)
    Xd = torch.from_numpy(X).cuda()
    H1 = dev.forward(Xd, 8).cpu().numpy()
    assert dev.query(5) == 16
    assert_close(H1, ref, np.float32)
    assert np.array_equal(H1, dev.forward(Xd, 8).cpu().numpy())
    monkeypatch.setenv("RNNB_LSTM_CLUSTER", "0")
    H0 = dev.forward(Xd, 8).cpu().numpy()
    assert dev.query(5) == 0
    assert_close(H0, ref, np.float32)
    # same products in the same order on both paths
    assert np.array_equal(H0, H1)
    dev.close()


def test_lstm_cluster_not_used_when_u_does_not_fit(P, oracle):
    import torch
    w = oracle.generate_layers("lstm", 64, 512, 1, 3, np.float32)[0]
    X = np.random.default_rng(1).standard_normal((20, 64)).astype(np.float32)
    dev = P.DeviceLstm(w)
    H = dev.forward(torch.from_numpy(X).cuda(), 4).cpu().numpy()
    assert dev.query(5) == 0
    assert_close(H, oracle.lstm_blocked(w, X, 4), np.float32)
    dev.close()
