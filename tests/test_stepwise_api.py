"""paper_1803_11389_b200.stepwise: drop-in for the reference's step
executors (cells.py:146-229).  CPU: argument checks; GPU (`-m gpu`): a
chain of single steps equals the layer run at T_b = 1 and both match the
oracle's stepwise restatement (oracle/oracle_strict.c) within the fp32 /
f64 bounds of tests/test_gpu_parity.py."""

import numpy as np
import pytest

import paper_1803_11389_b200 as P
from paper_1803_11389_b200 import stepwise as S


def _layer(oracle, kind, d, seed, dtype):
    m = oracle.generate_layers(kind, d, d, 1, seed, dtype)[0]
    cls = {"sru": P.SruWeights, "qrnn": P.QrnnWeights, "lstm": P.LstmWeights}[kind]
    return cls(*[np.ascontiguousarray(a) for a in m]), m


def test_step_argument_errors(oracle):
    w, _ = _layer(oracle, "qrnn", 8, 1, np.float32)
    st = P.zero_state(8, 8, np.float32)
    with pytest.raises(ValueError, match="input length"):
        S.qrnn_step(w, np.zeros(7, np.float32), st)
    bad = P.CellState(c=np.zeros(7, np.float32), h=np.zeros(8, np.float32), x_prev=np.zeros(8, np.float32))
    with pytest.raises(ValueError, match="state width"):
        S.qrnn_step(w, np.zeros(8, np.float32), bad)
    with pytest.raises(ValueError, match="input must be"):
        S.run_layer_stepwise(P.CellKind.QRNN, w, np.zeros((3, 7), np.float32))
    cfg = P.RnnConfig(P.CellKind.QRNN, 8, 8, n_layers=1, precision="f32")
    with pytest.raises(ValueError, match="does not match config d_in"):
        S.run_stepwise(cfg, P.WeightSet(P.CellKind.QRNN, "f32", [w]), np.zeros((3, 9), np.float32))


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["sru", "qrnn", "lstm"])
@pytest.mark.parametrize("dtype", [np.float32, np.float64])
def test_step_chain_equals_layer_and_oracle(oracle, kind, dtype):
    d, L = 64, 19
    w, mats = _layer(oracle, kind, d, 31, dtype)
    X = np.random.default_rng(5).standard_normal((L, d)).astype(dtype)
    k = P.CellKind.parse(kind)
    state = P.zero_state(d, d, dtype)
    hs = []
    for t in range(L):
        state = S.step(k, w, X[t], state)
        hs.append(state.h)
    chain = np.stack(hs)
    layer = S.run_layer_stepwise(k, w, X)
    if kind == "lstm":
        ref = oracle.lstm_stepwise(w, X)
    else:
        ref = oracle.layer_stepwise(kind, mats, X)[0]
    tol = 1e-5 if dtype == np.float32 else 1e-12
    scale = max(float(np.max(np.abs(ref))), 1e-30)
    assert np.max(np.abs(chain - ref)) / scale <= tol
    assert np.max(np.abs(layer - ref)) / scale <= tol
    assert chain.dtype == dtype and layer.dtype == dtype
    assert np.array_equal(state.x_prev, X[-1])
