"""Pin the CPU oracle (oracle/) to the reference before trusting it.

Every fixture under tests/golden/ was produced by the reference package
itself (tests/golden/make_golden.py imports /root/reference/pkg/src).  The
oracle is a C restatement, so the only allowed differences are libm-vs-numpy
tanh ulps: f32 <= 1e-6 absolute on O(0.1..1) values, f64 <= 1e-14.
"""

import json
import os

import numpy as np
import pytest

from conftest import GOLDEN

TOL = {"f32": 1e-6, "f64": 1e-14}


def _json(name):
    with open(os.path.join(GOLDEN, name)) as f:
        return json.load(f)


def test_splitmix_known_answers(oracle):
    kat = _json("splitmix.json")
    # published first value of SplitMix64 from seed 0 (kernels.py:256-257)
    assert int(oracle.raw_stream(0, 1)[0]) == 0xE220A8397B1DCDAF
    assert [int(v) for v in oracle.raw_stream(0, 4)] == kat["seed0_first4"]
    assert [int(v) for v in oracle.raw_stream(42, 8)] == kat["seed42_first8"]
    u = oracle.uniform_array(oracle.raw_stream(42, 8))
    assert u.tolist() == kat["uniform_seed42_first8"]
    for raw, val in kat["uniform_weight_kat"].items():
        assert oracle.uniform_array(np.array([int(raw)], np.uint64))[0] == val


@pytest.mark.parametrize("kind", ["sru", "qrnn"])
def test_d2_golden_vectors(oracle, kind):
    """The reference test-suite's hand-checked d=2 goldens (1e-12, f64)."""
    g = _json("cells_d2.json")[kind]
    fields = oracle.SRU_FIELDS if kind == "sru" else oracle.QRNN_FIELDS
    layer = [np.array(g["weights"][f], np.float64) for f in fields]
    X = np.array(g["X"], np.float64)
    H, c, _ = oracle.layer_stepwise(kind, layer, X)
    assert np.max(np.abs(H - np.array(g["H"]))) < 1e-12
    assert np.max(np.abs(c - np.array(g["C"][-1]))) < 1e-12
    for t, (h_pub, c_pub) in enumerate(g["golden_published"]):
        assert np.max(np.abs(H[t] - np.array(h_pub))) < 1e-12
    # blocked at every block size reproduces the stepwise goldens
    for T in (1, 2, 3, 8):
        for k in ("reference", "fast"):
            Hb, cb, _ = oracle.layer_blocked(kind, layer, X, T, kernel=k)
            assert np.max(np.abs(Hb - np.array(g["H"]))) < 1e-12
            assert np.max(np.abs(cb - np.array(g["C"][-1]))) < 1e-12


def _cases():
    return _json("blocked_cases.json")


@pytest.mark.parametrize("case", _cases(), ids=lambda c: f"{c['kind']}-{c['precision']}-d{c['d']}-L{c['L']}-n{c['n_layers']}")
def test_oracle_matches_reference_run_blocked(oracle, case):
    g = np.load(os.path.join(GOLDEN, "blocked_cases.npz"))
    dt = np.float32 if case["precision"] == "f32" else np.float64
    tol = TOL[case["precision"]]
    layers = oracle.generate_layers(case["kind"], case["d"], case["d"], case["n_layers"], case["wseed"], dt)
    X = oracle.generate_sequence(case["L"], case["d"], case["xseed"], dt)
    n = case["case"]
    st = oracle.run_stepwise(case["kind"], layers, X)
    assert np.max(np.abs(st - g[f"c{n}_stepwise"])) <= tol
    for T in case["T_b"]:
        for kernel in ("fast", "reference"):
            H, cs, xcs = oracle.run_blocked(case["kind"], layers, X, T, kernel=kernel, return_state=True)
            assert np.max(np.abs(H - g[f"c{n}_T{T}_H"])) <= tol
            assert np.max(np.abs(np.stack(cs) - g[f"c{n}_T{T}_c"])) <= tol
            if case["kind"] == "qrnn":
                assert np.array_equal(xcs[0], g[f"c{n}_T{T}_xc"][0])  # layer 0: raw input row
                assert np.max(np.abs(np.stack(xcs) - g[f"c{n}_T{T}_xc"])) <= tol


def test_oracle_t1_reference_blocked_is_bitwise_stepwise(oracle):
    """blocked.py with T=1 and the strict kernel runs the stepwise ops
    (test_blocked.py:240-247 property, restated for the oracle)."""
    for kind in ("sru", "qrnn"):
        layers = oracle.generate_layers(kind, 16, 16, 1, 5, np.float32)
        X = oracle.generate_sequence(20, 16, 6, np.float32)
        a = oracle.run_stepwise(kind, layers, X)
        b = oracle.run_blocked(kind, layers, X, 1, kernel="reference")
        assert a.tobytes() == b.tobytes()


def test_oracle_block_size_independence(oracle):
    layers = oracle.generate_layers("sru", 32, 32, 1, 7, np.float32)
    X = oracle.generate_sequence(128, 32, 8, np.float32)
    a = oracle.run_blocked("sru", layers, X, 4)
    b = oracle.run_blocked("sru", layers, X, 64)
    assert np.max(np.abs(a - b)) <= 2e-4


def test_oracle_thread_count_invariance(oracle):
    layers = oracle.generate_layers("qrnn", 300, 300, 1, 9, np.float32)
    X = oracle.generate_sequence(40, 300, 10, np.float32)
    before = oracle.get_threads()
    try:
        oracle.set_threads(1)
        a = oracle.run_blocked("qrnn", layers, X, 16)
        oracle.set_threads(4)
        b = oracle.run_blocked("qrnn", layers, X, 16)
    finally:
        oracle.set_threads(before)
    assert a.tobytes() == b.tobytes()


def test_oracle_baseline_cfg1_against_reference(oracle):
    """BASELINE cfg1 (SRU 512, L=256) with the repo's seeded workload,
    reference outputs from make_golden.py."""
    from paper_1803_11389_b200 import workloads
    g = np.load(os.path.join(GOLDEN, "baseline_cfg.npz"))
    w = workloads.make("cfg1")
    layers = [lay.mats() for lay in w.layers]
    for T in (1, 4, 16):
        H, cs, _ = oracle.run_blocked("sru", layers, w.X, T, return_state=True)
        assert np.max(np.abs(cs[0] - g[f"cfg1_T{T}_c"])) <= 1e-5
        if T == 16:
            ref = g["cfg1_T16_H"]
            assert np.max(np.abs(H - ref)) / np.max(np.abs(ref)) <= 1e-6


# ---------------------------------------------------------------------------
# LSTM partial precompute (blocked.py:271-305, cells.py:153-164)


def test_lstm_d2_golden_vectors(oracle):
    """The reference suite's hand-checked d=2 LSTM goldens (test_cells.py
    LSTM_GOLDEN, 1e-12) through both oracle paths."""
    g = _json("cells_d2.json")["lstm"]
    w = [np.array(g["weights"][f], np.float64) for f in oracle.LSTM_FIELDS]
    X = np.array(g["X"], np.float64)
    H, c, h = oracle.lstm_stepwise(w, X, return_state=True)
    for t, (h_exp, c_exp) in enumerate(g["golden_published"]):
        assert np.max(np.abs(H[t] - h_exp)) < 1e-12
    assert np.max(np.abs(c - g["golden_published"][-1][1])) < 1e-12
    for T in (1, 2):
        Hb = oracle.lstm_blocked(w, X, T, kernel="reference")
        assert np.max(np.abs(Hb - np.array(g[f"H_precomputed_T{T}"]))) < 1e-15


def _lstm_cases():
    return _json("lstm_cases.json")


@pytest.mark.parametrize("case", _lstm_cases(), ids=lambda c: f"{c['precision']}-{c['d_in']}x{c['d_h']}-L{c['L']}")
def test_oracle_matches_reference_lstm(oracle, case):
    """lstm_run_precomputed (kernel='fast') and run_stepwise outputs made by
    the reference; weights regenerated by the oracle's SplitMix64
    restatement where the fixture omits them (checked equal where present)."""
    z = np.load(os.path.join(GOLDEN, "lstm_cases.npz"))
    n = case["case"]
    dt = np.float32 if case["precision"] == "f32" else np.float64
    gen = oracle.generate_layers("lstm", case["d_in"], case["d_h"], 1, case["wseed"], dt)[0]
    if f"l{n}_w_forget" in z:
        ref_w = [z[f"l{n}_{f}"] for f in oracle.LSTM_FIELDS]
        assert all(np.array_equal(a, b) for a, b in zip(ref_w, gen))
    X = z[f"l{n}_X"]
    assert np.array_equal(X, oracle.generate_sequence(case["L"], case["d_in"], case["xseed"], dt))
    tol = 1e-6 if dt == np.float32 else 1e-14
    assert np.max(np.abs(oracle.lstm_stepwise(gen, X) - z[f"l{n}_stepwise"])) <= tol
    for T in case["T_b"]:
        assert np.max(np.abs(oracle.lstm_blocked(gen, X, T) - z[f"l{n}_T{T}_H"])) <= tol
