"""Host-side logic that needs no GPU: block planning, drop-in types and
their ValueErrors, trace events, workloads."""

import numpy as np
import pytest

import paper_1803_11389_b200 as P
from paper_1803_11389_b200 import blocked, workloads


def test_plan_blocks_matches_reference_semantics():
    assert [l for _, l in P.plan_blocks(100, 32).blocks] == [32, 32, 32, 4]
    assert P.plan_blocks(5, 8).blocks == ((0, 5),)
    assert len(P.plan_blocks(1024, 32).blocks) == 32
    for L in (1, 2, 7, 33, 100, 257):
        for T in (1, 2, 5, 32, 300):
            cur = 0
            for s, l in P.plan_blocks(L, T).blocks:
                assert s == cur and 1 <= l <= T
                cur += l
            assert cur == L
    with pytest.raises(ValueError):
        P.plan_blocks(0, 4)
    with pytest.raises(ValueError):
        P.plan_blocks(4, 0)


def test_types_validate_like_reference():
    with pytest.raises(ValueError):
        P.SruWeights(np.zeros((2, 3)), np.zeros((2, 3)), np.zeros((2, 3)), np.zeros(2), np.zeros(2))
    with pytest.raises(ValueError):
        P.QrnnWeights(*([np.zeros((2, 2))] * 5 + [np.zeros((2, 3))]))
    with pytest.raises(ValueError):
        P.RnnConfig(P.CellKind.SRU, 4, 5)
    with pytest.raises(ValueError):
        P.RnnConfig(P.CellKind.QRNN, 4, 4, precision="f16")
    with pytest.raises(ValueError):
        P.CellKind.parse("gru")
    assert P.CellKind.parse("QRNN") is P.CellKind.QRNN
    cfg = P.RnnConfig(P.CellKind.QRNN, 3, 5, n_layers=2)
    assert cfg.layer_dims(0) == (3, 5) and cfg.layer_dims(1) == (5, 5)


def test_trace_events_match_reference_counts():
    """GEMM events 3*ceil(L/T) (SRU) / 6*ceil(L/T) (QRNN); stacked 1 / 2
    per block (reference test_blocked.py:291-322 contract)."""
    L, T = 256, 32
    nb = -(-L // T)
    for kind, per in ((P.CellKind.SRU, 3), (P.CellKind.QRNN, 6)):
        w = (P.SruWeights(*([np.zeros((16, 16))] * 3 + [np.zeros(16)] * 2)) if kind is P.CellKind.SRU
             else P.QrnnWeights(*([np.zeros((16, 16))] * 6)))
        tr = P.KernelTrace()
        for _, l in P.plan_blocks(L, T).blocks:
            blocked._trace_block(tr, kind, w, l, False)
        assert tr.count(P.PHASE_GEMM) == per * nb
        assert tr.count(P.PHASE_GEMV) == 0
        tr2 = P.KernelTrace()
        for _, l in P.plan_blocks(64, 16).blocks:
            blocked._trace_block(tr2, kind, w, l, True)
        assert tr2.count(P.PHASE_GEMM) == (4 if kind is P.CellKind.SRU else 8)
        for line in tr.lines():
            ph, m, k, n = line.split(",")
            assert ph in (P.PHASE_GEMM, P.PHASE_BIAS) and int(m) > 0 and int(n) > 0
        # touches equal the reference traffic model (traffic.py:92-107)
        want = (3 if kind is P.CellKind.SRU else 6) * 16 * 16 * nb
        assert tr.touches(P.PHASE_GEMM) == want


def test_workloads_shapes_and_determinism():
    w1 = workloads.make("cfg1")
    assert w1.X.shape == (256, 512) and w1.kind is P.CellKind.SRU
    assert w1.layers[0].w_cand.shape == (512, 512)
    assert np.all(np.abs(w1.layers[0].w_cand) <= 1 / np.sqrt(512))
    assert (w1.layers[0].b_forget == 0).all()
    again = workloads.make("cfg1")
    assert again.X.tobytes() == w1.X.tobytes()
    w2 = workloads.make("cfg2", scale=1 / 64)
    assert w2.X.shape == (32, 1024) and len(w2.layers[0].mats()) == 6
    assert np.all(np.abs(w2.layers[0].w_out_prev) <= 1 / np.sqrt(2048))
    w3 = workloads.make("cfg3", scale=1 / 256)
    assert w3.proj.shape == (1024, 120) and w3.logits.shape == (2000, 1024) and len(w3.layers) == 6
    assert workloads.flops_per_step(workloads.make("cfg2", scale=1 / 2048)) == 2 * 3 * 1024 * 2 * 1024


def test_product_path_has_no_cpu_fallback():
    """Without CUDA the product entry points raise instead of computing."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    w = P.SruWeights(*([np.zeros((4, 4), np.float32)] * 3 + [np.zeros(4, np.float32)] * 2))
    cfg = P.RnnConfig(P.CellKind.SRU, 4, 4)
    with pytest.raises(RuntimeError):
        P.run_blocked(cfg, P.WeightSet(P.CellKind.SRU, "f32", [w]), np.zeros((3, 4), np.float32), 2)


def test_top_level_names_match_the_reference_package():
    """Every name rnnblock/__init__.py exports exists at our package's top
    level (drop-in `import paper_1803_11389_b200 as rnnblock`); the list is
    the reference's own export list, restated."""
    import paper_1803_11389_b200 as P
    names = ["BenchRecord", "BenchResult", "SpeedupRow", "bench", "emit_csv", "speedup", "summarize", "verify",
             "BlockPlan", "GateBlock", "KernelTrace", "finalize_outputs", "lstm_run_precomputed", "plan_blocks",
             "precompute_gates_qrnn", "precompute_gates_sru", "recurrence_sweep", "run_blocked",
             "CellKind", "CellState", "LstmWeights", "QrnnWeights", "SruWeights", "lstm_step", "qrnn_step",
             "run_stepwise", "sru_step", "zero_state", "Rng64", "gemm", "gemv", "sigmoid", "tanh_act",
             "uniform_weight", "PRESETS", "RnnConfig", "WeightSet", "count_params", "generate_sequence",
             "generate_weights", "load_sequence", "load_weights", "preset_config", "save_sequence",
             "save_weights", "TrafficReport", "estimate_traffic", "validate_against_trace", "weight_bytes"]
    missing = [n for n in names if not hasattr(P, n)]
    assert not missing, missing
    assert P.Rng64(0).next() == 0xE220A8397B1DCDAF
    assert P.uniform_weight(0) == -0.1
