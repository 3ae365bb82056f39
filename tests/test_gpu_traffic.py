"""The trace contract end to end: a GPU run's KernelTrace validates against
the reference traffic model (traffic.validate_against_trace), per phase."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("kind,stack", [("sru", False), ("sru", True), ("qrnn", False), ("qrnn", True), ("lstm", False)])
def test_trace_validates(oracle, kind, stack):
    import paper_1803_11389_b200 as P
    from paper_1803_11389_b200 import traffic
    d, L, T = 16, 50, 8
    cfg = P.RnnConfig(P.CellKind.parse(kind), d, d, n_layers=1 if kind == "lstm" else 2, precision="f32")
    layers = oracle.generate_layers(kind, d, d, cfg.n_layers, 3, np.float32)
    X = oracle.generate_sequence(L, d, 4, np.float32)
    trace = P.KernelTrace()
    if kind == "lstm":
        P.lstm_run_precomputed(P.LstmWeights(*layers[0]), X, T, trace=trace)
    else:
        cls = P.SruWeights if kind == "sru" else P.QrnnWeights
        ws = P.WeightSet(cfg.kind, "f32", [cls(*m) for m in layers])
        P.run_blocked(cfg, ws, X, T, trace=trace, stack_gates=stack)
    cmp = traffic.validate_against_trace(traffic.estimate_traffic(cfg, L, T), trace)
    assert cmp.ok, cmp
