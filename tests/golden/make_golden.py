"""Generate the golden fixtures under tests/golden/ FROM THE REFERENCE ITSELF.

Run in the build container only (the reference is not on the GPU box):

    NUMBA_CACHE_DIR=/tmp/nc PYTHONDONTWRITEBYTECODE=1 \
        python tests/golden/make_golden.py

It imports rnnblock from /root/reference/pkg/src (read-only, unmodified)
and writes:

* ``cells_d2.json``     -- the reference test-suite's hand-checked d=2 weight
                           sets and golden (h, c) vectors (pkg/tests/test_cells.py
                           SRU_GOLDEN / QRNN_GOLDEN), recomputed here through
                           ``run_layer_stepwise`` so the file holds what the
                           reference actually produces;
* ``splitmix.json``     -- SplitMix64 / uniform_weight known answers;
* ``blocked_cases.npz`` -- run_blocked(kernel="fast") and run_stepwise outputs
                           plus the final c (replayed with the public block
                           building blocks) for small seeded
                           SRU/QRNN cases incl. remainder blocks, T_b > L,
                           f32/f64 and stacks;
* ``baseline_cfg.npz``  -- the reference on BASELINE cfg1 (full) and cfg2
                           (c_T + row subsample), inputs from
                           paper_1803_11389_b200.workloads (seeded PCG64);
* ``lstm_cases.npz``    -- lstm_run_precomputed / run_stepwise on seeded
                           LSTM layers (weights and inputs included).
"""

import json
import os
import sys

os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
sys.dont_write_bytecode = True

import numpy as np

REF_SRC = "/root/reference/pkg/src"
REF_TESTS = "/root/reference/pkg/tests"
HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REF_SRC)
sys.path.insert(0, REPO)

import rnnblock as rb  # noqa: E402
from rnnblock import blocked as rbb  # noqa: E402
from rnnblock import cells as rbc  # noqa: E402
from rnnblock import kernels as rbk  # noqa: E402


def replay_final_state(cfg, ws, X, T):
    """c_T and x_carry per layer through the reference's own public block
    building blocks, in run_blocked's order (blocked.py:237-267)."""
    plan = rbb.plan_blocks(X.shape[0], T)
    layer_in = X
    cs, xcs = [], []
    for w in ws.layers:
        out = np.empty((plan.seq_len, w.d_h), layer_in.dtype)
        c = np.zeros(w.d_h, layer_in.dtype)
        xc = np.zeros(w.d_in, layer_in.dtype)
        for s, l in plan.blocks:
            Xb = np.ascontiguousarray(layer_in[s:s + l].T)
            if cfg.kind is rbc.CellKind.SRU:
                g = rbb.precompute_gates_sru(w, Xb, "fast")
            else:
                g = rbb.precompute_gates_qrnn(w, Xb, xc, "fast")
                xc = Xb[:, -1].copy()
            C = rbb.recurrence_sweep(g.forget, g.cand, c)
            c = C[:, -1].copy()
            H = rbb.finalize_outputs(cfg.kind, g, C, Xb if cfg.kind is rbc.CellKind.SRU else None)
            out[s:s + l] = H.T
        cs.append(c)
        xcs.append(xc)
        layer_in = out
    return layer_in, cs, xcs


def cells_d2():
    sys.path.insert(0, REF_TESTS)
    import test_cells as tc  # the reference's own test module (read only)
    out = {}
    sru = tc.sru_w2()
    X = np.array(tc.SRU_X4, np.float64)
    H = rbc.run_layer_stepwise(rbc.CellKind.SRU, sru, X)
    st = rbc.zero_state(2, 2, np.float64)
    cs = []
    for x in X:
        st = rbc.sru_step(sru, x, st)
        cs.append(st.c.tolist())
    out["sru"] = {
        "weights": {k: getattr(sru, k).tolist() for k in ("w_cand", "w_forget", "w_highway",
                                                         "b_forget", "b_highway")},
        "X": X.tolist(), "H": H.tolist(), "C": cs,
        "golden_published": tc.SRU_GOLDEN,
    }
    q = tc.qrnn_w2()
    Xq = np.array([[0.3, -0.5], [0.6, 0.2]], np.float64)
    Hq = rbc.run_layer_stepwise(rbc.CellKind.QRNN, q, Xq)
    st = rbc.zero_state(2, 2, np.float64)
    cs = []
    for x in Xq:
        st = rbc.qrnn_step(q, x, st)
        cs.append(st.c.tolist())
    out["qrnn"] = {
        "weights": {k: getattr(q, k).tolist() for k in ("w_cand", "w_cand_prev", "w_forget",
                                                       "w_forget_prev", "w_out", "w_out_prev")},
        "X": Xq.tolist(), "H": Hq.tolist(), "C": cs,
        "golden_published": tc.QRNN_GOLDEN,
    }
    lw = tc.lstm_w2()
    Xl = np.array([[0.5, -0.3], [-0.4, 0.2]], np.float64)
    st = rbc.zero_state(2, 2, np.float64)
    hs, cs = [], []
    for x in Xl:
        st = rbc.lstm_step(lw, x, st)
        hs.append(st.h.tolist())
        cs.append(st.c.tolist())
    out["lstm"] = {
        "weights": {k: getattr(lw, k).tolist() for k in LSTM_FIELDS},
        "X": Xl.tolist(), "H": hs, "C": cs,
        "H_precomputed_T1": rbb.lstm_run_precomputed(lw, Xl, 1).tolist(),
        "H_precomputed_T2": rbb.lstm_run_precomputed(lw, Xl, 2).tolist(),
        "golden_published": tc.LSTM_GOLDEN,
    }
    with open(os.path.join(HERE, "cells_d2.json"), "w") as f:
        json.dump(out, f, indent=1)


def splitmix():
    raws0 = rbk.raw_stream(0, 4)
    raws42 = rbk.raw_stream(42, 8)
    out = {
        "seed0_first4": [int(v) for v in raws0],
        "seed42_first8": [int(v) for v in raws42],
        "uniform_seed42_first8": [float(v) for v in rbk.uniform_array(raws42)],
        "uniform_weight_kat": {str(r): rbk.uniform_weight(r)
                               for r in (0, (1 << 64) - 1, 1 << 63, 0x123456789ABCDEF0)},
    }
    with open(os.path.join(HERE, "splitmix.json"), "w") as f:
        json.dump(out, f, indent=1)


CASES = [
    # kind, precision, d, L, n_layers, T_b list
    ("sru", "f32", 8, 1, 1, (1, 4)),
    ("sru", "f32", 16, 100, 1, (1, 3, 32, 128)),
    ("sru", "f32", 64, 256, 1, (1, 16, 64)),
    ("sru", "f64", 24, 64, 3, (8,)),
    ("sru", "f32", 32, 64, 2, (16,)),
    ("qrnn", "f32", 8, 5, 1, (1, 2, 8)),
    ("qrnn", "f32", 16, 100, 1, (1, 3, 32)),
    ("qrnn", "f32", 64, 256, 1, (1, 16, 64)),
    ("qrnn", "f64", 48, 96, 1, (16,)),
    ("qrnn", "f32", 33, 70, 2, (7, 32)),
]
WSEED, XSEED = 42, 43

LSTM_FIELDS = ("w_forget", "w_input", "w_output", "w_cand", "u_forget", "u_input", "u_output", "u_cand",
               "b_forget", "b_input", "b_output", "b_cand")
LSTM_CASES = [
    # precision, d_in, d_h, L, T_b list
    ("f32", 8, 8, 16, (1, 4, 16)),
    ("f32", 64, 64, 128, (1, 16, 128)),
    ("f32", 96, 160, 75, (8, 32)),
    ("f64", 32, 48, 40, (1, 7)),
    ("f32", 350, 350, 64, (16,)),
]


def lstm_cases():
    """lstm_run_precomputed (kernel="fast") per T_b and run_stepwise for
    seeded LSTM layers (weights generated by the reference)."""
    arrays, index = {}, []
    for n, (prec, din, dh, L, Tbs) in enumerate(LSTM_CASES):
        cfg = rb.RnnConfig(rbc.CellKind.LSTM, din, dh, n_layers=1, precision=prec)
        ws = rb.generate_weights(cfg, 700 + n)
        X = rb.generate_sequence(L, din, 800 + n, prec)
        if din * dh <= 160 * 160:  # larger weight sets are regenerated by the oracle's SplitMix64 restatement
            for f in LSTM_FIELDS:
                arrays[f"l{n}_{f}"] = getattr(ws.layers[0], f)
        arrays[f"l{n}_X"] = X
        arrays[f"l{n}_stepwise"] = rb.run_stepwise(cfg, ws, X)
        for T in Tbs:
            arrays[f"l{n}_T{T}_H"] = rbb.lstm_run_precomputed(ws.layers[0], X, T, kernel="fast")
        index.append({"case": n, "precision": prec, "d_in": din, "d_h": dh, "L": L, "T_b": list(Tbs),
                      "wseed": 700 + n, "xseed": 800 + n})
    np.savez_compressed(os.path.join(HERE, "lstm_cases.npz"), **arrays)
    with open(os.path.join(HERE, "lstm_cases.json"), "w") as f:
        json.dump(index, f, indent=1)


def blocked_cases():
    arrays = {}
    index = []
    for n, (kind, prec, d, L, nl, Tbs) in enumerate(CASES):
        cfg = rb.RnnConfig(rbc.CellKind.parse(kind), d, d, n_layers=nl, precision=prec)
        ws = rb.generate_weights(cfg, WSEED + n)
        X = rb.generate_sequence(L, d, XSEED + n, prec)
        step = rb.run_stepwise(cfg, ws, X)
        arrays[f"c{n}_stepwise"] = step
        for T in Tbs:
            H = rb.run_blocked(cfg, ws, X, T, kernel="fast")
            H2, cs, xcs = replay_final_state(cfg, ws, X, T)
            assert H.tobytes() == H2.tobytes()
            arrays[f"c{n}_T{T}_H"] = H
            arrays[f"c{n}_T{T}_c"] = np.stack(cs)
            if kind == "qrnn":
                arrays[f"c{n}_T{T}_xc"] = np.stack(xcs)
        index.append({"case": n, "kind": kind, "precision": prec, "d": d, "L": L,
                      "n_layers": nl, "T_b": list(Tbs), "wseed": WSEED + n, "xseed": XSEED + n})
    np.savez_compressed(os.path.join(HERE, "blocked_cases.npz"), **arrays)
    with open(os.path.join(HERE, "blocked_cases.json"), "w") as f:
        json.dump(index, f, indent=1)


def baseline_cfgs():
    from paper_1803_11389_b200 import workloads
    out = {}
    w1 = workloads.make("cfg1")
    cfg = rb.RnnConfig(rbc.CellKind.SRU, 512, 512, precision="f32")
    ws = rb.WeightSet(rbc.CellKind.SRU, "f32", [rbc.SruWeights(*lay.mats()) for lay in w1.layers])
    for T in (1, 4, 16):
        H, cs, _ = replay_final_state(cfg, ws, w1.X, T)
        out[f"cfg1_T{T}_c"] = cs[0]
        if T == 16:
            out["cfg1_T16_H"] = H
    w2 = workloads.make("cfg2")
    cfg = rb.RnnConfig(rbc.CellKind.QRNN, 1024, 1024, precision="f32")
    ws = rb.WeightSet(rbc.CellKind.QRNN, "f32", [rbc.QrnnWeights(*lay.mats()) for lay in w2.layers])
    H, cs, _ = replay_final_state(cfg, ws, w2.X, 32)
    rows = np.arange(0, 2048, 61)
    out["cfg2_T32_rows"] = rows
    out["cfg2_T32_Hrows"] = H[rows]
    out["cfg2_T32_c"] = cs[0]
    out["cfg2_T32_Hsum"] = np.array([H.astype(np.float64).sum()])
    np.savez_compressed(os.path.join(HERE, "baseline_cfg.npz"), **out)


def model_files():
    """Reference-written RNNW / RNNX files (model_io.save_weights /
    save_sequence) for the file-format tests."""
    from rnnblock import model_io as rbm
    specs = [("sru2_f32.rnnw", "sru", 24, 24, 2, "f32", 31), ("qrnn1_f64.rnnw", "qrnn", 20, 12, 1, "f64", 32),
             ("lstm1_f32.rnnw", "lstm", 10, 14, 1, "f32", 33)]
    index = {}
    for name, kind, din, dh, nl, prec, seed in specs:
        cfg = rb.RnnConfig(rbc.CellKind.parse(kind), din, dh, n_layers=nl, precision=prec)
        rbm.save_weights(rb.generate_weights(cfg, seed), os.path.join(HERE, name))
        index[name] = {"kind": kind, "d_in": din, "d_h": dh, "n_layers": nl, "precision": prec, "seed": seed}
    for name, L, W, prec, seed in (("seq_f32.rnnx", 37, 24, "f32", 34), ("seq_f64.rnnx", 11, 20, "f64", 35)):
        rbm.save_sequence(rb.generate_sequence(L, W, seed, prec), os.path.join(HERE, name))
        index[name] = {"seq_len": L, "width": W, "precision": prec, "seed": seed}
    with open(os.path.join(HERE, "model_files.json"), "w") as f:
        json.dump(index, f, indent=1)


def traffic():
    """estimate_traffic / expected_phase_touches / lstm_split_bytes of the
    reference's traffic model for a grid of configs."""
    from rnnblock import traffic as rbt
    out = []
    for kind, din, dh, nl, prec in (("sru", 512, 512, 1, "f32"), ("qrnn", 1024, 1024, 1, "f32"),
                                    ("lstm", 350, 350, 2, "f32"), ("qrnn", 300, 200, 3, "f64"),
                                    ("lstm", 64, 96, 1, "f64")):
        cfg = rb.RnnConfig(rbc.CellKind.parse(kind), din, dh, n_layers=nl, precision=prec)
        for L, T in ((2048, 1), (2048, 32), (1000, 7), (5, 64)):
            r = rbt.estimate_traffic(cfg, L, T)
            row = {"kind": kind, "d_in": din, "d_h": dh, "n_layers": nl, "precision": prec, "L": L, "T": T,
                   "weight_bytes": r.weight_bytes, "blocks": r.blocks, "est": r.est_weight_traffic,
                   "per_step": r.per_step_traffic, "ratio": r.ratio_vs_t1,
                   "touches": rbt.expected_phase_touches(cfg, L, T)}
            if kind == "lstm":
                row["split"] = list(rbt.lstm_split_bytes(cfg))
            out.append(row)
    with open(os.path.join(HERE, "traffic.json"), "w") as f:
        json.dump(out, f, indent=1)


def bench_csv():
    """emit_csv of fixed rows by the reference (bench.py:194-229)."""
    import importlib
    rbbench = importlib.import_module("rnnblock.bench")
    from rnnblock import traffic as rbt
    recs = [rbbench.BenchRecord("qrnn", "blocked", 16, 16, 64, T, 8, r, 10.0 / T + 0.25 * r)
            for T in (1, 4) for r in range(3)]
    rbbench.emit_csv(recs, os.path.join(HERE, "bench_records.csv"), kind="records")
    rows = rbbench.summarize(recs) + [rbbench.SpeedupRow("LSTM", 673.667, None)]
    rbbench.emit_csv(rows, os.path.join(HERE, "bench_summary.csv"), kind="summary")
    cfg = rb.RnnConfig(rbc.CellKind.QRNN, 64, 64, precision="f32")
    rbbench.emit_csv([rbt.estimate_traffic(cfg, 100, T) for T in (1, 8)], os.path.join(HERE, "bench_traffic.csv"),
                     kind="traffic")


if __name__ == "__main__":
    parts = sys.argv[1:] or ["cells_d2", "splitmix", "blocked_cases", "baseline_cfgs", "lstm_cases", "model_files", "traffic", "bench_csv"]
    for part in parts:
        globals()[part]()
    print("golden fixtures written to", HERE, parts)
