"""GPU rows in the reference's bench / CSV surface.

A separate tool (no backend dispatch inside the reference API): the same
record / summary / traffic CSV schemas (rnnblock bench.py:183-229), the same
T=1 speed-up convention (bench.py:50-54, 100 * median(T=1) / median(T)) and
the same verify-before-timing rule and exit codes as ``rnnblock bench``
(cli.py:1-11), with rows timed on the GPU by CUDA events.

Verification needs no CPU oracle: every block size is checked against the
f64 GPU run at T=1 (the most accurate path of this build) with the
reference's ORACLE_TOLERANCE.

    python -m paper_1803_11389_b200.bench_gpu bench --cell qrnn --preset large --seq-len 2048 --out q.csv
"""

import argparse
import csv
import statistics
import sys
from dataclasses import dataclass, field

import numpy as np

from . import model_io
from .cells import CellKind, LstmWeights, QrnnWeights, RnnConfig, SruWeights, WeightSet
from .traffic import MODEL_ASSUMPTION, TrafficReport, estimate_traffic

ORACLE_TOLERANCE = {"f32": 1e-4, "f64": 1e-9}
IMPLS = ("gpu-blocked", "gpu-lstm-precomputed")
DEFAULT_BLOCKS = "1,2,4,8,16,32,64,128"
PRESET_WIDTH = {CellKind.LSTM: {"small": 350, "large": 700}, CellKind.SRU: {"small": 512, "large": 1024},
                CellKind.QRNN: {"small": 512, "large": 1024}}


@dataclass(frozen=True)
class BenchRecord:
    cell: str
    impl: str
    d_in: int
    d_h: int
    seq_len: int
    block: int
    threads: int      # GPU rows: streaming multiprocessors of the device
    repeat: int
    elapsed_ms: float


@dataclass(frozen=True)
class SpeedupRow:
    label: str
    median_ms: float
    speedup_pct: float = None


def speedup(base_ms: float, t_ms: float) -> float:
    """100 * base / t, one decimal place (bench.py:50-54)."""
    if base_ms <= 0 or t_ms <= 0:
        raise ValueError("times must be positive")
    return round(100.0 * base_ms / t_ms, 1)


@dataclass(frozen=True)
class VerifyRow:
    block: int
    max_abs_diff: float
    tolerance: float
    passed: bool


@dataclass
class VerifyReport:
    cell: str
    precision: str
    seq_len: int
    rows: list = field(default_factory=list)

    @property
    def passed(self) -> bool:
        return all(r.passed for r in self.rows)


def _runner(cfg, weights, precision):
    """Device handles for the network; returns fn(X_device, T) -> H_device."""
    from .device import DeviceLstm, DeviceStack
    if cfg.kind is CellKind.LSTM:
        devs = [DeviceLstm(w, mode=precision) for w in weights.layers]

        def run(X, T):
            for d in devs:
                X = d.forward(X, T)
            return X
        return run, devs
    st = DeviceStack(cfg.kind, weights.layers, mode=precision)
    return (lambda X, T: st.forward(X, T)), [st]


def verify(cfg, weights, X, t_list, tolerance=None) -> VerifyReport:
    import torch
    tol = ORACLE_TOLERANCE[cfg.precision] if tolerance is None else tolerance
    ref_run, ref_devs = _runner(cfg, _cast(weights, "f64"), "f64")
    ref = ref_run(torch.from_numpy(np.asarray(X, np.float64)).cuda(), 1).cpu().numpy()
    run, devs = _runner(cfg, weights, cfg.precision)
    Xd = torch.from_numpy(np.ascontiguousarray(X)).cuda()
    report = VerifyReport(cell=cfg.kind.value, precision=cfg.precision, seq_len=X.shape[0])
    for T in t_list:
        diff = float(np.max(np.abs(run(Xd, T).cpu().numpy().astype(np.float64) - ref)))
        report.rows.append(VerifyRow(block=T, max_abs_diff=diff, tolerance=tol, passed=diff <= tol))
    for d in ref_devs + devs:
        d.close()
    return report


def _cast(weights, precision):
    dt = np.float64 if precision == "f64" else np.float32
    cls = type(weights.layers[0])
    return WeightSet(weights.kind, precision, [cls(*[np.asarray(m, dt) for m in lay.mats()]) for lay in weights.layers])


@dataclass
class BenchResult:
    records: list = field(default_factory=list)
    summaries: list = field(default_factory=list)
    warnings: list = field(default_factory=list)
    threads: int = 0


def bench(cfg, weights, X, t_list, repeats: int = 5, threads: int = 1, warmup: int = 1) -> BenchResult:
    """CUDA-event timed forwards of the whole sequence per block size
    (bench.py:124-153's signature; `threads`, the reference's CPU worker
    count, is validated and otherwise unused: the GPU result and timing do
    not depend on it, and records carry the multiprocessor count)."""
    import torch
    if repeats < 1:
        raise ValueError("repeats must be >= 1")
    if threads < 1:
        raise ValueError("threads must be >= 1")
    sms = torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count
    result = BenchResult(threads=sms)
    impl = "gpu-lstm-precomputed" if cfg.kind is CellKind.LSTM else "gpu-blocked"
    run, devs = _runner(cfg, weights, cfg.precision)
    Xd = torch.from_numpy(np.ascontiguousarray(X)).cuda()
    for T in t_list:
        for _ in range(warmup):
            run(Xd, T)
        torch.cuda.synchronize()
        for rep in range(repeats):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            run(Xd, T)
            e1.record()
            torch.cuda.synchronize()
            result.records.append(BenchRecord(cell=cfg.kind.value, impl=impl, d_in=cfg.d_in, d_h=cfg.d_h,
                                              seq_len=X.shape[0], block=T, threads=sms, repeat=rep,
                                              elapsed_ms=float(e0.elapsed_time(e1))))
    for d in devs:
        d.close()
    result.summaries = summarize(result.records)
    return result


def summarize(records) -> list:
    """One SpeedupRow per (cell, impl, block) in first-seen order: the median
    time and the speed-up against the same (cell, impl) at block 1."""
    times = {}
    for r in records:
        times.setdefault((r.cell, r.impl, r.block), []).append(r.elapsed_ms)
    med = {key: statistics.median(ts) for key, ts in times.items()}
    return [SpeedupRow(label=f"{cell.upper()}-{block}", median_ms=m,
                       speedup_pct=None if (cell, impl, 1) not in med else speedup(med[(cell, impl, 1)], m))
            for (cell, impl, block), m in med.items()]


@dataclass(frozen=True)
class _Schema:
    """A CSV layout: the row type it accepts and (header, cell formatter) per column."""
    row_type: type
    columns: tuple

    @property
    def header(self):
        return [name for name, _ in self.columns]

    def cells(self, row):
        return [fmt(row) for _, fmt in self.columns]


def _attr(name, fmt=str):
    return lambda row: fmt(getattr(row, name))


# The reference's record / summary / traffic CSV layouts (its bench CSVs are
# pinned byte for byte by tests/golden/bench_*.csv): floats keep repr().
_SCHEMAS = {
    "records": _Schema(BenchRecord, tuple((c, _attr(c, repr if c == "elapsed_ms" else str)) for c in (
        "cell", "impl", "d_in", "d_h", "seq_len", "block", "threads", "repeat", "elapsed_ms"))),
    "summary": _Schema(SpeedupRow, (
        ("label", _attr("label")), ("median_ms", _attr("median_ms", repr)),
        ("speedup_pct", lambda r: "-" if r.speedup_pct is None else f"{r.speedup_pct:.1f}"))),
    "traffic": _Schema(TrafficReport, (
        ("cell", lambda r: r.config.kind.value), ("d_h", lambda r: str(r.config.d_h)),
        ("precision", lambda r: r.config.precision), ("L", _attr("seq_len")), ("T", _attr("block_size")),
        ("weight_bytes", _attr("weight_bytes")), ("blocks", _attr("blocks")),
        ("est_traffic_bytes", _attr("est_weight_traffic")), ("ratio_vs_T1", _attr("ratio_vs_t1", repr)))),
}


def _schema_for(row):
    for name, sch in _SCHEMAS.items():
        if isinstance(row, sch.row_type):
            return name
    raise ValueError(f"no CSV layout for {type(row).__name__}")


def emit_csv(rows, path, kind: str = None) -> None:
    """Write records, summary rows or traffic reports under the layout's
    fixed header (one row type per file)."""
    if kind is None:
        if not rows:
            raise ValueError("empty row list needs an explicit kind")
        kind = _schema_for(rows[0])
    if kind not in _SCHEMAS:
        raise ValueError(f"unknown CSV kind {kind!r}")
    sch = _SCHEMAS[kind]
    if any(_schema_for(r) != kind for r in rows):
        raise ValueError("mixed row types in one CSV")
    with open(path, "w", newline="") as f:
        w = csv.writer(f)
        w.writerow(sch.header)
        w.writerows(sch.cells(r) for r in rows)


_TABLE = (("Model", "<12", lambda r: r.label), ("Median (ms)", ">12", lambda r: f"{r.median_ms:.3f}"),
          ("Speed-up", ">10", lambda r: "-" if r.speedup_pct is None else f"{r.speedup_pct:.1f}%"))


def format_summary_table(rows) -> str:
    head = " ".join(f"{name:{align}}" for name, align, _ in _TABLE)
    body = [" ".join(f"{cell(r):{align}}" for _, align, cell in _TABLE) for r in rows]
    return "\n".join([head] + body)


# ---------------------------------------------------------------------------
# CLI (cli.py conventions: exit 0 ok, 1 verification failure, 2 bad args, 3 I/O)


def _blocks(text):
    try:
        b = [int(v) for v in text.split(",") if v.strip()]
    except ValueError:
        raise SystemExit(2)
    if not b or any(v < 1 for v in b):
        raise SystemExit(2)
    return b


def _model(args):
    """cli.py:100-130: weights from generate_weights(cfg, seed) (the
    reference's SplitMix64 stream, generated on the GPU: byte-identical to
    rnnblock's for the same seed) or a file; the input from
    generate_sequence(seq_len, d_in, seed + 1) or a file."""
    if args.weights:
        ws = model_io.load_weights(args.weights)
        cfg = model_io.config_of(ws)
    else:
        kind = CellKind.parse(args.cell)
        d = args.width or PRESET_WIDTH[kind][args.preset]
        cfg = RnnConfig(kind, d, d, n_layers=args.layers, precision=args.precision)
        ws = model_io.generate_weights(cfg, args.seed)
    if args.input:
        X = model_io.load_sequence(args.input)
    else:
        X = model_io.generate_sequence(args.seq_len, cfg.d_in, args.seed + 1, cfg.precision)
    return cfg, ws, X


def main(argv=None):
    p = argparse.ArgumentParser(prog="paper_1803_11389_b200.bench_gpu")
    sub = p.add_subparsers(dest="cmd", required=True)
    g = sub.add_parser("gen-weights", help="generate a weight file (cli.py:144-148)")
    g.add_argument("--cell", choices=["lstm", "sru", "qrnn"], default="qrnn")
    g.add_argument("--preset", choices=["small", "large"], default="small")
    g.add_argument("--width", type=int)
    g.add_argument("--layers", type=int, default=1)
    g.add_argument("--precision", choices=["f32", "f64"], default="f32")
    g.add_argument("--seed", type=int, default=42)
    g.add_argument("--out", required=True)
    g = sub.add_parser("gen-seq", help="generate an input-sequence file (cli.py:151-155)")
    g.add_argument("--seq-len", type=int, default=1024)
    g.add_argument("--width", type=int, required=True)
    g.add_argument("--precision", choices=["f32", "f64"], default="f32")
    g.add_argument("--seed", type=int, default=42)
    g.add_argument("--out", required=True)
    for name in ("bench", "verify", "traffic"):
        s = sub.add_parser(name)
        s.add_argument("--cell", choices=["lstm", "sru", "qrnn"], default="qrnn")
        s.add_argument("--preset", choices=["small", "large"], default="small")
        s.add_argument("--width", type=int)
        s.add_argument("--layers", type=int, default=1)
        s.add_argument("--precision", choices=["f32", "f64"], default="f32")
        s.add_argument("--seed", type=int, default=42)
        s.add_argument("--seq-len", type=int, default=1024)
        s.add_argument("--blocks", default=DEFAULT_BLOCKS)
        s.add_argument("--weights")
        s.add_argument("--input")
        s.add_argument("--out")
        if name == "bench":
            s.add_argument("--repeats", type=int, default=5)
            s.add_argument("--skip-verify", action="store_true")
            # cli.py's CPU worker count; accepted for drop-in use, the GPU
            # kernels' results never depend on a thread count
            s.add_argument("--threads", type=int, default=1)
    args = p.parse_args(argv)
    if args.cmd == "gen-weights":
        kind = CellKind.parse(args.cell)
        d = args.width or PRESET_WIDTH[kind][args.preset]
        try:
            cfg = RnnConfig(kind, d, d, n_layers=args.layers, precision=args.precision)
        except ValueError as e:
            print(f"error: {e}", file=sys.stderr)
            return 2
        model_io.save_weights(model_io.generate_weights(cfg, args.seed), args.out)
        print(f"wrote {cfg.precision} {cfg.kind.value} weights (d={cfg.d_h}) to {args.out}")
        return 0
    if args.cmd == "gen-seq":
        try:
            X = model_io.generate_sequence(args.seq_len, args.width, args.seed, args.precision)
        except ValueError as e:
            print(f"error: {e}", file=sys.stderr)
            return 2
        model_io.save_sequence(X, args.out)
        print(f"wrote {args.seq_len}x{args.width} {args.precision} sequence to {args.out}")
        return 0
    try:
        cfg, ws, X = _model(args)
    except model_io.FileFormatError as e:
        print(f"error: {e}", file=sys.stderr)
        return 3
    except OSError as e:
        print(f"error: {e}", file=sys.stderr)
        return 3
    blocks = _blocks(args.blocks)
    if args.cmd == "traffic":
        reps = [estimate_traffic(cfg, X.shape[0], T) for T in blocks]
        print(f"model assumption: {MODEL_ASSUMPTION}")
        for r in reps:
            print(f"T={r.block_size:<4d} blocks={r.blocks:<5d} est={r.est_weight_traffic:>14,d} B  "
                  f"ratio_vs_T1={r.ratio_vs_t1:.6f}")
        if args.out:
            emit_csv(reps, args.out, kind="traffic")
        return 0
    if args.cmd == "verify" or not args.skip_verify:
        rep = verify(cfg, ws, X, blocks)
        for r in rep.rows:
            print(f"T={r.block:<4d} max|diff|={r.max_abs_diff:.3e} tol={r.tolerance:g} "
                  f"{'ok' if r.passed else 'FAIL'}")
        if not rep.passed:
            print("refusing to time an unverified configuration", file=sys.stderr)
            return 1
        if args.cmd == "verify":
            return 0
    res = bench(cfg, ws, X, blocks, repeats=args.repeats)
    print(format_summary_table(res.summaries))
    if args.out:
        raw = args.out[:-4] + ".raw.csv" if args.out.endswith(".csv") else args.out + ".raw.csv"
        emit_csv(res.summaries, args.out, kind="summary")
        emit_csv(res.records, raw, kind="records")
        print(f"wrote {args.out} and {raw}")
    return 0


if __name__ == "__main__":
    sys.exit(main())
