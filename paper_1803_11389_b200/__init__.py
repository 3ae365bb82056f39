"""B200-native single-stream blocked SRU/QRNN inference (arXiv 1803.11389).

Drop-in for the reference package's blocked path (rnnblock ``run_blocked``
and its unit-level ops, types and trace contract).  All compute runs in
hand-written sm_100a CUDA kernels in ``librnnb.so`` behind a C ABI
(include/rnnb.h); there is no CPU fallback.

Fast path: ``DeviceStack`` (weights resident in HBM, forward on device
tensors).  Drop-in path: ``run_blocked(cfg, weights, X, block_size)``.
LSTM partial precompute: ``lstm_run_precomputed`` / ``DeviceLstm``.
"""

from .blocked import (
    PHASE_BIAS,
    PHASE_GEMM,
    PHASE_GEMV,
    BlockPlan,
    GateBlock,
    KernelTrace,
    TraceEvent,
    finalize_outputs,
    lstm_run_precomputed,
    plan_blocks,
    precompute_gates_qrnn,
    precompute_gates_sru,
    recurrence_sweep,
    run_blocked,
)
from .cells import (
    PRECISIONS,
    CellKind,
    CellState,
    LstmWeights,
    QrnnWeights,
    RnnConfig,
    SruWeights,
    WeightSet,
    zero_state,
)
from .device import DeviceLstm, DeviceStack
from .bench_gpu import BenchRecord, BenchResult, SpeedupRow, bench, emit_csv, speedup, summarize, verify
from .kernels import Rng64, gemm, gemv, sigmoid, tanh_act, uniform_weight
from .model_io import (
    PRESETS,
    count_params,
    generate_sequence,
    generate_weights,
    load_sequence,
    load_weights,
    preset_config,
    save_sequence,
    save_weights,
)
from .stepwise import lstm_step, qrnn_step, run_stepwise, sru_step
from .traffic import TrafficReport, estimate_traffic, validate_against_trace, weight_bytes

__version__ = "0.1.0"

__all__ = [
    "PHASE_BIAS", "PHASE_GEMM", "PHASE_GEMV", "BlockPlan", "GateBlock", "KernelTrace",
    "TraceEvent", "finalize_outputs", "lstm_run_precomputed", "plan_blocks",
    "precompute_gates_qrnn", "precompute_gates_sru", "recurrence_sweep", "run_blocked",
    "PRECISIONS", "CellKind", "CellState", "QrnnWeights", "RnnConfig", "SruWeights",
    "WeightSet", "zero_state", "DeviceStack", "LstmWeights", "DeviceLstm",
    # the rest of rnnblock's top-level names (rnnblock/__init__.py)
    "BenchRecord", "BenchResult", "SpeedupRow", "bench", "emit_csv", "speedup", "summarize", "verify",
    "Rng64", "gemm", "gemv", "sigmoid", "tanh_act", "uniform_weight",
    "PRESETS", "count_params", "generate_sequence", "generate_weights", "load_sequence", "load_weights",
    "preset_config", "save_sequence", "save_weights",
    "lstm_step", "qrnn_step", "run_stepwise", "sru_step",
    "TrafficReport", "estimate_traffic", "validate_against_trace", "weight_bytes",
]
