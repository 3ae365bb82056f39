"""Drop-in blocked executor API (rnnblock blocked.py) on the B200 kernels.

Same names, signatures, return types and ``ValueError`` conditions as the
reference's blocked.py, so reference callers and tests can switch imports:

  plan_blocks / BlockPlan          blocked.py:31-50
  GateBlock                        blocked.py:53-71
  KernelTrace / TraceEvent, PHASE_* blocked.py:74-108
  precompute_gates_sru / _qrnn     blocked.py:123-150   -> rnnb_gates
  recurrence_sweep                 blocked.py:165-176   -> rnnb_sweep
  finalize_outputs                 blocked.py:179-193   -> rnnb_finalize
  run_blocked                      blocked.py:221-268   -> rnnb_forward_host

Every call goes through librnnb.so on the GPU; there is no CPU path.  The
``kernel`` argument is validated like the reference's (kernels.py:213-224)
but selects nothing: there is one CUDA implementation.  ``trace`` receives
the same events the reference logs for the chosen ``stack_gates`` (one per
logical weight-touching product / bias add), so the traffic model's
``validate_against_trace`` keeps working; the CUDA side fuses them into one
launch per layer.
"""

import ctypes
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .cells import LSTM_FIELDS, CellKind, LstmWeights
from .device import DeviceLstm, DeviceStack, _stream_ptr

KERNELS = ("reference", "tiled", "fast")

PHASE_GEMM = "precompute.gemm"
PHASE_BIAS = "precompute.bias"
PHASE_GEMV = "recurrent.gemv"


@dataclass(frozen=True)
class BlockPlan:
    seq_len: int
    block_size: int
    blocks: tuple  # ordered (start, length) ranges tiling [0, seq_len)


def plan_blocks(seq_len: int, block_size: int) -> BlockPlan:
    """ceil(seq_len / block_size) blocks; the last one takes the remainder."""
    if seq_len < 1:
        raise ValueError("seq_len must be >= 1")
    if block_size < 1:
        raise ValueError("block_size must be >= 1")
    blocks = tuple((s, min(block_size, seq_len - s)) for s in range(0, seq_len, block_size))
    return BlockPlan(seq_len=seq_len, block_size=block_size, blocks=blocks)


@dataclass
class GateBlock:
    """Per-block gate values, one column per time step (cand, forget, out_gate)."""

    cand: np.ndarray
    forget: np.ndarray
    out_gate: np.ndarray

    def __post_init__(self):
        if not (self.cand.shape == self.forget.shape == self.out_gate.shape):
            raise ValueError("gate matrices must share one shape")

    @property
    def length(self):
        return self.cand.shape[1]


@dataclass(frozen=True)
class TraceEvent:
    phase: str
    m: int
    k: int
    n: int

    def line(self) -> str:
        return f"{self.phase},{self.m},{self.k},{self.n}"


@dataclass
class KernelTrace:
    """Call log of the weight-touching operations of a run."""

    events: list = field(default_factory=list)

    def add(self, phase: str, m: int, k: int, n: int) -> None:
        self.events.append(TraceEvent(phase, m, k, n))

    def lines(self):
        return [e.line() for e in self.events]

    def count(self, phase: str) -> int:
        return sum(1 for e in self.events if e.phase == phase)

    def touches(self, phase: str = None) -> int:
        return sum(e.m * e.k for e in self.events if phase is None or e.phase == phase)


# ---------------------------------------------------------------------------
# argument checks with the reference's ValueError conditions


def _check_kernel(kernel):
    if kernel not in KERNELS:
        raise ValueError(f"unknown kernel {kernel!r}")


def _check_matrix(a, name):
    if not isinstance(a, np.ndarray) or a.ndim != 2:
        raise ValueError(f"{name} must be a 2-d ndarray")
    if a.shape[0] < 1 or a.shape[1] < 1:
        raise ValueError(f"{name} must have at least one row and one column")
    if not a.flags.c_contiguous:
        raise ValueError(f"{name} must be C-contiguous (row-major)")


def _mode_for(dtype):
    dtype = np.dtype(dtype)
    if dtype == np.float32:
        return "f32"
    if dtype == np.float64:
        return "f64"
    raise ValueError(f"unsupported dtype {dtype}")


def _check_layer_dtypes(layer, fields, dtype):
    for f in fields:
        a = getattr(layer, f)
        if np.asarray(a).dtype != dtype:
            raise ValueError(f"dtype mismatch: {np.asarray(a).dtype} vs {dtype}")
    for f in fields:
        a = getattr(layer, f)
        if np.ndim(a) == 2:
            _check_matrix(a, f)


def _sru_fields():
    return ("w_cand", "w_forget", "w_highway", "b_forget", "b_highway")


def _qrnn_fields():
    return ("w_cand", "w_cand_prev", "w_forget", "w_forget_prev", "w_out", "w_out_prev")


def _trace_block(trace, kind, w, l, stack_gates):
    """The events the reference logs for one block (blocked.py:111-120,
    123-150, 200-218)."""
    if trace is None:
        return
    d_h, d_in = w.d_h, w.d_in
    if kind is CellKind.SRU:
        if stack_gates:
            trace.add(PHASE_GEMM, 3 * d_h, d_in, l)
            trace.add(PHASE_BIAS, d_h, 1, l)
            trace.add(PHASE_BIAS, d_h, 1, l)
        else:
            trace.add(PHASE_GEMM, d_h, d_in, l)
            trace.add(PHASE_GEMM, d_h, d_in, l)
            trace.add(PHASE_BIAS, d_h, 1, l)
            trace.add(PHASE_GEMM, d_h, d_in, l)
            trace.add(PHASE_BIAS, d_h, 1, l)
    else:
        if stack_gates:
            trace.add(PHASE_GEMM, 3 * d_h, d_in, l)
            trace.add(PHASE_GEMM, 3 * d_h, d_in, l)
        else:
            for _ in range(6):
                trace.add(PHASE_GEMM, d_h, d_in, l)


# ---------------------------------------------------------------------------
# unit-level ops


def _torch():
    import torch
    return torch


def precompute_gates_sru(w, Xb: np.ndarray, kernel: str = "fast", trace: KernelTrace = None,
                         *, mode: str = None) -> GateBlock:
    """Gate values for a block of inputs (columns of Xb): one fused launch."""
    if Xb.ndim != 2 or Xb.shape[0] != w.d_in:
        raise ValueError(f"input block must be [{w.d_in} x T], got {Xb.shape}")
    _check_kernel(kernel)
    _check_layer_dtypes(w, _sru_fields(), Xb.dtype)
    _trace_block(trace, CellKind.SRU, w, Xb.shape[1], False)
    return _gates(CellKind.SRU, w, Xb, None, mode or _mode_for(Xb.dtype))


def precompute_gates_qrnn(w, Xb: np.ndarray, x_carry: np.ndarray, kernel: str = "fast",
                          trace: KernelTrace = None, *, mode: str = None) -> GateBlock:
    """Two-tap gate values for a block; x_carry is the input just before it."""
    if Xb.ndim != 2 or Xb.shape[0] != w.d_in:
        raise ValueError(f"input block must be [{w.d_in} x T], got {Xb.shape}")
    if x_carry.shape != (w.d_in,):
        raise ValueError(f"x_carry must have length {w.d_in}")
    _check_kernel(kernel)
    _check_layer_dtypes(w, _qrnn_fields(), Xb.dtype)
    _trace_block(trace, CellKind.QRNN, w, Xb.shape[1], False)
    return _gates(CellKind.QRNN, w, Xb, x_carry, mode or _mode_for(Xb.dtype))


def _gates(kind, w, Xb, x_carry, mode):
    torch = _torch()
    st = DeviceStack(kind, [w], mode=mode)
    try:
        Xt = torch.from_numpy(np.ascontiguousarray(Xb.T, dtype=st.np_dtype)).cuda()
        xc = None
        if x_carry is not None:
            xc = torch.from_numpy(np.ascontiguousarray(x_carry, dtype=st.np_dtype)).cuda()
        G = st.gates(0, Xt, xc).cpu().numpy().astype(Xb.dtype, copy=False)
    finally:
        st.close()
    return GateBlock(cand=np.ascontiguousarray(G[0]), forget=np.ascontiguousarray(G[1]),
                     out_gate=np.ascontiguousarray(G[2]))


def _dev(a, dtype):
    torch = _torch()
    return torch.from_numpy(np.ascontiguousarray(a, dtype=dtype)).cuda()


def recurrence_sweep(forget: np.ndarray, cand: np.ndarray, c_init: np.ndarray) -> np.ndarray:
    """Resolve c_t = f_t*c_{t-1} + (1-f_t)*cand_t across the block (GPU)."""
    if forget.ndim != 2 or forget.shape != cand.shape:
        raise ValueError("forget and candidate blocks must share one 2-d shape")
    if c_init.shape != (forget.shape[0],):
        raise ValueError("c_init length must match the block height")
    torch = _torch()
    dt = forget.dtype if forget.dtype in (np.float32, np.float64) else np.float64
    F, Xh, c0 = _dev(forget, dt), _dev(cand, dt), _dev(c_init, dt)
    C = torch.empty_like(F)
    lib = _lib.load()
    _lib.check(lib.rnnb_sweep(ctypes.c_void_p(F.data_ptr()), ctypes.c_void_p(Xh.data_ptr()),
                              ctypes.c_void_p(c0.data_ptr()), ctypes.c_void_p(C.data_ptr()),
                              F.shape[0], F.shape[1],
                              _lib.DT_F64 if dt == np.float64 else _lib.DT_F32, _stream_ptr(None)))
    return C.cpu().numpy()


def finalize_outputs(kind: CellKind, gates: GateBlock, C: np.ndarray, Xb: np.ndarray = None) -> np.ndarray:
    """Mix the resolved memory cells into outputs (GPU)."""
    if C.shape != gates.cand.shape:
        raise ValueError("memory-cell block shape does not match the gates")
    if kind is CellKind.SRU:
        if Xb is None:
            raise ValueError("SRU output needs the raw input block")
        if Xb.shape != C.shape:
            raise ValueError("input block shape does not match")
    elif kind is not CellKind.QRNN:
        raise ValueError(f"no blocked output path for {kind}")
    torch = _torch()
    dt = C.dtype if C.dtype in (np.float32, np.float64) else np.float64
    O, Cd = _dev(gates.out_gate, dt), _dev(C, dt)
    Xd = _dev(Xb, dt) if Xb is not None else None
    H = torch.empty_like(Cd)
    lib = _lib.load()
    _lib.check(lib.rnnb_finalize(_lib.SRU if kind is CellKind.SRU else _lib.QRNN,
                                 ctypes.c_void_p(O.data_ptr()), ctypes.c_void_p(Cd.data_ptr()),
                                 ctypes.c_void_p(Xd.data_ptr()) if Xd is not None else None,
                                 ctypes.c_void_p(H.data_ptr()), Cd.shape[0], Cd.shape[1],
                                 _lib.DT_F64 if dt == np.float64 else _lib.DT_F32, _stream_ptr(None)))
    return H.cpu().numpy()


# ---------------------------------------------------------------------------
# whole network


def run_blocked(cfg, weights, X: np.ndarray, block_size: int, kernel: str = "fast",
                trace: KernelTrace = None, stack_gates: bool = False, *, mode: str = None,
                return_state: bool = False):
    """Blocked execution of the whole network on the GPU; returns [L x d_h].

    Per layer ONE fused launch: block projection, c-scan and output mix for
    every block of ``block_size`` steps, c (and the QRNN x_carry) carried
    across blocks.  ``mode`` (extension) selects "bf16"/"tf32" tensor-core
    numerics; default follows X's dtype like the reference.  With
    ``return_state`` also returns the final c and x_carry of every layer.
    """
    if cfg.kind not in (CellKind.SRU, CellKind.QRNN):
        raise ValueError("blocked execution covers SRU and QRNN; use lstm_run_precomputed for LSTM")
    if not isinstance(X, np.ndarray) or X.ndim != 2 or X.shape[1] != cfg.d_in:
        raise ValueError(f"input must be [L x {cfg.d_in}], got {getattr(X, 'shape', None)}")
    plan = plan_blocks(X.shape[0], block_size)
    _check_kernel(kernel)
    fields = _sru_fields() if cfg.kind is CellKind.SRU else _qrnn_fields()
    for w in weights.layers:
        _check_layer_dtypes(w, fields, X.dtype)
    mode = mode or _mode_for(X.dtype)
    for w in weights.layers:
        for _, l in plan.blocks:
            _trace_block(trace, cfg.kind, w, l, stack_gates)
    st = DeviceStack(cfg.kind, weights.layers, mode=mode)
    try:
        c = np.zeros(sum(st.d_h), st.np_dtype)
        xc = np.zeros(sum(st.d_in), st.np_dtype)
        out = st.forward_host(np.ascontiguousarray(X, dtype=st.np_dtype), block_size,
                              c_state=c, x_carry=xc)
    finally:
        st.close()
    out = out.astype(X.dtype, copy=False)
    if not return_state:
        return out
    cs, xcs, co, xo = [], [], 0, 0
    for dh, din in zip(st.d_h, st.d_in):
        cs.append(c[co:co + dh].astype(X.dtype, copy=False))
        xcs.append(xc[xo:xo + din].astype(X.dtype, copy=False))
        co += dh
        xo += din
    return out, cs, xcs


def lstm_run_precomputed(w: LstmWeights, X: np.ndarray, block_size: int, kernel: str = "fast",
                         trace: KernelTrace = None) -> np.ndarray:
    """LSTM with the input-side products batched (blocked.py:271-305).

    Same signature, validation, trace events and result as the reference: per
    block the four W x products + biases (GEMM + BIAS events), per step the
    four U h products (GEMV events).  On the GPU the input-side products of
    the whole sequence are one GEMM launch (blocks only decide where the
    reference batches them, never their values) and the recurrence is one
    persistent launch with U resident in shared memory.
    """
    if X.ndim != 2 or X.shape[1] != w.d_in:
        raise ValueError(f"input must be [L x {w.d_in}], got {X.shape}")
    plan = plan_blocks(X.shape[0], block_size)
    _check_kernel(kernel)
    for f in LSTM_FIELDS:
        a = np.asarray(getattr(w, f))
        if a.dtype != X.dtype:
            raise ValueError(f"dtype mismatch: {a.dtype} vs {X.dtype}")
        if a.ndim == 2:
            _check_matrix(a, f)
    mode = _mode_for(X.dtype)
    if trace is not None:
        for _, length in plan.blocks:
            for wm, bv in ((w.w_forget, w.b_forget), (w.w_input, w.b_input), (w.w_output, w.b_output),
                           (w.w_cand, w.b_cand)):
                trace.add(PHASE_GEMM, wm.shape[0], wm.shape[1], length)
                trace.add(PHASE_BIAS, bv.shape[0], 1, length)
            for _ in range(length):
                for _ in range(4):
                    trace.add(PHASE_GEMV, w.d_h, w.d_h, 1)
    dev = DeviceLstm(w, mode=mode)
    try:
        out = dev.forward_host(np.ascontiguousarray(X), block_size)
    finally:
        dev.close()
    return out.astype(X.dtype, copy=False)
