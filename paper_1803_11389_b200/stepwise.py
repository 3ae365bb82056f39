"""Drop-in for the reference's step-at-a-time executors (rnnblock
cells.py:146-229): ``sru_step``, ``qrnn_step``, ``lstm_step``, ``step``,
``run_layer_stepwise``, ``run_stepwise``.

In the reference these are the correctness oracle the blocked path is
checked against (bench.py:88-103); here they run on the GPU like
everything else (no CPU fallback), for callers that use them directly:

* one step = one launch of the layer kernel over a single time step with
  the carried state in/out (c; the QRNN x_{t-1} tap; LSTM h);
* ``run_layer_stepwise`` / ``run_stepwise`` = the blocked kernels at
  T_b = 1, i.e. every weight applied to one step at a time, which is the
  stepwise recurrence (each step's gates, then c, then h).

Same validation and ``ValueError`` messages as the reference.  The test
suite's CPU oracle (oracle/) is the checker of these functions, never their
implementation.
"""

import numpy as np

from .cells import CellKind, CellState, zero_state


def _check_step_args(w, x_t, state):
    # cells.py:146-150
    if x_t.shape != (w.d_in,):
        raise ValueError(f"input length {x_t.shape} does not match d_in={w.d_in}")
    if state.c.shape != (w.d_h,) or state.h.shape != (w.d_h,):
        raise ValueError("state width does not match d_h")


def _mode(dtype):
    if dtype == np.float32:
        return "f32"
    if dtype == np.float64:
        return "f64"
    raise ValueError(f"unsupported dtype {dtype}; expected float32 or float64")


def _blocked_step(kind, w, x_t, state):
    from .device import DeviceStack
    dt = x_t.dtype
    st = DeviceStack(kind, [w], mode=_mode(dt))
    try:
        c = np.array(state.c, dtype=dt, copy=True)
        xp = np.array(state.x_prev, dtype=dt, copy=True) if kind is CellKind.QRNN else None
        h = st.forward_host(x_t.reshape(1, -1), 1, c_state=c, x_carry=xp)[0]
    finally:
        st.close()
    return CellState(c=c, h=h, x_prev=x_t)


def sru_step(w, x_t: np.ndarray, state: CellState, kernel: str = "reference") -> CellState:
    """One SRU step (cells.py:167-176)."""
    _check_step_args(w, x_t, state)
    return _blocked_step(CellKind.SRU, w, x_t, state)


def qrnn_step(w, x_t: np.ndarray, state: CellState, kernel: str = "reference") -> CellState:
    """One QRNN step; x_{-1} is state.x_prev (cells.py:179-189)."""
    _check_step_args(w, x_t, state)
    return _blocked_step(CellKind.QRNN, w, x_t, state)


def lstm_step(w, x_t: np.ndarray, state: CellState, kernel: str = "reference") -> CellState:
    """One LSTM step, gates on h_{t-1} (cells.py:153-164)."""
    from .device import DeviceLstm
    _check_step_args(w, x_t, state)
    dt = x_t.dtype
    dl = DeviceLstm(w, mode=_mode(dt))
    try:
        c = np.array(state.c, dtype=dt, copy=True)
        hs = np.array(state.h, dtype=dt, copy=True)
        h = dl.forward_host(x_t.reshape(1, -1), 1, c_state=c, h_state=hs)[0]
    finally:
        dl.close()
    return CellState(c=c, h=h, x_prev=x_t)


_STEP_FN = {CellKind.LSTM: lstm_step, CellKind.SRU: sru_step, CellKind.QRNN: qrnn_step}


def step(kind: CellKind, w, x_t, state, kernel: str = "reference") -> CellState:
    return _STEP_FN[kind](w, x_t, state, kernel)


def run_layer_stepwise(kind: CellKind, w, X: np.ndarray, kernel: str = "reference") -> np.ndarray:
    """One layer over X from the zero state (cells.py:203-214)."""
    if X.ndim != 2 or X.shape[1] != w.d_in:
        raise ValueError(f"input must be [L x {w.d_in}], got {X.shape}")
    if kind is CellKind.LSTM:
        from .device import DeviceLstm
        dl = DeviceLstm(w, mode=_mode(X.dtype))
        try:
            return dl.forward_host(np.ascontiguousarray(X), 1)
        finally:
            dl.close()
    from .device import DeviceStack
    st = DeviceStack(kind, [w], mode=_mode(X.dtype))
    try:
        return st.forward_host(np.ascontiguousarray(X), 1)
    finally:
        st.close()


def run_stepwise(cfg, weights, X: np.ndarray, kernel: str = "reference") -> np.ndarray:
    """The whole (possibly stacked) network one step at a time (cells.py:217-229)."""
    if X.shape[1] != cfg.d_in:
        raise ValueError(f"input width {X.shape[1]} does not match config d_in={cfg.d_in}")
    out = X
    for layer in weights.layers:
        out = run_layer_stepwise(cfg.kind, layer, np.ascontiguousarray(out), kernel)
    return out


__all__ = ["sru_step", "qrnn_step", "lstm_step", "step", "run_layer_stepwise", "run_stepwise", "zero_state"]
