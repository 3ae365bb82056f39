"""Drop-in types of the blocked SRU/QRNN path.

Same names, fields, validation and ``ValueError`` behaviour as the
reference package's types, so reference callers keep working:

* ``CellKind``                    -- rnnblock cells.py:27-37
* ``SruWeights`` / ``QrnnWeights`` -- cells.py:78-126 (canonical field order,
                                     model_io.py:29-33)
* ``CellState`` / ``zero_state``   -- cells.py:129-143
* ``RnnConfig`` / ``WeightSet``    -- model_io.py:75-110

* ``LstmWeights``                 -- cells.py:46-75 (for lstm_run_precomputed;
                                     the blocked entry point rejects LSTM the
                                     way the reference does, blocked.py:231-233)
"""

from dataclasses import dataclass, field
from enum import Enum

import numpy as np

PRECISIONS = {"f32": np.float32, "f64": np.float64}


class CellKind(Enum):
    LSTM = "lstm"
    SRU = "sru"
    QRNN = "qrnn"

    @classmethod
    def parse(cls, name: str) -> "CellKind":
        try:
            return cls(name.lower())
        except ValueError:
            raise ValueError(f"unknown cell kind {name!r}; expected lstm, sru, or qrnn") from None


def _expect(cond, msg):
    if not cond:
        raise ValueError(msg)


SRU_FIELDS = ("w_cand", "w_forget", "w_highway", "b_forget", "b_highway")
LSTM_FIELDS = ("w_forget", "w_input", "w_output", "w_cand", "u_forget", "u_input", "u_output", "u_cand",
               "b_forget", "b_input", "b_output", "b_cand")
QRNN_FIELDS = ("w_cand", "w_cand_prev", "w_forget", "w_forget_prev", "w_out", "w_out_prev")


@dataclass
class LstmWeights:
    """f, i, o = sigma(W x + U h + b); cand = tanh(W_c x + U_c h + b_c);
    c = f c + i cand; h = o tanh(c) (cells.py:153-164)."""

    w_forget: np.ndarray
    w_input: np.ndarray
    w_output: np.ndarray
    w_cand: np.ndarray
    u_forget: np.ndarray
    u_input: np.ndarray
    u_output: np.ndarray
    u_cand: np.ndarray
    b_forget: np.ndarray
    b_input: np.ndarray
    b_output: np.ndarray
    b_cand: np.ndarray

    def __post_init__(self):
        d_h, d_in = self.w_forget.shape
        for w in (self.w_input, self.w_output, self.w_cand):
            _expect(w.shape == (d_h, d_in), "input-side weight shapes disagree")
        for u in (self.u_forget, self.u_input, self.u_output, self.u_cand):
            _expect(u.shape == (d_h, d_h), "recurrent weights must be square d_h x d_h")
        for b in (self.b_forget, self.b_input, self.b_output, self.b_cand):
            _expect(b.shape == (d_h,), "bias length must equal d_h")

    @property
    def d_in(self):
        return self.w_forget.shape[1]

    @property
    def d_h(self):
        return self.w_forget.shape[0]

    def mats(self):
        return tuple(getattr(self, f) for f in LSTM_FIELDS)


@dataclass
class SruWeights:
    """x-hat = W x; f = sigma(W_f x + b_f); r = sigma(W_r x + b_r);
    c = f c + (1-f) x-hat; h = r tanh(c) + (1-r) x (cells.py:167-176)."""

    w_cand: np.ndarray
    w_forget: np.ndarray
    w_highway: np.ndarray
    b_forget: np.ndarray
    b_highway: np.ndarray

    def __post_init__(self):
        d_h, d_in = self.w_cand.shape
        _expect(d_in == d_h, "SRU requires d_in == d_h")
        _expect(self.w_forget.shape == (d_h, d_in), "weight shapes disagree")
        _expect(self.w_highway.shape == (d_h, d_in), "weight shapes disagree")
        _expect(self.b_forget.shape == (d_h,), "bias length must equal d_h")
        _expect(self.b_highway.shape == (d_h,), "bias length must equal d_h")

    @property
    def d_in(self):
        return self.w_cand.shape[1]

    @property
    def d_h(self):
        return self.w_cand.shape[0]

    def mats(self):
        return tuple(getattr(self, f) for f in SRU_FIELDS)


@dataclass
class QrnnWeights:
    """Two taps per gate, no biases (cells.py:104-126, 179-189)."""

    w_cand: np.ndarray
    w_cand_prev: np.ndarray
    w_forget: np.ndarray
    w_forget_prev: np.ndarray
    w_out: np.ndarray
    w_out_prev: np.ndarray

    def __post_init__(self):
        shape = self.w_cand.shape
        for w in (self.w_cand_prev, self.w_forget, self.w_forget_prev,
                  self.w_out, self.w_out_prev):
            _expect(w.shape == shape, "all six tap matrices must share one shape")

    @property
    def d_in(self):
        return self.w_cand.shape[1]

    @property
    def d_h(self):
        return self.w_cand.shape[0]

    def mats(self):
        return tuple(getattr(self, f) for f in QRNN_FIELDS)


@dataclass
class CellState:
    """Recurrent carriers (cells.py:129-135); x_prev is the QRNN t-1 tap."""

    c: np.ndarray
    h: np.ndarray
    x_prev: np.ndarray


def zero_state(d_in: int, d_h: int, dtype) -> CellState:
    return CellState(c=np.zeros(d_h, dtype), h=np.zeros(d_h, dtype),
                     x_prev=np.zeros(d_in, dtype))


@dataclass(frozen=True)
class RnnConfig:
    """model_io.py:75-99."""

    kind: CellKind
    d_in: int
    d_h: int
    n_layers: int = 1
    precision: str = "f32"

    def __post_init__(self):
        if self.d_in < 1 or self.d_h < 1:
            raise ValueError("d_in and d_h must be >= 1")
        if self.n_layers < 1:
            raise ValueError("n_layers must be >= 1")
        if self.precision not in PRECISIONS:
            raise ValueError(f"precision must be one of {sorted(PRECISIONS)}")
        if self.kind is CellKind.SRU and self.d_in != self.d_h:
            raise ValueError("SRU requires d_in == d_h")

    @property
    def dtype(self):
        return PRECISIONS[self.precision]

    def layer_dims(self, layer: int) -> tuple:
        return (self.d_in if layer == 0 else self.d_h, self.d_h)


@dataclass
class WeightSet:
    """model_io.py:102-110."""

    kind: CellKind
    precision: str
    layers: list = field(default_factory=list)

    @property
    def dtype(self):
        return PRECISIONS[self.precision]
