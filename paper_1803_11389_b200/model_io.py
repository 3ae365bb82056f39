"""RNNW / RNNX files behind the reference's
interface (rnnblock model_io.py: save/load_weights, save/load_sequence, the
same exception classes), plus loaders that go from a file straight into the
device layouts through the C ABI (``rnnb_stack_load_rnnw``,
``rnnb_lstm_load_rnnw``, ``rnnb_rnnx_load``).

Saves are byte-identical to the reference's files; every load -- host or
device -- goes through the one native parser (csrc/rnnw_io.cu), which checks
sizes against the file before any allocation and reports the reference's
exception class (mapped back in _lib.check).
"""

import ctypes
import dataclasses
import os
import struct

import numpy as np

from . import _lib
from .cells import PRECISIONS, CellKind, LstmWeights, QrnnWeights, RnnConfig, SruWeights, WeightSet

_WEIGHT_MAGIC = b"RNNW"
_SEQ_MAGIC = b"RNNX"
_VERSION = 1
_KIND_CODES = {CellKind.LSTM: 0, CellKind.SRU: 1, CellKind.QRNN: 2}
_KIND_FROM = {v: k for k, v in _KIND_CODES.items()}
_PREC_CODES = {"f32": 0, "f64": 1}
_PREC_FROM = {v: k for k, v in _PREC_CODES.items()}
_LAYER_CLASS = {CellKind.LSTM: LstmWeights, CellKind.SRU: SruWeights, CellKind.QRNN: QrnnWeights}


class FileFormatError(ValueError):
    """Base class of serialisation errors (model_io.py:55)."""


class BadMagicError(FileFormatError):
    pass


class UnsupportedVersionError(FileFormatError):
    pass


class TruncatedFileError(FileFormatError):
    pass


class ShapeConsistencyError(FileFormatError):
    pass


def layer_spec(kind, d_in, d_h):
    """Canonical shapes of one layer (model_io.py:133-139)."""
    if kind is CellKind.LSTM:
        return [(d_h, d_in)] * 4 + [(d_h, d_h)] * 4 + [(d_h,)] * 4
    if kind is CellKind.SRU:
        return [(d_h, d_in)] * 3 + [(d_h,)] * 2
    return [(d_h, d_in)] * 6


def _dt(precision):
    return np.dtype("<f4") if precision == "f32" else np.dtype("<f8")


# File layouts (model_io.py:1-33): fixed little-endian headers, then
# row-major payloads in canonical field order.
_RNNW_HEADER = struct.Struct("<4sIBBHI")   # magic, version, kind, precision, reserved, n_layers
_RNNW_LAYER = struct.Struct("<II")         # d_in, d_h
_RNNX_HEADER = struct.Struct("<4sIBBHII")  # magic, version, precision, 2 reserved, seq_len, width


def _write(path, chunks):
    with open(path, "wb") as f:
        for c in chunks:
            f.write(c)


def save_weights(ws: WeightSet, path) -> None:
    dt = _dt(ws.precision)

    def chunks():
        yield _RNNW_HEADER.pack(_WEIGHT_MAGIC, _VERSION, _KIND_CODES[ws.kind], _PREC_CODES[ws.precision], 0,
                                len(ws.layers))
        for layer in ws.layers:
            yield _RNNW_LAYER.pack(layer.d_in, layer.d_h)
            for fld in dataclasses.fields(layer):
                yield np.ascontiguousarray(getattr(layer, fld.name), dtype=dt).tobytes()
    _write(path, chunks())


def save_sequence(X: np.ndarray, path) -> None:
    if X.ndim != 2:
        raise ValueError("sequence must be a 2-d array")
    if X.dtype not in (np.float32, np.float64):
        raise ValueError(f"unsupported dtype {X.dtype}")
    precision = "f32" if X.dtype == np.float32 else "f64"
    _write(path, (_RNNX_HEADER.pack(_SEQ_MAGIC, _VERSION, _PREC_CODES[precision], 0, 0, *X.shape),
                  np.ascontiguousarray(X, dtype=_dt(precision)).tobytes()))


def load_weights(path) -> WeightSet:
    """Parsed and validated by the native reader (csrc/rnnw_io.cu: sizes are
    checked against the file before anything is allocated; failures raise
    the reference's exception classes), then split into the layer
    dataclasses."""
    kind, precision, dims = weights_info(path)
    specs = [layer_spec(kind, d_in, d_h) for d_in, d_h in dims]
    flat = np.empty(sum(int(np.prod(s)) for spec in specs for s in spec), dtype=PRECISIONS[precision])
    _lib.check(_lib.load().rnnb_rnnw_read(_path(path), flat.ctypes.data_as(ctypes.c_void_p), flat.size,
                                          _lib.DT_F64 if precision == "f64" else _lib.DT_F32))
    layers, pos = [], 0
    for spec in specs:
        arrays = []
        for shape in spec:
            n = int(np.prod(shape))
            arrays.append(flat[pos:pos + n].reshape(shape).copy())
            pos += n
        layers.append(_LAYER_CLASS[kind](*arrays))
    return WeightSet(kind=kind, precision=precision, layers=layers)


def load_sequence(path) -> np.ndarray:
    """Native reader (rnnb_rnnx_load into host memory)."""
    precision, seq_len, width = sequence_info(path)
    out = np.empty((seq_len, width), dtype=PRECISIONS[precision])
    _lib.check(_lib.load().rnnb_rnnx_load(_path(path), out.ctypes.data_as(ctypes.c_void_p),
                                          _lib.DT_F64 if precision == "f64" else _lib.DT_F32, 0, None))
    return out


# ---------------------------------------------------------------------------
# native: file -> device


def _path(p):
    return os.fsencode(os.fspath(p))


def weights_info(path):
    """(kind, precision, [(d_in, d_h), ...]) of an RNNW file, validated natively."""
    lib = _lib.load()
    k, p, n = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
    _lib.check(lib.rnnb_rnnw_info(_path(path), ctypes.byref(k), ctypes.byref(p), ctypes.byref(n), None, None, 0))
    din = (ctypes.c_int64 * n.value)()
    dh = (ctypes.c_int64 * n.value)()
    _lib.check(lib.rnnb_rnnw_info(_path(path), ctypes.byref(k), ctypes.byref(p), ctypes.byref(n), din, dh, n.value))
    return _KIND_FROM[k.value], _PREC_FROM[p.value], list(zip(list(din), list(dh)))


def sequence_info(path):
    lib = _lib.load()
    p, L, W = ctypes.c_int(), ctypes.c_int64(), ctypes.c_int64()
    _lib.check(lib.rnnb_rnnx_info(_path(path), ctypes.byref(p), ctypes.byref(L), ctypes.byref(W)))
    return _PREC_FROM[p.value], L.value, W.value


def load_weights_device(path, mode=None, device=None, layer=0):
    """An RNNW file straight into a device handle: ``DeviceStack`` for
    SRU/QRNN, ``DeviceLstm`` (layer ``layer``) for LSTM.  mode defaults to
    the file's precision."""
    import torch

    from .device import DeviceLstm, DeviceStack
    kind, precision, dims = weights_info(path)
    mode = mode or precision
    dev = torch.cuda.current_device() if device is None else int(device)
    lib = _lib.load()
    h = ctypes.c_void_p()
    if kind is CellKind.LSTM:
        _lib.check(lib.rnnb_lstm_load_rnnw(ctypes.byref(h), _path(path), int(layer), _lib.MODES[mode], dev))
        obj = DeviceLstm.__new__(DeviceLstm)
        obj.lib, obj.mode, obj.device, obj._h = lib, mode, dev, h
        obj.d_in, obj.d_h = dims[layer]
        return obj
    _lib.check(lib.rnnb_stack_load_rnnw(ctypes.byref(h), _path(path), _lib.MODES[mode], dev))
    obj = DeviceStack.__new__(DeviceStack)
    obj.lib, obj.kind, obj.mode, obj.device, obj._h = lib, _KIND_CODES[kind], mode, dev, h
    obj.d_in = [d[0] for d in dims]
    obj.d_h = [d[1] for d in dims]
    return obj


def load_sequence_device(path, dtype=None, device=None, stream=None):
    """An RNNX payload into a new CUDA tensor (pinned staging, async H2D)."""
    import torch

    from .device import _stream_ptr
    precision, L, W = sequence_info(path)
    dtype = dtype or (torch.float64 if precision == "f64" else torch.float32)
    out = torch.empty((L, W), dtype=dtype, device=device if device is not None else "cuda")
    dt = _lib.DT_F64 if dtype == torch.float64 else _lib.DT_F32
    _lib.check(_lib.load().rnnb_rnnx_load(_path(path), ctypes.c_void_p(out.data_ptr()), dt, 1, _stream_ptr(stream)))
    return out


def config_of(ws: WeightSet) -> RnnConfig:
    first = ws.layers[0]
    return RnnConfig(ws.kind, first.d_in, first.d_h, n_layers=len(ws.layers), precision=ws.precision)


# ---------------------------------------------------------------------------
# deterministic generation (model_io.py:147-188) on the device


def count_params(cfg: RnnConfig) -> int:
    """model_io.py:147-152."""
    total = 0
    for layer in range(cfg.n_layers):
        d_in, d_h = cfg.layer_dims(layer)
        total += sum(int(np.prod(s)) for s in layer_spec(cfg.kind, d_in, d_h))
    return total


def _splitmix_uniform(seed, n, dtype):
    """Elements 0..n-1 of SplitMix64(seed) through the weight transform, cast
    to dtype -- generated on the GPU (rnnb_splitmix_uniform), copied back."""
    import torch
    if not torch.cuda.is_available():
        raise _lib.RnnbError("CUDA is not available: generation runs on the GPU (no CPU fallback)")
    lib = _lib.load()
    tdt = torch.float32 if np.dtype(dtype) == np.float32 else torch.float64
    out = torch.empty(max(int(n), 1), dtype=tdt, device="cuda")
    _lib.check(lib.rnnb_splitmix_uniform(ctypes.c_uint64(int(seed) & 0xFFFFFFFFFFFFFFFF), ctypes.c_uint64(0),
                                         int(n), ctypes.c_void_p(out.data_ptr()),
                                         _lib.DT_F32 if tdt == torch.float32 else _lib.DT_F64,
                                         ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)))
    return out[:n].cpu().numpy()


def generate_weights(cfg: RnnConfig, seed: int) -> WeightSet:
    """Every parameter from one SplitMix64 stream in canonical order, the
    transform in float64 then cast (model_io.py:155-177): byte-identical to
    the reference's weights for the same (cfg, seed)."""
    values = _splitmix_uniform(seed, count_params(cfg), cfg.dtype)
    layers, pos = [], 0
    for layer in range(cfg.n_layers):
        d_in, d_h = cfg.layer_dims(layer)
        arrays = []
        for shape in layer_spec(cfg.kind, d_in, d_h):
            n = int(np.prod(shape))
            arrays.append(np.ascontiguousarray(values[pos:pos + n].reshape(shape)))
            pos += n
        layers.append(_LAYER_CLASS[cfg.kind](*arrays))
    return WeightSet(kind=cfg.kind, precision=cfg.precision, layers=layers)


def generate_sequence(seq_len: int, width: int, seed: int, precision: str = "f32") -> np.ndarray:
    """Input matrix [seq_len x width] from SplitMix64(seed) (model_io.py:180-188)."""
    if seq_len < 1 or width < 1:
        raise ValueError("seq_len and width must be >= 1")
    if precision not in PRECISIONS:
        raise ValueError(f"precision must be one of {sorted(PRECISIONS)}")
    return _splitmix_uniform(seed, seq_len * width, PRECISIONS[precision]).reshape(seq_len, width)


PRESETS = {
    "lstm-small": (CellKind.LSTM, 350),
    "lstm-large": (CellKind.LSTM, 700),
    "sru-small": (CellKind.SRU, 512),
    "sru-large": (CellKind.SRU, 1024),
    "qrnn-small": (CellKind.QRNN, 512),
    "qrnn-large": (CellKind.QRNN, 1024),
}


def preset_config(name: str, precision: str = "f32", n_layers: int = 1) -> RnnConfig:
    """The paper's model sizes (model_io.py:116-130)."""
    if name not in PRESETS:
        raise ValueError(f"unknown preset {name!r}; expected one of {sorted(PRESETS)}")
    kind, width = PRESETS[name]
    return RnnConfig(kind=kind, d_in=width, d_h=width, n_layers=n_layers, precision=precision)
