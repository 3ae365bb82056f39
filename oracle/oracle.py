"""TEST INFRASTRUCTURE ONLY -- ctypes front end of the CPU oracle.

Only tests/, ``__graft_entry__.smoke()`` and bench.py (its ``cpu_baseline``
and ``--impl reference`` legs) may import this module, and only as the
checker or the CPU baseline; the product package never does.

The numerics live in ``oracle_strict.c`` / ``oracle_fast.c`` (a C
restatement of rnnblock's blocked.py / cells.py / kernels.py, cited there
line by line).  Build with ``make -C oracle`` (``__graft_entry__.build()``
does it).  Parity of this oracle with the reference itself is pinned by
tests/test_oracle_golden.py against fixtures the reference produced
(tests/golden/make_golden.py).
"""

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
def _host_isa():
    try:
        with open("/proc/cpuinfo") as f:
            flags = f.read()
        return "v4" if (" avx512f" in flags and " avx512vl" in flags and " avx512bw" in flags) else "v3"
    except OSError:
        return "v3"


ISA = os.environ.get("ORACLE_ISA", _host_isa())
LIB_PATH = os.path.join(_HERE, "_build", f"liboracle_{ISA}.so")

SRU, QRNN = 1, 2
KERNELS = {"reference": 0, "fast": 1}

# canonical field order per layer (rnnblock model_io.py:29-33)
SRU_FIELDS = ("w_cand", "w_forget", "w_highway", "b_forget", "b_highway")
QRNN_FIELDS = ("w_cand", "w_cand_prev", "w_forget", "w_forget_prev", "w_out", "w_out_prev")

_lib = None


def build():
    import subprocess
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        i64, vp, ci = ctypes.c_int64, ctypes.c_void_p, ctypes.c_int
        for sfx in ("f32", "f64"):
            f = getattr(L, f"orc_layer_blocked_{sfx}")
            f.argtypes = [ci, i64, i64, vp, vp, i64, i64, ci, vp, vp, vp]
            f.restype = ci
            f = getattr(L, f"orc_layer_stepwise_{sfx}")
            f.argtypes = [ci, i64, i64, vp, vp, i64, vp, vp, vp]
            f.restype = ci
            for g in ("gemm_ref", "gemm_fast"):
                f = getattr(L, f"orc_{g}_{sfx}")
                f.argtypes = [vp, vp, vp, i64, i64, i64]
                f.restype = None
            f = getattr(L, f"orc_gemv_ref_{sfx}")
            f.argtypes = [vp, vp, vp, i64, i64]
            f.restype = None
            f = getattr(L, f"orc_lstm_blocked_{sfx}")
            f.argtypes = [i64, i64, vp, vp, i64, i64, ci, vp, vp, vp]
            f.restype = ci
            f = getattr(L, f"orc_lstm_stepwise_{sfx}")
            f.argtypes = [i64, i64, vp, vp, i64, vp, vp, vp]
            f.restype = ci
        L.orc_sm64_fill.argtypes = [ctypes.c_uint64, vp, i64]
        L.orc_uniform.argtypes = [vp, vp, i64]
        L.orc_set_threads.argtypes = [ci]
        L.orc_get_threads.restype = ci
        _lib = L
    return _lib


def _sfx(dtype):
    dtype = np.dtype(dtype)
    if dtype == np.float32:
        return "f32"
    if dtype == np.float64:
        return "f64"
    raise ValueError(f"oracle supports float32/float64, got {dtype}")


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def kind_code(kind):
    name = getattr(kind, "value", kind)
    name = str(name).lower()
    if name in ("sru", "1"):
        return SRU
    if name in ("qrnn", "2"):
        return QRNN
    raise ValueError(f"oracle covers SRU and QRNN, got {kind!r}")


def layer_mats(kind, layer, dtype):
    """Canonical-order arrays of one layer (dataclass or sequence)."""
    fields = SRU_FIELDS if kind_code(kind) == SRU else QRNN_FIELDS
    if isinstance(layer, (list, tuple)):
        mats = list(layer)
    elif isinstance(layer, dict):
        mats = [layer[f] for f in fields]
    else:
        mats = [getattr(layer, f) for f in fields]
    return [np.ascontiguousarray(m, dtype=dtype) for m in mats]


def set_threads(n):
    lib().orc_set_threads(int(n))


def get_threads():
    return lib().orc_get_threads()


def _layer(fn, kind, layer, X, *extra, c=None, xc=None):
    dtype = X.dtype
    k = kind_code(kind)
    mats = layer_mats(kind, layer, dtype)
    dh, din = mats[0].shape
    X = np.ascontiguousarray(X)
    if X.ndim != 2 or X.shape[1] != din:
        raise ValueError(f"input must be [L x {din}], got {X.shape}")
    H = np.empty((X.shape[0], dh), dtype)
    arr = (ctypes.c_void_p * len(mats))(*[m.ctypes.data for m in mats])
    c_buf = None if c is None else np.ascontiguousarray(c, dtype=dtype).copy()
    x_buf = None if xc is None else np.ascontiguousarray(xc, dtype=dtype).copy()
    rc = fn(k, din, dh, arr, _ptr(X), X.shape[0], *extra, _ptr(H),
            None if c_buf is None else _ptr(c_buf), None if x_buf is None else _ptr(x_buf))
    if rc != 0:
        raise ValueError("oracle rejected the arguments")
    return H, c_buf, x_buf


def layer_blocked(kind, layer, X, block_size, kernel="fast", c=None, xc=None):
    """One layer, blocked (blocked.py:246-266); returns (H, c_T, x_carry)."""
    if block_size < 1:
        raise ValueError("block_size must be >= 1")
    fn = getattr(lib(), f"orc_layer_blocked_{_sfx(X.dtype)}")
    c = np.zeros(layer_mats(kind, layer, X.dtype)[0].shape[0], X.dtype) if c is None else c
    xc = np.zeros(X.shape[1], X.dtype) if xc is None else xc
    return _layer(fn, kind, layer, X, int(block_size), KERNELS[kernel], c=c, xc=xc)


def layer_stepwise(kind, layer, X, c=None, xc=None):
    fn = getattr(lib(), f"orc_layer_stepwise_{_sfx(X.dtype)}")
    c = np.zeros(layer_mats(kind, layer, X.dtype)[0].shape[0], X.dtype) if c is None else c
    xc = np.zeros(X.shape[1], X.dtype) if xc is None else xc
    return _layer(fn, kind, layer, X, c=c, xc=xc)


def run_blocked(kind, layers, X, block_size, kernel="fast", return_state=False):
    """Whole network, layer-major like blocked.py:237-267.  With
    return_state, also the per-layer final c and x_carry."""
    out = np.ascontiguousarray(X)
    cs, xcs = [], []
    for layer in layers:
        out, c, xc = layer_blocked(kind, layer, out, block_size, kernel)
        cs.append(c)
        xcs.append(xc)
    return (out, cs, xcs) if return_state else out


def run_stepwise(kind, layers, X, return_state=False):
    """cells.py:217-228 with the strict gemv."""
    out = np.ascontiguousarray(X)
    cs, xcs = [], []
    for layer in layers:
        out, c, xc = layer_stepwise(kind, layer, out)
        cs.append(c)
        xcs.append(xc)
    return (out, cs, xcs) if return_state else out


def gemm(A, B, kernel="reference"):
    """kernels.py:203-225 (B is [k x n])."""
    A = np.ascontiguousarray(A)
    B = np.ascontiguousarray(B, dtype=A.dtype)
    m, k = A.shape
    n = B.shape[1]
    C = np.empty((m, n), A.dtype)
    sfx = _sfx(A.dtype)
    if kernel == "fast":
        Bt = np.ascontiguousarray(B.T)
        getattr(lib(), f"orc_gemm_fast_{sfx}")(_ptr(A), _ptr(Bt), _ptr(C), m, k, n)
    else:
        getattr(lib(), f"orc_gemm_ref_{sfx}")(_ptr(A), _ptr(B), _ptr(C), m, k, n)
    return C


def gemv(A, x):
    A = np.ascontiguousarray(A)
    x = np.ascontiguousarray(x, dtype=A.dtype)
    y = np.empty(A.shape[0], A.dtype)
    getattr(lib(), f"orc_gemv_ref_{_sfx(A.dtype)}")(_ptr(A), _ptr(x), _ptr(y), A.shape[0], A.shape[1])
    return y


def raw_stream(seed, n):
    """SplitMix64 (kernels.py:253-289)."""
    out = np.empty(n, np.uint64)
    lib().orc_sm64_fill(ctypes.c_uint64(seed & ((1 << 64) - 1)), _ptr(out), n)
    return out


def uniform_array(raws):
    """kernels.py:302-305."""
    raws = np.ascontiguousarray(raws, dtype=np.uint64)
    out = np.empty(raws.shape[0], np.float64)
    lib().orc_uniform(_ptr(raws), _ptr(out), raws.shape[0])
    return out


def layer_spec(kind, d_in, d_h):
    """model_io.py:133-139."""
    if str(getattr(kind, "value", kind)).lower() == "lstm":
        return [(d_h, d_in)] * 4 + [(d_h, d_h)] * 4 + [(d_h,)] * 4
    if kind_code(kind) == SRU:
        return [(d_h, d_in)] * 3 + [(d_h,)] * 2
    return [(d_h, d_in)] * 6


def generate_layers(kind, d_in, d_h, n_layers, seed, dtype):
    """model_io.py:157-177 restated: one SplitMix64 stream, canonical order,
    float64 transform then cast; stacked layers read width d_h."""
    specs = []
    for li in range(n_layers):
        specs.append(layer_spec(kind, d_in if li == 0 else d_h, d_h))
    total = sum(int(np.prod(s)) for spec in specs for s in spec)
    values = uniform_array(raw_stream(seed, total))
    layers, pos = [], 0
    for spec in specs:
        mats = []
        for shape in spec:
            n = int(np.prod(shape))
            mats.append(values[pos:pos + n].astype(dtype).reshape(shape))
            pos += n
        layers.append(mats)
    return layers


def generate_sequence(seq_len, width, seed, dtype):
    """model_io.py:180-188."""
    return uniform_array(raw_stream(seed, seq_len * width)).astype(dtype).reshape(seq_len, width)


# ---------------------------------------------------------------------------
# LSTM

LSTM_FIELDS = ("w_forget", "w_input", "w_output", "w_cand", "u_forget", "u_input", "u_output", "u_cand",
               "b_forget", "b_input", "b_output", "b_cand")


def lstm_mats(w, dtype):
    if isinstance(w, (list, tuple)):
        mats = list(w)
    elif isinstance(w, dict):
        mats = [w[f] for f in LSTM_FIELDS]
    else:
        mats = [getattr(w, f) for f in LSTM_FIELDS]
    return [np.ascontiguousarray(m, dtype=dtype) for m in mats]


def _lstm(fn, w, X, *extra, c=None, h=None):
    X = np.ascontiguousarray(X)
    mats = lstm_mats(w, X.dtype)
    dh, din = mats[0].shape
    if X.ndim != 2 or X.shape[1] != din:
        raise ValueError(f"input must be [L x {din}], got {X.shape}")
    H = np.empty((X.shape[0], dh), X.dtype)
    arr = (ctypes.c_void_p * 12)(*[m.ctypes.data for m in mats])
    c_buf = np.zeros(dh, X.dtype) if c is None else np.ascontiguousarray(c, dtype=X.dtype).copy()
    h_buf = np.zeros(dh, X.dtype) if h is None else np.ascontiguousarray(h, dtype=X.dtype).copy()
    rc = fn(din, dh, arr, _ptr(X), X.shape[0], *extra, _ptr(H), _ptr(c_buf), _ptr(h_buf))
    if rc != 0:
        raise ValueError("oracle rejected the arguments")
    return H, c_buf, h_buf


def lstm_blocked(w, X, block_size, kernel="fast", c=None, h=None, return_state=False):
    """lstm_run_precomputed (blocked.py:271-305); returns H (and c_T, h_T)."""
    if block_size < 1:
        raise ValueError("block_size must be >= 1")
    fn = getattr(lib(), f"orc_lstm_blocked_{_sfx(X.dtype)}")
    H, c, h = _lstm(fn, w, X, int(block_size), KERNELS[kernel], c=c, h=h)
    return (H, c, h) if return_state else H


def lstm_stepwise(w, X, c=None, h=None, return_state=False):
    """lstm_step (cells.py:153-164) over the sequence, strict gemv."""
    fn = getattr(lib(), f"orc_lstm_stepwise_{_sfx(X.dtype)}")
    H, c, h = _lstm(fn, w, X, c=c, h=h)
    return (H, c, h) if return_state else H
