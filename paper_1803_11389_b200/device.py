"""Device-resident stack handle: weights uploaded once, forward on HBM tensors.

This is the explicit-handle form of the drop-in API (the
reference re-stacks weights on every ``run_blocked`` call and tests mutate
weights between calls, so a fast path must take an explicit handle rather
than cache by identity).  torch is only the allocator/stream plumbing here;
all compute goes through ``librnnb.so`` (include/rnnb.h).
"""

import ctypes

import numpy as np

from . import _lib
from .cells import CellKind, LSTM_FIELDS, QRNN_FIELDS, SRU_FIELDS


def _torch():
    import torch
    return torch


def kind_code(kind):
    if isinstance(kind, CellKind):
        if kind is CellKind.SRU:
            return _lib.SRU
        if kind is CellKind.QRNN:
            return _lib.QRNN
        raise ValueError("blocked execution covers SRU and QRNN; use lstm_run_precomputed for LSTM")
    return kind_code(CellKind.parse(str(kind)))


def canonical_mats(kind, layer):
    fields = SRU_FIELDS if kind_code(kind) == _lib.SRU else QRNN_FIELDS
    if isinstance(layer, (list, tuple)):
        return list(layer)
    if isinstance(layer, dict):
        return [layer[f] for f in fields]
    return [getattr(layer, f) for f in fields]


def _stream_ptr(stream):
    torch = _torch()
    if stream is None:
        stream = torch.cuda.current_stream()
    return ctypes.c_void_p(stream.cuda_stream)


class DeviceStack:
    """Layers of one cell kind resident on one GPU.

    mode: "f32" | "f64" (the reference precisions, FFMA/DFMA), "bf16"
    (bf16 weights, x rounded to bf16 at the product, fp32 accumulate) or
    "tf32" (weights and x rounded to tf32 at the product).
    """

    def __init__(self, kind, layers, mode="f32", device=None, wide=False, highway_offsets=None):
        torch = _torch()
        if not torch.cuda.is_available():
            raise _lib.RnnbError("CUDA is not available: the blocked path has no CPU fallback")
        self.lib = _lib.load()
        self.kind = kind_code(kind)
        if mode not in _lib.MODES:
            raise ValueError(f"mode must be one of {sorted(_lib.MODES)}")
        self.mode = mode
        self.device = torch.cuda.current_device() if device is None else int(device)
        mats = [canonical_mats(kind, lay) for lay in layers]
        if not mats:
            raise ValueError("a stack needs at least one layer")
        self.d_in = [int(np.shape(m[0])[1]) for m in mats]
        self.d_h = [int(np.shape(m[0])[0]) for m in mats]
        n = len(mats)
        din = (ctypes.c_int64 * n)(*self.d_in)
        dh = (ctypes.c_int64 * n)(*self.d_h)
        h = ctypes.c_void_p()
        flags = _lib.FLAG_WIDE_SRU if wide else 0
        _lib.check(self.lib.rnnb_stack_create_ex(ctypes.byref(h), self.kind, n, din, dh,
                                                 _lib.MODES[mode], self.device, flags))
        self._h = h
        for li, m in enumerate(mats):
            self.set_layer(li, m)
        for li, off in enumerate(highway_offsets or []):
            _lib.check(self.lib.rnnb_stack_set_highway(self._h, li, int(off)))

    @property
    def n_layers(self):
        return len(self.d_h)

    @property
    def dtype(self):
        torch = _torch()
        return torch.float64 if self.mode == "f64" else torch.float32

    @property
    def np_dtype(self):
        return np.float64 if self.mode == "f64" else np.float32

    def set_layer(self, li, mats):
        src = np.float64 if self.mode == "f64" else np.float32
        arrs = [np.ascontiguousarray(np.asarray(m), dtype=src) for m in mats]
        ptrs = (ctypes.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
        dt = _lib.DT_F64 if src is np.float64 else _lib.DT_F32
        _lib.check(self.lib.rnnb_stack_set_layer(self._h, li, ptrs, len(arrs), dt))

    def _check_dev(self, t, name):
        torch = _torch()
        if not isinstance(t, torch.Tensor) or not t.is_cuda:
            raise ValueError(f"{name} must be a CUDA tensor")
        if t.device.index != self.device:
            raise ValueError(f"{name} is on {t.device}, the stack on cuda:{self.device}")
        if t.dtype != self.dtype:
            raise ValueError(f"dtype mismatch: {t.dtype} vs {self.dtype}")
        if t.dim() != 2 or t.stride(1) != 1:
            raise ValueError(f"{name} must be a 2-d row-major tensor")

    def _check_state(self, t, n, name, host=False):
        """c_state / x_carry: exactly n elements of the stack's dtype, contiguous,
        on the stack's device (or host arrays for forward_host): the kernels
        read and write n elements through the pointer."""
        if t is None:
            return None
        if host:
            if not isinstance(t, np.ndarray) or t.dtype != self.np_dtype or t.size != n or not t.flags.c_contiguous:
                raise ValueError(f"{name} must be a contiguous {np.dtype(self.np_dtype).name} array of {n} elements")
            return t.ctypes.data_as(ctypes.c_void_p)
        torch = _torch()
        if not isinstance(t, torch.Tensor) or not t.is_cuda:
            raise ValueError(f"{name} must be a CUDA tensor")
        if t.dtype != self.dtype:
            raise ValueError(f"{name} dtype mismatch: {t.dtype} vs {self.dtype}")
        if t.numel() != n or not t.is_contiguous():
            raise ValueError(f"{name} must be a contiguous tensor of {n} elements, got {tuple(t.shape)}")
        if t.device.index != self.device:
            raise ValueError(f"{name} is on {t.device}, the stack on cuda:{self.device}")
        return ctypes.c_void_p(t.data_ptr())

    def forward(self, X, block_size, out=None, c_state=None, x_carry=None, stream=None):
        """run_blocked on device tensors; X [L x d_in] -> [L x d_h]."""
        torch = _torch()
        self._check_dev(X, "X")
        L = X.shape[0]
        if X.shape[1] != self.d_in[0]:
            raise ValueError(f"input must be [L x {self.d_in[0]}], got {tuple(X.shape)}")
        if out is None:
            out = torch.empty((L, self.d_h[-1]), dtype=self.dtype, device=X.device)
        self._check_dev(out, "out")
        if out.shape != (L, self.d_h[-1]):
            raise ValueError(f"out must be [{L} x {self.d_h[-1]}], got {tuple(out.shape)}")
        cp = self._check_state(c_state, sum(self.d_h), "c_state")
        xp = self._check_state(x_carry, sum(self.d_in), "x_carry")
        _lib.check(self.lib.rnnb_forward(self._h, ctypes.c_void_p(X.data_ptr()), X.stride(0), L,
                                         int(block_size), ctypes.c_void_p(out.data_ptr()),
                                         out.stride(0), cp, xp, _stream_ptr(stream)))
        return out

    def forward_ptr(self, x_ptr, ldx, L, block_size, h_ptr, ldh, peers=(), c_state=None, x_carry=None,
                    stream=None):
        """rnnb_forward_ex on raw device addresses (the multi-GPU partitions:
        X may be a slot of this rank's input ring, H and `peers` mapped peer
        buffers; ldh < 0 stores rows in reverse time order)."""
        peers = [int(p) for p in peers]
        arr = (ctypes.c_void_p * max(1, len(peers)))(*peers) if peers else None
        cp = self._check_state(c_state, sum(self.d_h), "c_state")
        xp = self._check_state(x_carry, sum(self.d_in), "x_carry")
        _lib.check(self.lib.rnnb_forward_ex(self._h, ctypes.c_void_p(int(x_ptr)), int(ldx), int(L), int(block_size),
                                            ctypes.c_void_p(int(h_ptr)), int(ldh), cp, xp, len(peers), arr,
                                            _stream_ptr(stream)))

    def forward_host(self, X, block_size, out=None, c_state=None, x_carry=None, stream=None):
        """End-to-end call on HOST arrays: H2D, forward, D2H inside the C call."""
        X = np.ascontiguousarray(X, dtype=self.np_dtype)
        if X.ndim != 2 or X.shape[1] != self.d_in[0]:
            raise ValueError(f"input must be [L x {self.d_in[0]}], got {X.shape}")
        if out is None:
            out = np.empty((X.shape[0], self.d_h[-1]), self.np_dtype)
        elif (not isinstance(out, np.ndarray) or out.dtype != self.np_dtype or not out.flags.c_contiguous
              or out.shape != (X.shape[0], self.d_h[-1])):
            raise ValueError(f"out must be a contiguous [{X.shape[0]} x {self.d_h[-1]}] array")
        cp = self._check_state(c_state, sum(self.d_h), "c_state", host=True)
        xp = self._check_state(x_carry, sum(self.d_in), "x_carry", host=True)
        _lib.check(self.lib.rnnb_forward_host(self._h, X.ctypes.data_as(ctypes.c_void_p), X.shape[0],
                                              int(block_size), out.ctypes.data_as(ctypes.c_void_p),
                                              cp, xp, _stream_ptr(stream)))
        return out

    def gates(self, layer, Xt, x_carry=None, stream=None):
        """Activated gates [3, d_h, l] for one time-major block Xt [l x d_in]."""
        torch = _torch()
        self._check_dev(Xt, "Xt")
        l = Xt.shape[0]
        G = torch.empty((3, self.d_h[layer], l), dtype=self.dtype, device=Xt.device)
        xp = ctypes.c_void_p(x_carry.data_ptr()) if x_carry is not None else None
        _lib.check(self.lib.rnnb_gates(self._h, layer, ctypes.c_void_p(Xt.data_ptr()), Xt.stride(0), l, xp,
                                       ctypes.c_void_p(G.data_ptr()), l, _stream_ptr(stream)))
        return G

    def query(self, what, layer=0):
        v = ctypes.c_int64()
        _lib.check(self.lib.rnnb_query(self._h, what, layer, ctypes.byref(v)))
        return v.value

    @property
    def weight_bytes(self):
        return self.query(0)

    @property
    def last_launches(self):
        return self.query(1)

    def close(self):
        if getattr(self, "_h", None):
            self.lib.rnnb_stack_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()


class DeviceLinear:
    """Dense layer Y = X W^T (+ b) resident on one GPU (include/rnnb.h
    rnnb_linear_*): the cfg3 acoustic model's input projection and logits,
    kernels.gemm(W, X^T) (kernels.py:203-225) in the time-major layout.
    mode: "f32" / "f64" / "f32x3" (FFMA GEMM) or "bf16" / "tf32" (tcgen05)."""

    def __init__(self, W, bias=None, mode="f32", device=None):
        torch = _torch()
        if not torch.cuda.is_available():
            raise _lib.RnnbError("CUDA is not available: the dense layers have no CPU fallback")
        self.lib = _lib.load()
        if mode not in _lib.MODES:
            raise ValueError(f"mode must be one of {sorted(_lib.MODES)}")
        self.mode = mode
        self.device = torch.cuda.current_device() if device is None else int(device)
        src = np.float64 if mode == "f64" else np.float32
        W = np.ascontiguousarray(np.asarray(W), dtype=src)
        if W.ndim != 2:
            raise ValueError("W must be a 2-d [d_out x d_in] array")
        self.d_out, self.d_in = (int(v) for v in W.shape)
        h = ctypes.c_void_p()
        _lib.check(self.lib.rnnb_linear_create(ctypes.byref(h), self.d_in, self.d_out, _lib.MODES[mode],
                                               self.device))
        self._h = h
        b = None if bias is None else np.ascontiguousarray(np.asarray(bias), dtype=src)
        if b is not None and b.shape != (self.d_out,):
            raise ValueError(f"bias must have shape ({self.d_out},)")
        dt = _lib.DT_F64 if src is np.float64 else _lib.DT_F32
        _lib.check(self.lib.rnnb_linear_set_weights(self._h, W.ctypes.data_as(ctypes.c_void_p),
                                                    None if b is None else b.ctypes.data_as(ctypes.c_void_p), dt))

    @property
    def dtype(self):
        torch = _torch()
        return torch.float64 if self.mode == "f64" else torch.float32

    def forward(self, X, out=None, stream=None):
        """X [L x d_in] CUDA tensor -> [L x d_out]."""
        torch = _torch()
        if not isinstance(X, torch.Tensor) or not X.is_cuda or X.dim() != 2 or X.stride(1) != 1:
            raise ValueError("X must be a 2-d row-major CUDA tensor")
        if X.dtype != self.dtype:
            raise ValueError(f"dtype mismatch: {X.dtype} vs {self.dtype}")
        if X.device.index != self.device:
            raise ValueError(f"X is on {X.device}, the layer on cuda:{self.device}")
        if X.shape[1] != self.d_in:
            raise ValueError(f"input must be [L x {self.d_in}], got {tuple(X.shape)}")
        L = X.shape[0]
        if out is None:
            out = torch.empty((L, self.d_out), dtype=self.dtype, device=X.device)
        _lib.check(self.lib.rnnb_linear_forward(self._h, ctypes.c_void_p(X.data_ptr()), X.stride(0), L,
                                                ctypes.c_void_p(out.data_ptr()), out.stride(0), _stream_ptr(stream)))
        return out

    def query(self, what):
        v = ctypes.c_int64()
        _lib.check(self.lib.rnnb_linear_query(self._h, what, ctypes.byref(v)))
        return v.value

    def close(self):
        if getattr(self, "_h", None):
            self.lib.rnnb_linear_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class DeviceLstm:
    """One LSTM layer resident on one GPU (lstm_run_precomputed,
    blocked.py:271-305): the input-side products for the sequence in one
    GEMM launch, the recurrence in one persistent cooperative launch with
    each CTA's rows of U in shared memory.  mode: "f32" | "f64"."""

    def __init__(self, w, mode="f32", device=None):
        torch = _torch()
        if not torch.cuda.is_available():
            raise _lib.RnnbError("CUDA is not available: the LSTM path has no CPU fallback")
        self.lib = _lib.load()
        if mode not in ("f32", "f64"):
            raise ValueError("LSTM modes are f32 and f64 (the reference precisions)")
        self.mode = mode
        self.device = torch.cuda.current_device() if device is None else int(device)
        mats = list(w) if isinstance(w, (list, tuple)) else [getattr(w, f) for f in LSTM_FIELDS]
        self.d_h, self.d_in = (int(v) for v in np.shape(mats[0]))
        h = ctypes.c_void_p()
        _lib.check(self.lib.rnnb_lstm_create(ctypes.byref(h), self.d_in, self.d_h, _lib.MODES[mode], self.device))
        self._h = h
        self.set_weights(mats)

    @property
    def dtype(self):
        torch = _torch()
        return torch.float64 if self.mode == "f64" else torch.float32

    @property
    def np_dtype(self):
        return np.float64 if self.mode == "f64" else np.float32

    def set_weights(self, mats):
        src = self.np_dtype
        arrs = [np.ascontiguousarray(np.asarray(m), dtype=src) for m in mats]
        ptrs = (ctypes.c_void_p * len(arrs))(*[a.ctypes.data for a in arrs])
        dt = _lib.DT_F64 if src is np.float64 else _lib.DT_F32
        _lib.check(self.lib.rnnb_lstm_set_weights(self._h, ptrs, len(arrs), dt))

    def forward(self, X, block_size, out=None, c_state=None, h_state=None, stream=None):
        """X [L x d_in] CUDA tensor -> [L x d_h]; c_state / h_state optional
        [d_h] CUDA tensors, in/out."""
        torch = _torch()
        if not isinstance(X, torch.Tensor) or not X.is_cuda or X.dim() != 2 or X.stride(1) != 1:
            raise ValueError("X must be a 2-d row-major CUDA tensor")
        if X.dtype != self.dtype:
            raise ValueError(f"dtype mismatch: {X.dtype} vs {self.dtype}")
        if X.shape[1] != self.d_in:
            raise ValueError(f"input must be [L x {self.d_in}], got {tuple(X.shape)}")
        L = X.shape[0]
        if X.device.index != self.device:
            raise ValueError(f"X is on {X.device}, the layer on cuda:{self.device}")
        if out is None:
            out = torch.empty((L, self.d_h), dtype=self.dtype, device=X.device)
        for t, name in ((out, "out"), (c_state, "c_state"), (h_state, "h_state")):
            if t is None:
                continue
            if not isinstance(t, torch.Tensor) or not t.is_cuda or t.dtype != self.dtype or t.device.index != self.device:
                raise ValueError(f"{name} must be a {self.dtype} tensor on cuda:{self.device}")
        if out.shape != (L, self.d_h) or out.stride(1) != 1:
            raise ValueError(f"out must be a row-major [{L} x {self.d_h}] tensor")
        for t, name in ((c_state, "c_state"), (h_state, "h_state")):
            if t is not None and (t.numel() != self.d_h or not t.is_contiguous()):
                raise ValueError(f"{name} must be a contiguous tensor of {self.d_h} elements")
        cp = ctypes.c_void_p(c_state.data_ptr()) if c_state is not None else None
        hp = ctypes.c_void_p(h_state.data_ptr()) if h_state is not None else None
        _lib.check(self.lib.rnnb_lstm_forward(self._h, ctypes.c_void_p(X.data_ptr()), X.stride(0), L,
                                              int(block_size), ctypes.c_void_p(out.data_ptr()), out.stride(0),
                                              cp, hp, _stream_ptr(stream)))
        return out

    def forward_host(self, X, block_size, out=None, c_state=None, h_state=None, stream=None):
        X = np.ascontiguousarray(X, dtype=self.np_dtype)
        if X.ndim != 2 or X.shape[1] != self.d_in:
            raise ValueError(f"input must be [L x {self.d_in}], got {X.shape}")
        if out is None:
            out = np.empty((X.shape[0], self.d_h), self.np_dtype)
        for t, name in ((c_state, "c_state"), (h_state, "h_state")):
            if t is not None and (not isinstance(t, np.ndarray) or t.dtype != self.np_dtype or t.size != self.d_h
                                  or not t.flags.c_contiguous):
                raise ValueError(f"{name} must be a contiguous {np.dtype(self.np_dtype).name} array of {self.d_h}")
        cp = c_state.ctypes.data_as(ctypes.c_void_p) if c_state is not None else None
        hp = h_state.ctypes.data_as(ctypes.c_void_p) if h_state is not None else None
        _lib.check(self.lib.rnnb_lstm_forward_host(self._h, X.ctypes.data_as(ctypes.c_void_p), X.shape[0],
                                                   int(block_size), out.ctypes.data_as(ctypes.c_void_p),
                                                   cp, hp, _stream_ptr(stream)))
        return out

    def query(self, what):
        v = ctypes.c_int64()
        _lib.check(self.lib.rnnb_lstm_query(self._h, what, ctypes.byref(v)))
        return v.value

    def close(self):
        if getattr(self, "_h", None):
            self.lib.rnnb_lstm_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
