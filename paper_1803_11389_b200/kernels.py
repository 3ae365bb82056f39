"""Drop-in for the reference's dense kernels and activations
(rnnblock kernels.py:181-241, 312-326) on the GPU.

Same names, signatures, argument checks and ``ValueError`` messages as the
reference, so callers of ``rnnblock.kernels`` keep working; the arithmetic
runs in librnnb.so (csrc/unit_ops.cu), with no CPU fallback.  Kernel names
keep the reference's meaning:

* ``"reference"`` / ``"tiled"``: ascending inner index, separately rounded
  multiply and add -- bitwise the reference kernels' chain;
* ``"fast"``: fused multiply-add (the reference's fast family reassociates;
  both are tolerance-checked against ``"reference"``).

The blocked path never calls these: its gate products and activations are
fused inside the layer kernels (csrc/ffma_ws.cuh, csrc/tc_layer.cuh).
"""

import ctypes

import numpy as np

from . import _lib

PRECISIONS = {"f32": np.float32, "f64": np.float64}
KERNELS = ("reference", "tiled", "fast")
DEFAULT_TILE = (64, 64)

_threads = None


def _check_matrix(a, name="matrix"):
    if not isinstance(a, np.ndarray) or a.ndim != 2:
        raise ValueError(f"{name} must be a 2-d ndarray")
    if a.shape[0] < 1 or a.shape[1] < 1:
        raise ValueError(f"{name} must have at least one row and one column")
    if not a.flags.c_contiguous:
        raise ValueError(f"{name} must be C-contiguous (row-major)")


def _check_vector(v, name="vector"):
    if not isinstance(v, np.ndarray) or v.ndim != 1:
        raise ValueError(f"{name} must be a 1-d ndarray")
    if v.shape[0] < 1:
        raise ValueError(f"{name} must not be empty")


def _torch_dev():
    import torch
    if not torch.cuda.is_available():
        raise _lib.RnnbError("CUDA is not available: the kernels have no CPU fallback")
    return torch


def _dt(dtype):
    if dtype == np.float32:
        return _lib.DT_F32
    if dtype == np.float64:
        return _lib.DT_F64
    raise ValueError(f"unsupported dtype {dtype}; expected float32 or float64")


def _gemm_dev(A, B, strict):
    torch = _torch_dev()
    lib = _lib.load()
    dt = _dt(A.dtype)
    a = torch.from_numpy(A).cuda()
    b = torch.from_numpy(B).cuda()
    c = torch.empty((A.shape[0], B.shape[1]), dtype=a.dtype, device=a.device)
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    _lib.check(lib.rnnb_gemm(1 if strict else 0, ctypes.c_void_p(a.data_ptr()), a.stride(0),
                             ctypes.c_void_p(b.data_ptr()), b.stride(0), ctypes.c_void_p(c.data_ptr()), c.stride(0),
                             A.shape[0], B.shape[1], A.shape[1], dt, s))
    return c.cpu().numpy()


def gemv(A: np.ndarray, x: np.ndarray, kernel: str = "reference") -> np.ndarray:
    """out[i] = sum_j A[i,j] x[j]  (kernels.py:181-200)."""
    _check_matrix(A, "A")
    _check_vector(x, "x")
    if A.shape[1] != x.shape[0]:
        raise ValueError(f"dimension mismatch: A is {A.shape}, x has length {x.shape[0]}")
    if A.dtype != x.dtype:
        raise ValueError(f"dtype mismatch: {A.dtype} vs {x.dtype}")
    if kernel not in ("reference", "fast"):
        raise ValueError(f"unknown kernel {kernel!r}")
    return _gemm_dev(A, np.ascontiguousarray(x.reshape(-1, 1)), kernel == "reference").reshape(-1)


def gemm(A: np.ndarray, B: np.ndarray, kernel: str = "reference", tile: tuple = DEFAULT_TILE) -> np.ndarray:
    """C[i,j] = sum_p A[i,p] B[p,j]  (kernels.py:203-233)."""
    _check_matrix(A, "A")
    _check_matrix(B, "B")
    if A.shape[1] != B.shape[0]:
        raise ValueError(f"dimension mismatch: A is {A.shape}, B is {B.shape}")
    if A.dtype != B.dtype:
        raise ValueError(f"dtype mismatch: {A.dtype} vs {B.dtype}")
    if kernel == "tiled":
        ti, tj = tile
        if ti < 1 or tj < 1:
            raise ValueError("tile sides must be >= 1")
    elif kernel not in ("reference", "fast"):
        raise ValueError(f"unknown kernel {kernel!r}")
    return _gemm_dev(A, B, kernel != "fast")


def _act(which, x):
    arr = np.asarray(x)
    if arr.dtype not in (np.float32, np.float64):
        arr = arr.astype(np.float64)  # numpy promotes Python/int inputs to float64 too
    torch = _torch_dev()
    lib = _lib.load()
    t = torch.from_numpy(np.ascontiguousarray(arr).reshape(-1)).cuda()
    s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    _lib.check(lib.rnnb_activation(which, ctypes.c_void_p(t.data_ptr()), ctypes.c_void_p(t.data_ptr()), t.numel(),
                                   _dt(arr.dtype), s))
    out = t.cpu().numpy().reshape(arr.shape)
    return out if arr.ndim else out[()]


def sigmoid(x):
    """0.5 * (1 + tanh(x / 2)): overflow-free and exactly symmetric (kernels.py:236-237)."""
    return _act(0, x)


def tanh_act(x):
    """tanh, dtype-preserving (kernels.py:240-241)."""
    return _act(1, x)


def set_compute_threads(n: int) -> int:
    """kernels.py:312-322.  The GPU kernels use one thread per output
    element and results never depend on the count; the value is recorded
    for get_compute_threads, clamped to the multiprocessor count."""
    global _threads
    if n < 1:
        raise ValueError("thread count must be >= 1")
    limit = 148
    try:
        import torch
        if torch.cuda.is_available():
            limit = torch.cuda.get_device_properties(0).multi_processor_count
    except Exception:
        pass
    _threads = min(n, limit)
    return _threads


def get_compute_threads() -> int:
    if _threads is None:
        return set_compute_threads(1 << 30)
    return _threads


# ---------------------------------------------------------------------------
# the reference's PRNG utilities (kernels.py:253-309): host-side scalar
# helpers for callers that draw values one at a time; bulk streams are
# generated on the GPU (model_io.generate_weights / generate_sequence)

_MASK64 = (1 << 64) - 1


class Rng64:
    """SplitMix64 stream (kernels.py:253-269); from seed 0 the first output
    is 0xE220A8397B1DCDAF."""

    def __init__(self, seed: int):
        self.state = seed & _MASK64

    def next(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & _MASK64
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & _MASK64
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & _MASK64
        return z ^ (z >> 31)


def uniform_weight(raw: int) -> float:
    """Top 24 bits of a raw draw to [-0.1, 0.1): (u / 2^24) * 0.2 - 0.1 in
    float64, in this operation order (kernels.py:292-299)."""
    u = (int(raw) & _MASK64) >> 40
    return (u / 16777216.0) * 0.2 - 0.1

