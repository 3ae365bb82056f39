"""Shared parity helpers for the GPU tests (test infrastructure).

Tolerances (BASELINE.json north_star):
* fp32 (FFMA and the fp32-accurate 3xTF32 tensor-core mode): normwise
  max|d| / max|ref| <= 1e-5 AND max|d| <= 1e-4 -- the reference's
  ORACLE_TOLERANCE (/root/reference/pkg/src/rnnblock/bench.py:25);
* TF32: <= 2e-3 normwise vs the fp32 oracle and <= 1e-5 vs the oracle run on
  tf32-rounded operands (per layer);
* BF16: <= 2e-2 normwise vs the fp32 oracle and <= 1e-3 vs the oracle run on
  bf16-rounded operands (per layer).
The "rounded operands" oracle rounds exactly what the tensor-core kernel
rounds: the weights and the layer input at the product; the SRU highway term
(1 - r) x uses the raw fp32 x (cells.py:115-131 reads x itself).
"""

import numpy as np

BOUND_VS_F32 = {"bf16": 2e-2, "tf32": 2e-3, "f32x3": 1e-5, "f32": 1e-5}
BOUND_VS_ROUNDED = {"bf16": 1e-3, "tf32": 1e-5}


def normwise(a, ref):
    ref = np.asarray(ref, np.float64)
    return float(np.max(np.abs(np.asarray(a, np.float64) - ref)) / max(np.max(np.abs(ref)), 1e-30))


def maxabs(a, ref):
    return float(np.max(np.abs(np.asarray(a, np.float64) - np.asarray(ref, np.float64))))


def assert_f32(a, ref, what=""):
    n, d = normwise(a, ref), maxabs(a, ref)
    assert n <= 1e-5 and d <= 1e-4, (what, n, d)
    return n


def round_tf32(a):
    """cvt.rna.tf32.f32 (round to nearest, ties away) kept in fp32."""
    u = np.ascontiguousarray(a, np.float32).view(np.uint32).astype(np.uint64)
    u = ((u + 0x1000) & 0xFFFFE000).astype(np.uint32)
    return u.view(np.float32)


def round_bf16(a):
    """__float2bfloat16_rn (round to nearest even) widened back to fp32."""
    u = np.ascontiguousarray(a, np.float32).view(np.uint32).astype(np.uint64)
    u = ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32)
    return u.view(np.float32)


ROUND = {"bf16": round_bf16, "tf32": round_tf32}


def _sig(z):
    return 0.5 * (1.0 + np.tanh(0.5 * z))


def rounded_layer(oracle, kind, mats, x, T, mode, c=None, xc=None):
    """One layer on the oracle with products on `mode`-rounded weights and
    input; for SRU the highway term is moved back onto the raw input:
    H = r tanh c + (1-r) xr  ->  + (1-r)(x - xr).  Returns (H, c_T)."""
    rnd = ROUND[mode]
    rl = [rnd(m) if np.ndim(m) == 2 else np.asarray(m, np.float32) for m in mats]
    xr = rnd(x)
    xcr = None if xc is None else rnd(xc)
    H, cT, _ = oracle.layer_blocked(kind, rl, xr, T, c=c, xc=xcr)
    if kind == "sru":
        z = xr @ rl[2].T  # sgemm: r is only needed to ~1e-7 against a 1e-3 bound
        r = _sig(z.astype(np.float64) + rl[4].astype(np.float64))
        H = (H + (1.0 - r) * (x.astype(np.float64) - xr.astype(np.float64))).astype(np.float32)
    return H, cT


def sru_wide_f64(mats, x_prod, x_hw, rows=None):
    """Wide SRU layer (d_in may exceed d_h; cfg5 layers 2-4) in float64, the
    cell of cells.py:115-131 applied per step: products on x_prod, highway
    (1 - r) * x_hw.  Used on a prefix of the sequence."""
    W, Wf, Wr, bf, br = mats
    x = np.asarray(x_prod, np.float64)
    n = x.shape[0] if rows is None else rows
    x = x[:n]
    xh = np.asarray(x_hw, np.float64)[:n]
    Z = x @ np.asarray(W, np.float64).T
    F = _sig(x @ np.asarray(Wf, np.float64).T + np.asarray(bf, np.float64))
    R = _sig(x @ np.asarray(Wr, np.float64).T + np.asarray(br, np.float64))
    c = np.zeros(W.shape[0])
    H = np.empty((n, W.shape[0]))
    for t in range(n):
        c = F[t] * c + (1.0 - F[t]) * Z[t]
        H[t] = R[t] * np.tanh(c) + (1.0 - R[t]) * xh[t]
    return H
