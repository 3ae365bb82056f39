"""Seeded synthetic workloads with BASELINE.json's shapes and distributions.

There is no dataset on this path: the paper times synthetic 1,024-sample
runs and BASELINE.json describes every config by shape and
distribution only.  Each config is drawn from ONE seed with numpy's
PCG64 ``Generator`` in float64 and then cast, weights first in the
reference's canonical field order (model_io.py:29-33), then the input X
(SURVEY.md §8d):

* cfg1  SRU  D=H=512,  L=256;  W, W_f, W_r ~ U(+-1/sqrt(512)), b = 0; x ~ N(0,1)
* cfg2  QRNN D=H=1024, L=2048, w=2; six taps ~ U(+-1/sqrt(2048)); x ~ N(0,1)
* cfg3  120 -> 1024 projection ~ U(+-1/sqrt(120)), 6 SRU-1024 ~ U(+-1/sqrt(1024))
        b = 0, logits 1024 -> 2000 ~ U(+-1/sqrt(1024)); L=4096 frames ~ N(0,1)
* cfg4  8 QRNN H=D=2048, w=2 ~ U(+-1/sqrt(4096)); L=65536; x ~ N(0,1)
* cfg5  bidirectional SRU, 4 layers, H=4096/dir (D_in 4096, then 8192)
        ~ U(+-1/sqrt(4096)); L=8192; x ~ N(0,1)

``scale`` shrinks L (and nothing else) for quick tests.
"""

from dataclasses import dataclass, field

import numpy as np

from .cells import CellKind, QrnnWeights, SruWeights

SEEDS = {"cfg1": 1001, "cfg2": 1002, "cfg3": 1003, "cfg4": 1004, "cfg5": 1005}
BLOCK_SIZES = {
    "cfg1": (1, 4, 16),
    "cfg2": (1, 2, 4, 8, 16, 32, 64),
    "cfg3": (1, 8, 32),
    "cfg4": (32,),
    "cfg5": (16, 64),
}


@dataclass
class Workload:
    name: str
    kind: CellKind
    layers: list
    X: np.ndarray
    block_sizes: tuple
    proj: np.ndarray = None        # cfg3 input projection [H x F]
    logits: np.ndarray = None      # cfg3 output layer [V x H]
    bidirectional: bool = False    # cfg5
    layers_bwd: list = field(default_factory=list)

    @property
    def seq_len(self):
        return self.X.shape[0]


def _u(rng, shape, fan_in, dtype):
    b = 1.0 / np.sqrt(fan_in)
    return rng.uniform(-b, b, size=shape).astype(dtype)


def _normal(rng, rows, cols, dtype, chunk=4096):
    out = np.empty((rows, cols), dtype)
    for r in range(0, rows, chunk):
        n = min(chunk, rows - r)
        out[r:r + n] = rng.standard_normal((n, cols)).astype(dtype)
    return out


def _sru_layer(rng, d_in, d_h, fan_in, dtype):
    return SruWeights(
        w_cand=_u(rng, (d_h, d_in), fan_in, dtype),
        w_forget=_u(rng, (d_h, d_in), fan_in, dtype),
        w_highway=_u(rng, (d_h, d_in), fan_in, dtype),
        b_forget=np.zeros(d_h, dtype),
        b_highway=np.zeros(d_h, dtype),
    )


def _qrnn_layer(rng, d_in, d_h, fan_in, dtype):
    return QrnnWeights(*[_u(rng, (d_h, d_in), fan_in, dtype) for _ in range(6)])


def make(name: str, seed: int = None, dtype=np.float32, scale: float = 1.0) -> Workload:
    seed = SEEDS[name] if seed is None else seed
    rng = np.random.Generator(np.random.PCG64(seed))

    def L(n):
        return max(1, int(round(n * scale)))

    if name == "cfg1":
        layers = [_sru_layer(rng, 512, 512, 512, dtype)]
        X = _normal(rng, L(256), 512, dtype)
        return Workload(name, CellKind.SRU, layers, X, BLOCK_SIZES[name])
    if name == "cfg2":
        layers = [_qrnn_layer(rng, 1024, 1024, 2048, dtype)]
        X = _normal(rng, L(2048), 1024, dtype)
        return Workload(name, CellKind.QRNN, layers, X, BLOCK_SIZES[name])
    if name == "cfg3":
        proj = _u(rng, (1024, 120), 120, dtype)
        layers = [_sru_layer(rng, 1024, 1024, 1024, dtype) for _ in range(6)]
        logits = _u(rng, (2000, 1024), 1024, dtype)
        X = _normal(rng, L(4096), 120, dtype)
        return Workload(name, CellKind.SRU, layers, X, BLOCK_SIZES[name], proj=proj, logits=logits)
    if name == "cfg4":
        layers = [_qrnn_layer(rng, 2048, 2048, 4096, dtype) for _ in range(8)]
        X = _normal(rng, L(65536), 2048, dtype)
        return Workload(name, CellKind.QRNN, layers, X, BLOCK_SIZES[name])
    if name == "cfg5":
        fwd, bwd = [], []
        for li in range(4):
            d_in = 4096 if li == 0 else 8192
            fwd.append(_sru_layer_wide(rng, d_in, 4096, dtype))
            bwd.append(_sru_layer_wide(rng, d_in, 4096, dtype))
        X = _normal(rng, L(8192), 4096, dtype)
        return Workload(name, CellKind.SRU, fwd, X, BLOCK_SIZES[name], bidirectional=True,
                        layers_bwd=bwd)
    raise ValueError(f"unknown workload {name!r}; expected cfg1..cfg5")


@dataclass
class WideSruWeights:
    """cfg5 layers 2-4 have d_in = 8192 != H = 4096, which the reference's
    SruWeights rejects (cells.py:89).  Same fields, no squareness check; the
    highway term uses the direction-aligned half of the input."""

    w_cand: np.ndarray
    w_forget: np.ndarray
    w_highway: np.ndarray
    b_forget: np.ndarray
    b_highway: np.ndarray

    @property
    def d_in(self):
        return self.w_cand.shape[1]

    @property
    def d_h(self):
        return self.w_cand.shape[0]

    def mats(self):
        return (self.w_cand, self.w_forget, self.w_highway, self.b_forget, self.b_highway)


def _sru_layer_wide(rng, d_in, d_h, dtype):
    return WideSruWeights(
        w_cand=_u(rng, (d_h, d_in), 4096, dtype),
        w_forget=_u(rng, (d_h, d_in), 4096, dtype),
        w_highway=_u(rng, (d_h, d_in), 4096, dtype),
        b_forget=np.zeros(d_h, dtype),
        b_highway=np.zeros(d_h, dtype),
    )


def flops_per_step(w: Workload) -> float:
    """Dense-contraction FLOPs per time step."""
    total = 0.0
    lists = [w.layers] + ([w.layers_bwd] if w.bidirectional else [])
    for layers in lists:
        for lay in layers:
            taps = 2 if w.kind is CellKind.QRNN else 1
            total += 2.0 * 3 * lay.d_h * taps * lay.d_in
    if w.proj is not None:
        total += 2.0 * w.proj.size
    if w.logits is not None:
        total += 2.0 * w.logits.size
    return total


def param_count(w: Workload) -> int:
    n = 0
    lists = [w.layers] + ([w.layers_bwd] if w.bidirectional else [])
    for layers in lists:
        for lay in layers:
            n += sum(int(m.size) for m in lay.mats())
    if w.proj is not None:
        n += w.proj.size
    if w.logits is not None:
        n += w.logits.size
    return n
