"""BASELINE cfg3: acoustic-model-shaped stacked SRU.

  frames [L x 120] -> linear projection [1024 x 120] -> 6 x SRU-1024
  (blocked, one fused kernel launch per layer) -> linear logits [2000 x 1024]

Every stage runs on this repository's kernels (librnnb.so): the SRU stack on
the blocked-path layer kernels (DeviceStack), the projection and the logits
on the dense-layer kernels (DeviceLinear: FFMA GEMM in f32, tcgen05 in
bf16 / tf32 with the recurrent layers' operand rounding).  The reference has
no dense layer type; the product they restate is kernels.gemm
(/root/reference/pkg/src/rnnblock/kernels.py:203-225).
"""

from .cells import CellKind
from .device import DeviceLinear, DeviceStack


class AcousticSRU:
    def __init__(self, proj, layers, logits, mode="f32", device=None):
        self.mode = mode
        self.stack = DeviceStack(CellKind.SRU, layers, mode=mode, device=device)
        self.proj = DeviceLinear(proj, mode=mode, device=self.stack.device)
        self.logits = DeviceLinear(logits, mode=mode, device=self.stack.device)

    def project(self, frames, stream=None):
        """frames [L x 120] -> [L x 1024] (the input projection)."""
        return self.proj.forward(frames, stream=stream)

    def classify(self, h, stream=None):
        """hidden [L x 1024] -> logits [L x 2000]."""
        return self.logits.forward(h, stream=stream)

    def forward(self, frames, block_size, stream=None):
        """frames [L x 120] (CUDA, fp32) -> logits [L x 2000] (fp32)."""
        h = self.stack.forward(self.project(frames, stream), block_size, stream=stream)
        return self.classify(h, stream)

    @property
    def last_launches(self):
        return self.proj.query(1) + self.stack.last_launches + self.logits.query(1)

    def close(self):
        self.stack.close()
        self.proj.close()
        self.logits.close()
