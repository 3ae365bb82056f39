"""BASELINE cfg3: acoustic-model-shaped stacked SRU.

  frames [L x 120] -> linear projection [1024 x 120] -> 6 x SRU-1024
  (blocked, one fused kernel launch per layer) -> linear logits [2000 x 1024]

The SRU stack runs on the blocked-path kernels (DeviceStack).  The input
projection and the logits are plain dense products outside the recurrent
path (the reference has no such layers; SURVEY.md §8c checks them with its
gemm), so they use the library GEMM (cuBLAS through torch.matmul) with TF32
disabled in the fp32 mode.
"""

import torch

from .cells import CellKind
from .device import DeviceStack


class AcousticSRU:
    def __init__(self, proj, layers, logits, mode="f32", device=None):
        self.mode = mode
        self.stack = DeviceStack(CellKind.SRU, layers, mode=mode, device=device)
        dev = torch.device("cuda", self.stack.device)
        wdt = torch.bfloat16 if mode == "bf16" else torch.float32
        self.wdt = wdt
        self.proj = torch.as_tensor(proj).to(dev, wdt)
        self.logits = torch.as_tensor(logits).to(dev, wdt)

    def _linear(self, x, w):
        prev = torch.backends.cuda.matmul.allow_tf32
        torch.backends.cuda.matmul.allow_tf32 = self.mode == "tf32"
        try:
            return (x.to(self.wdt) @ w.t()).float()
        finally:
            torch.backends.cuda.matmul.allow_tf32 = prev

    def forward(self, frames, block_size):
        """frames [L x 120] (CUDA, fp32) -> logits [L x 2000] (fp32)."""
        h = self._linear(frames, self.proj).contiguous()
        h = self.stack.forward(h, block_size)
        return self._linear(h, self.logits)

    def close(self):
        self.stack.close()
