"""Multi-GPU partitioning of the blocked path.

Two partitions, both one process per GPU over torch.distributed (NCCL on
CUDA tensors; the host logic is identical over gloo on CPU tensors, which
is how tests/test_partition.py covers it without GPUs):

* Layer pipelining of time chunks (BASELINE cfg4, deep QRNN stack).  Rank g
  owns a contiguous range of layers.  The sequence is cut into pipeline
  chunks of C steps (a multiple of T_b); rank g runs its layers over chunk
  k -- c and the QRNN x_{t-1} carry are carried across chunks exactly as
  across blocks (blocked.py:247-264) -- and sends the chunk's last-layer
  activations [C x d_h] to rank g+1 (point-to-point), while already
  computing chunk k+1.  Every rank issues the same arithmetic for every
  chunk whatever the GPU count, so outputs are bitwise identical across
  world sizes; the fill bubble is (G-1)/n_chunks.

* Hidden-dimension sharding with a per-layer all-gather (BASELINE cfg5, wide
  bidirectional SRU).  Rank g owns units [g*H/G, (g+1)*H/G) of each
  direction of each layer: the 3 gate rows of those units over the full
  input width, so its projection + scan is local and independent.  The
  direction outputs h-slices [L x H/G] are all-gathered into the next
  layer's input [L x 2H] (forward units then backward units).  The order is
  layer-major because the backward direction needs the whole sequence;
  the forward direction's all-gather is issued asynchronously and overlaps
  the backward direction's compute.  A unit's reduction never depends on
  G, so outputs are bitwise identical across world sizes.

Stage compute is pluggable: ``DeviceStage`` wraps a ``DeviceStack`` (CUDA
kernels); tests plug in the CPU oracle.
"""

import numpy as np
import torch
import torch.distributed as dist

from .cells import CellKind


# ---------------------------------------------------------------------------
# partition arithmetic


def layer_ranges(n_layers, world):
    """Contiguous layer ranges per rank, sizes differing by at most one."""
    if world < 1 or n_layers < world:
        raise ValueError("need at least one layer per rank")
    base, rem = divmod(n_layers, world)
    out, lo = [], 0
    for g in range(world):
        hi = lo + base + (1 if g < rem else 0)
        out.append((lo, hi))
        lo = hi
    return out


def unit_range(H, world, rank):
    """Units of one direction owned by `rank` (H divisible by world)."""
    if H % world:
        raise ValueError(f"hidden width {H} must divide by world size {world}")
    per = H // world
    return rank * per, (rank + 1) * per


def chunk_plan(L, chunk, block_size):
    """Pipeline chunks: multiples of T_b so chunk edges are block edges."""
    if chunk % block_size:
        raise ValueError("pipeline chunk must be a multiple of the block size")
    return [(s, min(chunk, L - s)) for s in range(0, L, chunk)]


# ---------------------------------------------------------------------------
# stage compute


class DeviceStage:
    """A contiguous layer range on one GPU with carried (c, x_carry) state."""

    def __init__(self, stack, block_size):
        self.stack = stack
        self.block_size = block_size
        dev = torch.device("cuda", stack.device)
        self.c = torch.zeros(sum(stack.d_h), dtype=stack.dtype, device=dev)
        self.xc = torch.zeros(sum(stack.d_in), dtype=stack.dtype, device=dev)

    def reset(self):
        self.c.zero_()
        self.xc.zero_()

    def __call__(self, x):
        return self.stack.forward(x, self.block_size, c_state=self.c, x_carry=self.xc)


# ---------------------------------------------------------------------------
# layer pipeline (cfg4)


def pipeline_forward(stage, X, L, d_out, chunk, block_size, rank, world, dtype, device, group=None):
    """Run the sequence through the rank pipeline; rank 0 feeds X (its
    layers read it directly), the last rank returns the output [L x d_out]
    (other ranks return None).  `stage(x_chunk) -> y_chunk` carries its own
    recurrent state across chunks."""
    plan = chunk_plan(L, chunk, block_size)
    out = torch.empty((L, d_out), dtype=dtype, device=device) if rank == world - 1 else None
    pending = []
    for s, n in plan:
        if rank == 0:
            x = X[s:s + n]
        else:
            x = torch.empty((n, stage_in_width(stage)), dtype=dtype, device=device)
            dist.recv(x, src=rank - 1, group=group)
        y = stage(x)
        if rank == world - 1:
            out[s:s + n] = y
        else:
            pending.append(dist.isend(y.contiguous(), dst=rank + 1, group=group))
            if len(pending) > 2:  # bounded double buffering
                pending.pop(0).wait()
    for p in pending:
        p.wait()
    return out


def stage_in_width(stage):
    return stage.d_in if hasattr(stage, "d_in") and isinstance(stage.d_in, int) else stage.stack.d_in[0]


# ---------------------------------------------------------------------------
# hidden sharding (cfg5)


class ShardedBidirSRU:
    """Bidirectional SRU stack, hidden dimension sharded over ranks.

    layers_fwd / layers_bwd: per layer the FULL weights (canonical SRU
    fields, [H x d_in] matrices); this rank slices its units.  `make_stage`
    builds the per-(layer, direction) compute for (mats, hw_offset):
    a callable x [L x d_in] -> h [L x H/G] over the whole sequence."""

    def __init__(self, layers_fwd, layers_bwd, rank, world, make_stage, group=None):
        self.rank, self.world, self.group = rank, world, group
        self.H = layers_fwd[0].mats()[0].shape[0]
        u0, u1 = unit_range(self.H, world, rank)
        self.u0, self.u1 = u0, u1
        self.stages = []
        for li, (lf, lb) in enumerate(zip(layers_fwd, layers_bwd)):
            per_dir = []
            for d, lay in enumerate((lf, lb)):
                m = lay.mats()
                mats = (m[0][u0:u1], m[1][u0:u1], m[2][u0:u1], m[3][u0:u1], m[4][u0:u1])
                d_in = m[0].shape[1]
                # highway: the layer's own input column of this unit; for stacked
                # layers the direction-aligned half of the concatenated input
                hw = u0 if d_in == self.H else d * self.H + u0
                per_dir.append(make_stage(mats, hw))
            self.stages.append(per_dir)

    def _gather(self, y_local, async_op=False):
        parts = [torch.empty_like(y_local) for _ in range(self.world)]
        h = dist.all_gather(parts, y_local.contiguous(), group=self.group, async_op=async_op)
        return parts, h

    def forward(self, X):
        x = X
        for per_dir in self.stages:
            yf = per_dir[0](x)
            parts_f, hf = self._gather(yf, async_op=True)       # overlaps the backward pass
            yb = torch.flip(per_dir[1](torch.flip(x, dims=[0]).contiguous()), dims=[0])
            parts_b, hb = self._gather(yb, async_op=False)
            hf.wait()
            x = torch.cat(parts_f + parts_b, dim=1).contiguous()
        return x


def wide_sru_stage_factory(block_size, mode, device):
    """make_stage for ShardedBidirSRU on the CUDA kernels."""
    from .device import DeviceStack

    def make(mats, hw_offset):
        st = DeviceStack(CellKind.SRU, [mats], mode=mode, device=device, wide=True,
                         highway_offsets=[hw_offset])
        return lambda x: st.forward(x, block_size)
    return make
