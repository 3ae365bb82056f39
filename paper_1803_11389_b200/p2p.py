"""Fused peer-memory partitions: the layer kernels' own
epilogue stores carry the activations to the GPU that needs them.

`partition.py` is the NCCL baseline: a rank computes a chunk, then
`dist.isend` / `dist.all_gather` move it between launches.  Here nothing
moves after the math: the LAST layer of a rank's stage stores each h value
straight into the consumer's buffer over NVLink (`rnnb_forward_ex`, mapped
peer addresses), and a stream-ordered flag (`rnnb_flag_signal`, a one-thread
release store after the layer kernel) tells the consumer the rows are
there; the consumer's stream waits on it with a stream wait-value operation
(`rnnb_flag_wait`), so no kernel ever spins on another rank.

* `P2PPipelineStage` -- layer pipelining of time chunks (BASELINE cfg4).
  Rank g > 0 owns an input ring of S slots [chunk x d_in] plus one `full`
  flag per slot; rank g < G-1 owns one `credit` flag per slot.  Chunk q
  (slot q % S, generation q // S + 1) on rank g: wait full[slot] >= gen
  (g > 0); wait credit[slot] >= gen - 1 (the next rank has consumed the
  slot's previous chunk; g < G-1); run the stage with its last layer storing
  into the NEXT rank's ring slot; signal next.full[slot] = gen and
  prev.credit[slot] = gen.  c and the QRNN x_{t-1} carry across chunks
  through the C ABI's state in/out, exactly as across blocks
  (blocked.py:247-264), so outputs are bitwise those of one unpartitioned
  call with the same chunk plan.

* `P2PBidirSRU` -- hidden-dimension sharding of a bidirectional SRU stack
  with the all-gather fused into the epilogue (BASELINE cfg5).  Rank g owns
  units [g H/G, (g+1) H/G) of each direction.  Each direction's last (only)
  layer of a stage stores its h slice into EVERY rank's next-layer input
  [L x 2H] at the slice's columns (its own copy plus G-1 mapped peers); the
  backward direction runs on a time-reversed copy of the input and stores
  with a negative row stride, i.e. straight into forward time order.  After
  a layer, a rank signals its flag on every rank; before the next layer it
  waits for all G flags.  Two intermediate buffers alternate (a rank writes
  layer l's output into a peer's buffer only after every rank finished
  layer l-1, which read the other buffer) and the last layer writes a third
  one, so a result is never overwritten by the next call.

Ranks connect either through CUDA IPC (one process per GPU:
`connect_ipc`, handles exchanged with `all_gather_object`) or directly
(`connect_local`: several rank objects in one process -- GPUs with peer
access, or emulated ranks sharing one GPU).  `run_local_*` enqueue the
ranks' work in global (chunk, rank) / (layer, rank) order: every wait then
depends only on work enqueued before it, so execution cannot deadlock even
if streams share a hardware queue.
"""

import ctypes

import torch
import torch.distributed as dist

from . import _lib
from .cells import CellKind
from .partition import chunk_plan, unit_range

FLAG_STRIDE = 32  # int32 flags one 128-byte line apart


def signal(device, addr, value, stream):
    _lib.check(_lib.load().rnnb_flag_signal(int(device), ctypes.c_void_p(int(addr)), int(value) & 0xFFFFFFFF,
                                            ctypes.c_void_p(stream.cuda_stream)))


def wait(device, addr, value, stream):
    _lib.check(_lib.load().rnnb_flag_wait(int(device), ctypes.c_void_p(int(addr)), int(value) & 0xFFFFFFFF,
                                          ctypes.c_void_p(stream.cuda_stream)))


class _PeerBuffers:
    """Named device tensors this rank exports; `self.peer[r][name]` is the
    address of rank r's tensor as this rank sees it."""

    rank = 0
    world = 1

    def _exports(self):
        raise NotImplementedError

    def connect_local(self, ranks):
        """All rank objects live in this process (addresses usable directly)."""
        self.peer = {o.rank: {n: t.data_ptr() for n, t in o._exports().items()} for o in ranks}
        self._opened = []

    def connect_ipc(self, group=None):
        """One process per GPU: export by CUDA IPC, import every peer's."""
        lib = _lib.load()
        mine = {}
        for n, t in self._exports().items():
            hb = ctypes.create_string_buffer(_lib.IPC_HANDLE_BYTES)
            off = ctypes.c_uint64()
            _lib.check(lib.rnnb_ipc_handle(ctypes.c_void_p(t.data_ptr()), hb, ctypes.byref(off)))
            mine[n] = (hb.raw, off.value)
        allt = [None] * self.world
        dist.all_gather_object(allt, (self.rank, mine), group=group)
        self.peer, self._opened = {}, []
        bases = {}
        for r, tab in allt:
            if r == self.rank:
                self.peer[r] = {n: t.data_ptr() for n, t in self._exports().items()}
                continue
            d = {}
            for n, (hb, off) in tab.items():
                if hb not in bases:  # one open per allocation
                    base = ctypes.c_void_p()
                    _lib.check(lib.rnnb_ipc_open(self.device, hb, ctypes.byref(base)))
                    bases[hb] = base.value
                    self._opened.append(base.value)
                d[n] = bases[hb] + off
            self.peer[r] = d

    def close(self):
        lib = _lib.load()
        for b in getattr(self, "_opened", []):
            lib.rnnb_ipc_close(self.device, ctypes.c_void_p(b))
        self._opened = []


# ---------------------------------------------------------------------------
# layer pipeline (cfg4)


class P2PPipelineStage(_PeerBuffers):
    """Rank `rank`'s contiguous layer range (a DeviceStack) in a G-stage
    pipeline whose hand-off is the last layer's epilogue stores."""

    def __init__(self, stack, rank, world, chunk, block_size, slots=2, stream=None):
        if chunk % block_size:
            raise ValueError("pipeline chunk must be a multiple of the block size")
        if slots < 1:
            raise ValueError("need at least one ring slot")
        if stack.dtype != torch.float32:
            raise ValueError("the peer-memory pipeline carries fp32 activations")
        self.stack, self.rank, self.world = stack, rank, world
        self.chunk, self.block_size, self.slots = chunk, block_size, slots
        self.device = stack.device
        dev = torch.device("cuda", self.device)
        self.d_in, self.d_out = stack.d_in[0], stack.d_h[-1]
        self.c = torch.zeros(sum(stack.d_h), dtype=torch.float32, device=dev)
        self.xc = torch.zeros(sum(stack.d_in), dtype=torch.float32, device=dev)
        self.ring = torch.empty((slots, chunk, self.d_in), dtype=torch.float32, device=dev) if rank > 0 else None
        self.full = torch.zeros(slots * FLAG_STRIDE, dtype=torch.int32, device=dev) if rank > 0 else None
        self.credit = torch.zeros(slots * FLAG_STRIDE, dtype=torch.int32, device=dev) if rank < world - 1 else None
        self.stream = stream if stream is not None else torch.cuda.Stream(device=dev)
        self.seq = 0  # chunks handed through so far (flags are monotone generations)
        self.peer = None

    def _exports(self):
        out = {}
        if self.ring is not None:
            out["ring"], out["full"] = self.ring, self.full
        if self.credit is not None:
            out["credit"] = self.credit
        return out

    def enqueue(self, L, X=None, out=None, chunks=None):
        """Enqueue this rank's sequence (or the chunk indices `chunks`) on its
        stream; returns at once.  Rank 0 reads X [L x d_in] (CUDA tensor on
        its device); the last rank writes out [L x d_out]."""
        if self.peer is None:
            raise RuntimeError("connect_local / connect_ipc first")
        if self.rank == 0 and (X is None or X.shape[0] != L or X.stride(1) != 1):
            raise ValueError("rank 0 needs X [L x d_in], row-major")
        if self.rank == self.world - 1 and (out is None or out.shape[0] != L or out.stride(1) != 1):
            raise ValueError("the last rank needs out [L x d_out], row-major")
        ops = pipeline_ops(self.rank, self.world, L, self.chunk, self.block_size, self.slots, self.seq)
        for op in ops if chunks is None else [o for o in ops if o[1] in chunks]:
            self._run(op, X, out)

    def advance(self, L):
        """Close a sequence: the next one continues the flag generations."""
        self.seq += len(chunk_plan(L, self.chunk, self.block_size))

    def _run(self, op, X, out):
        s, dev, kind = self.stream, self.device, op[0]
        flag = FLAG_STRIDE * 4
        if kind == "reset":
            s.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(s):
                self.c.zero_()
                self.xc.zero_()
        elif kind == "wait":
            _, _, buf, slot, gen = op
            wait(dev, getattr(self, buf).data_ptr() + slot * flag, gen, s)
        elif kind == "signal":
            _, _, peer, buf, slot, gen = op
            signal(dev, self.peer[peer][buf] + slot * flag, gen, s)
        elif kind == "stage":
            _, _, t0, n, src, dst = op
            if src[0] == "X":
                xp, ldx = X.data_ptr() + t0 * X.stride(0) * 4, X.stride(0)
            else:
                xp, ldx = self.ring[src[1]].data_ptr(), self.d_in
            if dst[0] == "out":
                hp, ldh = out.data_ptr() + t0 * out.stride(0) * 4, out.stride(0)
            else:  # the next rank's ring slot: the epilogue stores cross NVLink
                hp, ldh = self.peer[self.rank + 1]["ring"] + dst[1] * self.chunk * self.d_out * 4, self.d_out
            self.stack.forward_ptr(xp, ldx, n, self.block_size, hp, ldh, c_state=self.c, x_carry=self.xc, stream=s)
        else:
            raise ValueError(f"unknown op {kind}")

    def finish(self):
        torch.cuda.current_stream(self.device).wait_stream(self.stream)


def pipeline_ops(rank, world, L, chunk, block_size, slots, seq0=0):
    """This rank's schedule for one sequence, as data (the CUDA executor is
    P2PPipelineStage._run; tests execute it in a simulator).  Every op is
    (kind, chunk_index, ...):
      ("reset", 0)                                  zero c / x_carry
      ("wait", k, "full" | "credit", slot, gen)     stream waits own flag >= gen
      ("stage", k, t0, n, src, dst)                 src ("X",) | ("ring", slot);
                                                    dst ("out",) | ("peer_ring", slot)
      ("signal", k, peer, "full" | "credit", slot, gen)"""
    ops = [("reset", 0)]
    first, last = rank == 0, rank == world - 1
    for k, (t0, n) in enumerate(chunk_plan(L, chunk, block_size)):
        q = seq0 + k
        slot, gen = q % slots, q // slots + 1
        if not first:
            ops.append(("wait", k, "full", slot, gen))
        if not last and gen > 1:
            ops.append(("wait", k, "credit", slot, gen - 1))
        ops.append(("stage", k, t0, n, ("X",) if first else ("ring", slot), ("out",) if last else ("peer_ring", slot)))
        if not last:
            ops.append(("signal", k, rank + 1, "full", slot, gen))
        if not first:
            ops.append(("signal", k, rank - 1, "credit", slot, gen))
    return ops


def run_local_pipeline(stages, X, L):
    """Emulated / single-process pipeline: enqueue every rank's chunks in
    global (chunk, rank) order, return the last rank's output [L x d_out]."""
    last = stages[-1]
    out = torch.empty((L, last.d_out), dtype=torch.float32, device=torch.device("cuda", last.device))
    nk = len(chunk_plan(L, stages[0].chunk, stages[0].block_size))
    for k in range(nk):  # one chunk per rank at a time: every wait sits behind the work it needs
        for st in stages:
            st.enqueue(L, X if st.rank == 0 else None, out if st.rank == st.world - 1 else None, chunks=(k,))
    for st in stages:
        st.advance(L)
        st.finish()
    return out


# ---------------------------------------------------------------------------
# hidden-dimension sharding with the all-gather in the epilogue (cfg5)


class P2PBidirSRU(_PeerBuffers):
    """Rank `rank`'s units of a bidirectional SRU stack (cfg5) whose
    per-layer all-gather is the epilogue's stores into every rank's buffer.

    layers_fwd / layers_bwd: per layer the FULL weights (canonical SRU
    fields, [H x d_in]); this rank slices its units (as
    partition.ShardedBidirSRU)."""

    def __init__(self, layers_fwd, layers_bwd, rank, world, block_size, mode, seq_len, device=None, stream=None):
        from .device import DeviceStack
        self.rank, self.world, self.block_size, self.L = rank, world, block_size, seq_len
        self.device = torch.cuda.current_device() if device is None else device
        dev = torch.device("cuda", self.device)
        self.H = layers_fwd[0].mats()[0].shape[0]
        self.u0, self.u1 = unit_range(self.H, world, rank)
        self.n_layers = len(layers_fwd)
        self.d_in0 = layers_fwd[0].mats()[0].shape[1]
        self.stages = []
        for lf, lb in zip(layers_fwd, layers_bwd):
            per_dir = []
            for d, lay in enumerate((lf, lb)):
                m = lay.mats()
                mats = tuple(x[self.u0:self.u1] for x in m[:5])
                d_in = m[0].shape[1]
                hw = self.u0 if d_in == self.H else d * self.H + self.u0
                per_dir.append(DeviceStack(CellKind.SRU, [mats], mode=mode, device=self.device, wide=True,
                                           highway_offsets=[hw]))
            self.stages.append(per_dir)
        W = 2 * self.H
        self.act = torch.empty((2, seq_len, W), dtype=torch.float32, device=dev)
        self.final = torch.empty((seq_len, W), dtype=torch.float32, device=dev)
        self.flags = torch.zeros(2 * world * FLAG_STRIDE, dtype=torch.int32, device=dev)
        self.stream = stream if stream is not None else torch.cuda.Stream(device=dev)
        self.epoch = 0
        self.peer = None

    def _exports(self):
        return {"act": self.act, "final": self.final, "flags": self.flags}

    def enqueue(self, X, out, layers=None):
        """Enqueue this rank's schedule for one call (or only the ops of
        `layers`; index n_layers = the closing wait + result copy into out
        [L x 2H]) on its stream; returns at once."""
        if self.peer is None:
            raise RuntimeError("connect_local / connect_ipc first")
        if X is not None and (X.shape != (self.L, self.d_in0) or X.stride(1) != 1):
            raise ValueError(f"X must be [{self.L} x {self.d_in0}], row-major")
        for op in bidir_ops(self.rank, self.world, self.n_layers, self.epoch):
            if layers is None or op[1] in layers:
                self._run(op, X, out)

    def _buf(self, ref):
        """(name, local tensor, element offset inside the exported tensor)."""
        if ref[0] == "final":
            return "final", self.final, 0
        return "act", self.act[ref[1]], ref[1] * self.L * 2 * self.H

    def _run(self, op, X, out):
        s, dev, L, H, W = self.stream, self.device, self.L, self.H, 2 * self.H
        flag = FLAG_STRIDE * 4
        kind = op[0]
        if kind == "input":
            s.wait_stream(torch.cuda.current_stream(dev))
        elif kind == "wait":
            _, _, i, value = op
            wait(dev, self.flags.data_ptr() + i * flag, value, s)
        elif kind == "signal":
            _, _, p, i, value = op
            signal(dev, self.peer[p]["flags"] + i * flag, value, s)
        elif kind == "result":
            with torch.cuda.stream(s):
                out.copy_(self.final)
        elif kind == "dir":
            _, li, d, src, dst = op
            x = X if src[0] == "X" else self.act[src[1]]
            name, t, off = self._buf(dst)
            others = [p for p in range(self.world) if p != self.rank]
            st = self.stages[li][d]
            if d == 0:  # forward direction: time order, columns [u0, u1)
                col, row, ldh = self.u0, 0, W
                xp, ldx = x.data_ptr(), x.stride(0)
            else:  # backward: the input read in reverse (negative row stride, no copy on the
                # tensor-core path), negative-stride stores at [H + u0, H + u1)
                col, row, ldh = H + self.u0, (L - 1) * W, -W
                xp, ldx = x.data_ptr() + (L - 1) * x.stride(0) * x.element_size(), -x.stride(0)
            st.forward_ptr(xp, ldx, L, self.block_size, t.data_ptr() + (row + col) * 4, ldh,
                           peers=[self.peer[p][name] + (off + row + col) * 4 for p in others], stream=s)
        else:
            raise ValueError(f"unknown op {kind}")

    def close_call(self):
        self.epoch += 1

    def close(self):
        super().close()
        for per_dir in self.stages:
            for st in per_dir:
                st.close()

    def forward(self, X):
        """One process per GPU: the whole stack; returns [L x 2H]."""
        out = torch.empty((self.L, 2 * self.H), dtype=torch.float32, device=self.final.device)
        self.enqueue(X, out)
        self.close_call()
        torch.cuda.current_stream(self.device).wait_stream(self.stream)
        return out


def bidir_ops(rank, world, n_layers, epoch=0):
    """This rank's schedule for one call of the sharded bidirectional stack,
    as data (CUDA executor: P2PBidirSRU._run; tests simulate it).  Flags:
    own flags[p] (p < G) = layers rank p finished, flags[G + p] = calls whose
    result rank p has copied out.  Ops are (kind, layer, ...):
      ("input", 0)                 X is ready (stream order after the caller)
      ("wait", l, i, v)            own flags[i] >= v
      ("dir", l, d, src, dst)      direction d of layer l: reads src ("X",) |
                                   ("act", j); stores its unit slice into dst
                                   ("act", j) | ("final",) on EVERY rank
      ("signal", l, p, i, v)       flags[i] on rank p = v
      ("result", n_layers)         copy `final` out (the call's return value)"""
    tag = epoch * n_layers
    ops = [("input", 0)]
    for li in range(n_layers):
        if li > 0:  # every rank's slice of layer li-1 is in place
            ops += [("wait", li, p, tag + li) for p in range(world)]
        if li == n_layers - 1 and epoch > 0:  # every rank copied the previous call's result out
            ops += [("wait", li, world + p, epoch) for p in range(world)]
        src = ("X",) if li == 0 else ("act", (li - 1) % 2)
        dst = ("final",) if li == n_layers - 1 else ("act", li % 2)
        ops += [("dir", li, 0, src, dst), ("dir", li, 1, src, dst)]
        ops += [("signal", li, p, rank, tag + li + 1) for p in range(world)]
    ops += [("wait", n_layers, p, tag + n_layers) for p in range(world)]
    ops += [("result", n_layers)]
    ops += [("signal", n_layers, p, world + rank, epoch + 1) for p in range(world)]
    return ops


def run_local_bidir(ranks, X):
    """Emulated / single-process sharded stack: enqueue in global (layer,
    rank) order; returns every rank's copy of the output."""
    outs = [torch.empty((r.L, 2 * r.H), dtype=torch.float32, device=r.final.device) for r in ranks]
    for li in range(ranks[0].n_layers + 1):
        for r, o in zip(ranks, outs):
            r.enqueue(X, o, layers=(li,))
    for r in ranks:
        r.close_call()
        torch.cuda.current_stream(r.device).wait_stream(r.stream)
    return outs


def bidir_reference(layers_fwd, layers_bwd, X, block_size, mode, device=None):
    """Unsharded, unfused composition of the same stack (one GPU, torch
    flips and concatenation) -- what the fused, sharded run must equal."""
    from .device import DeviceStack
    x = X
    H = layers_fwd[0].mats()[0].shape[0]
    for lf, lb in zip(layers_fwd, layers_bwd):
        ys = []
        for d, lay in enumerate((lf, lb)):
            m = lay.mats()
            d_in = m[0].shape[1]
            hw = 0 if d_in == H else d * H
            st = DeviceStack(CellKind.SRU, [tuple(m[:5])], mode=mode, device=device, wide=True, highway_offsets=[hw])
            xin = x if d == 0 else torch.flip(x, dims=[0]).contiguous()
            y = st.forward(xin, block_size)
            ys.append(y if d == 0 else torch.flip(y, dims=[0]))
            st.close()
        x = torch.cat(ys, dim=1).contiguous()
    return x

