"""Test infrastructure: executes the peer-memory partitions' schedules
(paper_1803_11389_b200.p2p.pipeline_ops / bidir_ops) on a model of G
streams with flags, with no GPU.

Every rank runs its op list in order (stream order); a wait blocks until
its flag reaches the value; signals carry the signaller's vector clock, so
a satisfied wait merges it (the flag publishes everything before it).  Each
data access is recorded with its vector clock and a tag of what was
written; `check()` then proves for one interleaving:
  * progress: every rank ran to completion (no deadlock);
  * race freedom: every pair of overlapping accesses with a write is
    ordered by happens-before (vector clocks), i.e. no interleaving can
    reorder them;
  * data flow: every read sees the tag it must (the intended producer).
"""

import random

from paper_1803_11389_b200.p2p import bidir_ops, pipeline_ops
from paper_1803_11389_b200.partition import chunk_plan


class Deadlock(AssertionError):
    pass


class Sim:
    def __init__(self, world):
        self.world = world
        self.flags = {}     # (owner, name, index) -> (value, vclock)
        self.data = {}      # region -> tag
        self.log = []       # (rank, vclock, region, is_write, tag_seen_or_written)
        self.vc = [[0] * world for _ in range(world)]

    # ---- primitives used by the op interpreters
    def flag(self, owner, name, idx):
        return self.flags.get((owner, name, idx), (0, [0] * self.world))

    def try_wait(self, rank, owner_name_idx, value):
        v, clk = self.flag(*owner_name_idx)
        if v < value:
            return False
        self.vc[rank] = [max(a, b) for a, b in zip(self.vc[rank], clk)]
        return True

    def signal(self, rank, key, value):
        old, _ = self.flag(*key)
        assert value >= old, f"flag {key} went backwards: {old} -> {value}"
        self.flags[key] = (value, list(self.vc[rank]))

    def access(self, rank, region, write, tag=None, expect=None):
        if write:
            self.data[region] = tag
            self.log.append((rank, list(self.vc[rank]), region, True, tag))
        else:
            seen = self.data.get(region)
            if expect is not None:
                assert seen == expect, f"rank {rank} read {region}: saw {seen}, expected {expect}"
            self.log.append((rank, list(self.vc[rank]), region, False, seen))

    def tick(self, rank):
        self.vc[rank][rank] += 1

    # ---- checks
    def check_races(self, overlap):
        def hb(a, b):
            return all(x <= y for x, y in zip(a, b))
        for i, (ra, va, ga, wa, _) in enumerate(self.log):
            for rb, vb, gb, wb, _ in self.log[i + 1:]:
                if not (wa or wb) or not overlap(ga, gb):
                    continue
                assert hb(va, vb) or hb(vb, va), f"race: rank {ra} {ga} ({'w' if wa else 'r'}) vs rank {rb} {gb}"


def run(sim, programs, step, order=None, seed=0):
    """programs[r]: op list; step(sim, rank, op) -> False if the op blocks.
    order: None = random interleaving; else a list of (rank, n_ops) bursts
    executed in that order (each op must be runnable when reached)."""
    pcs = [0] * len(programs)
    rng = random.Random(seed)
    if order is not None:
        for r, n in order:
            for _ in range(n):
                op = programs[r][pcs[r]]
                if not step(sim, r, op):
                    raise Deadlock(f"rank {r} blocked at {op} in the enqueue order")
                sim.tick(r)
                pcs[r] += 1
        assert all(pc == len(p) for pc, p in zip(pcs, programs))
        return
    while True:
        live = [r for r in range(len(programs)) if pcs[r] < len(programs[r])]
        if not live:
            return
        rng.shuffle(live)
        for r in live:
            if step(sim, r, programs[r][pcs[r]]):
                sim.tick(r)
                pcs[r] += 1
                break
        else:
            raise Deadlock("no rank can make progress: " +
                           ", ".join(f"rank {r} at {programs[r][pcs[r]]}" for r in live))


# ---------------------------------------------------------------------------
# layer pipeline


def pipeline_programs(world, L, chunk, T_b, slots, calls=1):
    progs = []
    for g in range(world):
        ops, seq = [], 0
        for c in range(calls):
            ops += [(c,) + op for op in pipeline_ops(g, world, L, chunk, T_b, slots, seq)]
            seq += len(chunk_plan(L, chunk, T_b))
        progs.append(ops)
    return progs


def pipeline_step(sim, g, op):
    call, kind = op[0], op[1]
    world = sim.world
    if kind == "reset":
        return True
    if kind == "wait":
        _, _, k, buf, slot, gen = op
        return sim.try_wait(g, (g, buf, slot), gen)
    if kind == "signal":
        _, _, k, peer, buf, slot, gen = op
        sim.signal(g, (peer, buf, slot), gen)
        return True
    if kind == "stage":
        _, _, k, t0, n, src, dst = op
        if src[0] == "ring":
            sim.access(g, (g, "ring", src[1]), False, expect=("h", g - 1, call, k))
        if dst[0] == "peer_ring":
            sim.access(g, (g + 1, "ring", dst[1]), True, tag=("h", g, call, k))
        else:
            assert g == world - 1
            sim.access(g, (g, "out", call, k), True, tag=("h", g, call, k))
        return True
    raise AssertionError(op)


def pipeline_overlap(a, b):
    return a == b


def pipeline_global_order(world, L, chunk, T_b, slots, calls=1):
    """The bursts run_local_pipeline enqueues: chunk by chunk, rank by rank."""
    nk = len(chunk_plan(L, chunk, T_b))
    progs = pipeline_programs(world, L, chunk, T_b, slots, calls)
    order = []
    for c in range(calls):
        for k in range(nk):
            for g in range(world):
                n = sum(1 for op in progs[g] if op[0] == c and op[2] == k)
                order.append((g, n))
    return progs, order


# ---------------------------------------------------------------------------
# sharded bidirectional stack


def bidir_programs(world, n_layers, calls=1):
    progs = []
    for g in range(world):
        ops = []
        for c in range(calls):
            ops += [(c,) + op for op in bidir_ops(g, world, n_layers, c)]
        progs.append(ops)
    return progs


def bidir_step(n_layers):
    def step(sim, g, op):
        call, kind = op[0], op[1]
        world = sim.world
        if kind == "input":
            return True
        if kind == "wait":
            _, _, li, i, value = op
            return sim.try_wait(g, (g, "flags", i), value)
        if kind == "signal":
            _, _, li, p, i, value = op
            sim.signal(g, (p, "flags", i), value)
            return True
        if kind == "dir":
            _, _, li, d, src, dst = op
            if src[0] == "act":
                for dd in range(2):
                    for q in range(world):
                        sim.access(g, (g, ("act", src[1]), dd, q), False, expect=(call, li - 1, dd, q))
            name = "final" if dst[0] == "final" else ("act", dst[1])
            for p in range(world):
                sim.access(g, (p, name, d, g), True, tag=(call, li, d, g))
            return True
        if kind == "result":
            for dd in range(2):
                for q in range(world):
                    sim.access(g, (g, "final", dd, q), False, expect=(call, n_layers - 1, dd, q))
            return True
        raise AssertionError(op)
    return step


def bidir_overlap(a, b):
    return a == b


def bidir_global_order(world, n_layers, calls=1):
    """run_local_bidir's bursts: layer by layer (index n_layers = the closing
    wait and result copy), rank by rank."""
    progs = bidir_programs(world, n_layers, calls)
    order = []
    for c in range(calls):
        for li in range(n_layers + 1):
            for g in range(world):
                n = sum(1 for op in progs[g] if op[0] == c and op[2] == li)
                order.append((g, n))
    return progs, order
