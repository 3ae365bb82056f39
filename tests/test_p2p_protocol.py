"""Host logic of the fused peer-memory partitions (paper_1803_11389_b200/p2p.py),
on CPU: the schedules are executed by a model of streams + flags
(tests/p2p_sim.py) that proves progress, race freedom (vector clocks) and
data flow for random interleavings and for the order the single-process
emulation enqueues in.  The CUDA executor of the same schedules is tested
in tests/test_gpu_p2p.py."""

import pytest

import p2p_sim as S
from paper_1803_11389_b200.p2p import bidir_ops, pipeline_ops


@pytest.mark.parametrize("world,slots,L,chunk,T_b", [
    (2, 1, 256, 64, 32), (2, 2, 1000, 128, 32), (3, 2, 777, 96, 16), (4, 3, 4096, 256, 32), (8, 2, 2048, 64, 32),
])
@pytest.mark.parametrize("seed", [0, 1, 2])
def test_pipeline_schedule_random_interleavings(world, slots, L, chunk, T_b, seed):
    sim = S.Sim(world)
    progs = S.pipeline_programs(world, L, chunk, T_b, slots, calls=2)
    S.run(sim, progs, S.pipeline_step, seed=seed)
    sim.check_races(S.pipeline_overlap)


@pytest.mark.parametrize("world,slots", [(2, 1), (2, 2), (4, 2), (8, 3)])
def test_pipeline_enqueue_order_never_blocks(world, slots):
    # run_local_pipeline's (chunk, rank) order executed strictly in sequence:
    # every wait is already satisfied, so streams sharing a hardware queue
    # cannot deadlock
    progs, order = S.pipeline_global_order(world, 1000, 64, 32, slots, calls=2)
    sim = S.Sim(world)
    S.run(sim, progs, S.pipeline_step, order=order)
    sim.check_races(S.pipeline_overlap)


def test_pipeline_ops_shape():
    ops = pipeline_ops(1, 3, 300, 128, 32, 2)
    kinds = [o[0] for o in ops]
    assert kinds[0] == "reset"
    # middle rank: wait full, (credit from the 3rd chunk on), stage, signal next, signal prev
    assert kinds[1:6] == ["wait", "stage", "signal", "signal", "wait"]
    assert [o for o in ops if o[0] == "wait" and o[2] == "credit"] == [("wait", 2, "credit", 0, 1)]
    st = [o for o in ops if o[0] == "stage"]
    assert [(o[2], o[3]) for o in st] == [(0, 128), (128, 128), (256, 44)]
    with pytest.raises(ValueError):
        pipeline_ops(0, 2, 100, 48, 32, 2)


def test_pipeline_generations_continue_across_calls():
    a = pipeline_ops(0, 2, 256, 64, 32, 3, seq0=0)
    b = pipeline_ops(0, 2, 256, 64, 32, 3, seq0=4)
    gens_a = [o[-1] for o in a if o[0] == "signal"]
    gens_b = [o[-1] for o in b if o[0] == "signal"]
    assert max(gens_a) <= min(gens_b)


def test_pipeline_detects_a_broken_schedule():
    # without the credit waits a fast producer overwrites a slot the consumer
    # has not read: the simulator must flag it
    progs = S.pipeline_programs(2, 1024, 64, 32, 1, calls=1)
    progs[0] = [op for op in progs[0] if not (op[1] == "wait" and op[3] == "credit")]
    sim = S.Sim(2)
    with pytest.raises(AssertionError):
        S.run(sim, progs, S.pipeline_step, seed=3)
        sim.check_races(S.pipeline_overlap)


@pytest.mark.parametrize("world,n_layers", [(1, 1), (2, 1), (2, 2), (2, 4), (3, 3), (4, 4), (8, 4)])
@pytest.mark.parametrize("seed", [0, 1])
def test_bidir_schedule_random_interleavings(world, n_layers, seed):
    sim = S.Sim(world)
    progs = S.bidir_programs(world, n_layers, calls=3)
    S.run(sim, progs, S.bidir_step(n_layers), seed=seed)
    sim.check_races(S.bidir_overlap)


@pytest.mark.parametrize("world,n_layers", [(2, 2), (4, 4), (8, 3)])
def test_bidir_enqueue_order_never_blocks(world, n_layers):
    progs, order = S.bidir_global_order(world, n_layers, calls=2)
    sim = S.Sim(world)
    S.run(sim, progs, S.bidir_step(n_layers), order=order)
    sim.check_races(S.bidir_overlap)


def test_bidir_two_buffers_are_needed_and_enough():
    ops = bidir_ops(0, 2, 4)
    dsts = [o[4] for o in ops if o[0] == "dir"]
    assert dsts == [("act", 0)] * 2 + [("act", 1)] * 2 + [("act", 0)] * 2 + [("final",)] * 2
    # one shared intermediate buffer would race: rewrite the schedule to use act 0 only
    progs = S.bidir_programs(2, 3, calls=1)
    bad = []
    for p in progs:
        q = []
        for op in p:
            if op[1] == "dir":
                c, k, li, d, src, dst = op
                src = ("act", 0) if src[0] == "act" else src
                dst = ("act", 0) if dst[0] == "act" else dst
                op = (c, k, li, d, src, dst)
            q.append(op)
        bad.append(q)
    sim = S.Sim(2)
    with pytest.raises(AssertionError):
        S.run(sim, bad, S.bidir_step(3), seed=0)
        sim.check_races(S.bidir_overlap)
