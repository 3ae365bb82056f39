"""Fused peer-memory partitions on the CUDA kernels (paper_1803_11389_b200/p2p.py).

One GPU per gpurun call, so the G ranks are emulated as rank objects in one
process sharing cuda:0, each with its own stream and buffers; the "peer"
addresses are then the other ranks' local buffers, written by the same
epilogue stores that write mapped NVLink addresses across GPUs.  No kernel
waits on another (stream wait-value operations only) and the ranks' work
is enqueued in an order in which every wait follows the work it needs
(proved for every interleaving by tests/test_p2p_protocol.py).
"""

import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-30))


@pytest.mark.parametrize("kind,mode,D,T_b", [
    ("qrnn", "f32", 256, 32),   # warp-specialised FFMA kernel
    ("qrnn", "f32", 256, 1),    # register-resident FFMA kernel
    ("sru", "f32", 100, 8),     # generic FFMA kernel (unaligned width)
    ("qrnn", "f64", 64, 4),
    ("sru", "bf16", 256, 32),   # tcgen05 kernel
    ("qrnn", "tf32", 256, 16),
    ("qrnn", "f32x3", 256, 32),
])
def test_forward_ex_peer_destinations_equal_the_output(oracle, kind, mode, D, T_b):
    import torch
    import paper_1803_11389_b200 as P
    layers = oracle.generate_layers(kind, D, D, 2, 11, np.float32)
    st = P.DeviceStack(kind, layers, mode=mode)
    dt = st.dtype
    X = torch.from_numpy(np.random.default_rng(4).standard_normal((203, D))).to(dt).cuda()
    ref = st.forward(X, T_b)
    out = torch.full_like(ref, float("nan"))
    peers = [torch.full_like(ref, float("nan")) for _ in range(3)]
    st.forward_ptr(X.data_ptr(), X.stride(0), X.shape[0], T_b, out.data_ptr(), out.stride(0),
                   peers=[p.data_ptr() for p in peers])
    torch.cuda.synchronize()
    r = ref.cpu().numpy()
    for t in [out] + peers:
        assert t.cpu().numpy().tobytes() == r.tobytes()
    # and a plain forward after it stores nowhere else
    peers[0].fill_(7.0)
    st.forward(X, T_b)
    torch.cuda.synchronize()
    assert bool((peers[0] == 7.0).all())
    st.close()


@pytest.mark.parametrize("mode,T_b", [("f32", 32), ("f32", 1), ("bf16", 16)])
def test_negative_row_stride_stores_reversed_time(oracle, mode, T_b):
    import torch
    import paper_1803_11389_b200 as P
    layers = oracle.generate_layers("sru", 128, 128, 1, 3, np.float32)
    st = P.DeviceStack("sru", layers, mode=mode)
    X = torch.from_numpy(np.random.default_rng(5).standard_normal((97, 128)).astype(np.float32)).cuda()
    ref = st.forward(X, T_b)
    W = 3 * 128
    buf = torch.zeros((97, W), dtype=torch.float32, device="cuda")
    # rows in reverse time order into columns [128, 256) of a wider buffer
    st.forward_ptr(X.data_ptr(), 128, 97, T_b, buf[96, 128:].data_ptr(), -W)
    torch.cuda.synchronize()
    assert torch.equal(buf[:, 128:256], torch.flip(ref, dims=[0]))
    assert bool((buf[:, :128] == 0).all()) and bool((buf[:, 256:] == 0).all())
    st.close()


def test_forward_ex_validation(oracle):
    import torch
    import paper_1803_11389_b200 as P
    layers = oracle.generate_layers("qrnn", 64, 64, 1, 3, np.float32)
    st = P.DeviceStack("qrnn", layers)
    X = torch.zeros((8, 64), device="cuda")
    H = torch.zeros((8, 64), device="cuda")
    with pytest.raises(ValueError, match="n_peers"):
        st.forward_ptr(X.data_ptr(), 64, 8, 4, H.data_ptr(), 64, peers=[H.data_ptr()] * 8)
    with pytest.raises(ValueError, match="ldh"):
        st.forward_ptr(X.data_ptr(), 64, 8, 4, H.data_ptr(), -32)
    st.close()


def _chunked_reference(st, X, chunk, T_b):
    """The unpartitioned stack over the same chunk plan, state carried."""
    import torch
    from paper_1803_11389_b200.partition import chunk_plan
    L = X.shape[0]
    c = torch.zeros(sum(st.d_h), device="cuda")
    xc = torch.zeros(sum(st.d_in), device="cuda")
    out = torch.empty((L, st.d_h[-1]), device="cuda")
    for t0, n in chunk_plan(L, chunk, T_b):
        st.forward(X[t0:t0 + n], T_b, out=out[t0:t0 + n], c_state=c, x_carry=xc)
    return out


@pytest.mark.parametrize("mode", ["f32", "bf16"])
@pytest.mark.parametrize("world,slots", [(2, 2), (4, 1), (4, 3)])
def test_p2p_pipeline_emulated_bitwise(oracle, mode, world, slots):
    import torch
    import paper_1803_11389_b200 as P
    from paper_1803_11389_b200 import p2p
    from paper_1803_11389_b200.partition import layer_ranges
    n_layers, d, L, chunk, T_b = 4, 256, 1000, 128, 32
    layers = oracle.generate_layers("qrnn", d, d, n_layers, 21, np.float32)
    whole = P.DeviceStack("qrnn", layers, mode=mode)
    X = torch.from_numpy(np.random.default_rng(6).standard_normal((L, d)).astype(np.float32)).cuda()
    ref = _chunked_reference(whole, X, chunk, T_b).cpu().numpy()
    stages = []
    for g, (lo, hi) in enumerate(layer_ranges(n_layers, world)):
        st = P.DeviceStack("qrnn", layers[lo:hi], mode=mode)
        stages.append(p2p.P2PPipelineStage(st, g, world, chunk, T_b, slots=slots))
    for s in stages:
        s.connect_local(stages)
    for call in range(2):  # flag generations continue across calls
        got = p2p.run_local_pipeline(stages, X, L)
        torch.cuda.synchronize()
        assert got.cpu().numpy().tobytes() == ref.tobytes(), (mode, world, slots, call)
    if mode == "f32":
        # and the partitioned output is the reference's run_blocked output
        want = oracle.run_blocked("qrnn", [lay.mats() if hasattr(lay, "mats") else lay for lay in layers],
                                  X.cpu().numpy(), T_b)
        assert _rel(ref, want) <= 1e-5
    for s in stages:
        s.stack.close()
    whole.close()


@pytest.mark.parametrize("mode,tol", [("f32", 1e-6), ("bf16", 1e-3)])
@pytest.mark.parametrize("world", [1, 2, 4])
def test_p2p_bidir_emulated(mode, tol, world):
    import torch
    import dist_helpers as DH
    from paper_1803_11389_b200 import p2p
    H, d0, n_layers, L, T_b = 128, 128, 3, 300, 16  # cfg5 shape: d_in == H for layer 1
    fw, bw, _ = DH.make_bidir(H=H, d0=d0, n_layers=n_layers, seed=8)
    X = torch.from_numpy(np.random.default_rng(9).standard_normal((L, d0)).astype(np.float32)).cuda()
    ref = p2p.bidir_reference(fw, bw, X, T_b, mode).cpu().numpy()
    ranks = [p2p.P2PBidirSRU(fw, bw, g, world, T_b, mode, L) for g in range(world)]
    for r in ranks:
        r.connect_local(ranks)
    for call in range(2):
        outs = p2p.run_local_bidir(ranks, X)
        torch.cuda.synchronize()
        for o in outs:
            got = o.cpu().numpy()
            assert got.tobytes() == outs[0].cpu().numpy().tobytes()  # every rank holds the same gather
            assert _rel(got, ref) <= tol, (mode, world, call, _rel(got, ref))
    if mode == "f32":
        np_ref = DH.bidir_reference(fw, bw, X.cpu().numpy().astype(np.float64))
        assert _rel(outs[0].cpu().numpy(), np_ref) <= 1e-5


def _ipc_worker(rank, world, port, result_path):
    import torch
    import torch.distributed as dist
    import paper_1803_11389_b200 as P
    from paper_1803_11389_b200 import p2p
    from paper_1803_11389_b200.partition import layer_ranges
    import oracle as O
    os.environ["MASTER_ADDR"], os.environ["MASTER_PORT"] = "127.0.0.1", str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    torch.cuda.set_device(0)
    layers = O.generate_layers("qrnn", 128, 128, 2, 21, np.float32)
    lo, hi = layer_ranges(2, world)[rank]
    st = P.DeviceStack("qrnn", layers[lo:hi])
    stage = p2p.P2PPipelineStage(st, rank, world, 64, 32, slots=2)
    stage.connect_ipc()
    L = 640
    X = torch.from_numpy(np.random.default_rng(1).standard_normal((L, 128)).astype(np.float32)).cuda()
    out = torch.empty((L, 128), device="cuda") if rank == world - 1 else None
    stage.enqueue(L, X if rank == 0 else None, out)
    stage.advance(L)
    stage.finish()
    torch.cuda.synchronize()
    dist.barrier()
    if rank == world - 1:
        np.save(result_path, out.cpu().numpy())
    stage.close()
    dist.destroy_process_group()


@pytest.mark.skipif(os.environ.get("RNNB_TEST_IPC") == "0", reason="RNNB_TEST_IPC=0")
def test_p2p_pipeline_ipc_two_processes(tmp_path, oracle):
    """Two rank processes sharing cuda:0, the pipeline hand-off through CUDA
    IPC-mapped buffers and stream-ordered flags (no kernel waits on another
    process), bitwise equal to the unpartitioned stack.  A watchdog kills the
    ranks after 180 s instead of letting a hang block the suite."""
    import socket
    import torch
    import torch.multiprocessing as mp
    import paper_1803_11389_b200 as P
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    path = str(tmp_path / "out.npy")
    import time
    ctx = mp.start_processes(_ipc_worker, args=(2, port, path), nprocs=2, join=False, start_method="spawn")
    deadline = time.time() + 180
    while not ctx.join(timeout=5):
        if time.time() > deadline:
            for p in ctx.processes:
                p.kill()
            pytest.fail("IPC pipeline ranks did not finish within 180 s")
    got = np.load(path)
    layers = oracle.generate_layers("qrnn", 128, 128, 2, 21, np.float32)
    st = P.DeviceStack("qrnn", layers)
    X = torch.from_numpy(np.random.default_rng(1).standard_normal((640, 128)).astype(np.float32)).cuda()
    ref = _chunked_reference(st, X, 64, 32).cpu().numpy()
    assert got.tobytes() == ref.tobytes()


@pytest.mark.parametrize("mode,T_b", [("f32", 16), ("f32", 64), ("bf16", 16), ("bf16", 64), ("tf32", 32)])
def test_negative_input_stride_reads_time_reversed(oracle, mode, T_b):
    """rnnb_forward_ex with ldx < 0 (the bidirectional backward direction):
    bitwise the forward over an explicitly flipped copy, on the tensor-core
    path (operand conversion walks the rows backwards) and the FFMA path (one
    reversed copy by an own kernel); QRNN x_carry = the last row READ."""
    import torch
    import paper_1803_11389_b200 as P
    for kind in ("sru", "qrnn"):
        layers = oracle.generate_layers(kind, 192, 192, 2, 31, np.float32)
        X = torch.from_numpy(np.random.default_rng(4).standard_normal((203, 192)).astype(np.float32)).cuda()
        st = P.DeviceStack(kind, layers, mode=mode)
        flipped = torch.flip(X, dims=[0]).contiguous()
        xc1 = torch.zeros(384, device="cuda")
        want = st.forward(flipped, T_b, x_carry=xc1)
        out = torch.empty_like(want)
        xc2 = torch.zeros(384, device="cuda")
        st.forward_ptr(X.data_ptr() + 202 * X.stride(0) * 4, -X.stride(0), 203, T_b, out.data_ptr(), out.stride(0),
                       x_carry=xc2)
        torch.cuda.synchronize()
        assert out.cpu().numpy().tobytes() == want.cpu().numpy().tobytes(), (kind, mode)
        assert torch.equal(xc1, xc2)
        st.close()
