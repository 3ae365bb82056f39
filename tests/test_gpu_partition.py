"""The partition code on the CUDA kernels (world_size 1 here: one GPU per
gpurun call; the multi-rank host logic is covered by test_partition.py on
gloo), plus cfg3 (projection + SRU stack + logits) and cfg5-shaped wide SRU."""

import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pg():
    import torch
    import torch.distributed as dist
    if not dist.is_initialized():
        s = socket.socket()
        s.bind(("127.0.0.1", 0))
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(s.getsockname()[1])
        s.close()
        torch.cuda.set_device(0)
        dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    yield dist
    dist.destroy_process_group()


def test_pipeline_stage_on_gpu_bitwise_equals_whole_sequence(pg, oracle, monkeypatch):
    import torch
    monkeypatch.setenv("RNNB_F32_TC", "0")  # f32: FFMA kernels, chunking-invariant bitwise
    import paper_1803_11389_b200 as P
    from paper_1803_11389_b200 import partition
    layers = oracle.generate_layers("qrnn", 256, 256, 4, 7, np.float32)
    X = torch.from_numpy(np.random.default_rng(2).standard_normal((1024, 256)).astype(np.float32)).cuda()
    for mode in ("f32", "bf16"):
        st = P.DeviceStack("qrnn", layers, mode=mode)
        whole = st.forward(X, 32).cpu().numpy()
        stage = partition.DeviceStage(st, 32)
        out = partition.pipeline_forward(stage, X, 1024, 256, 256, 32, 0, 1, torch.float32, X.device)
        got = out.cpu().numpy()
        if mode == "f32":
            assert got.tobytes() == whole.tobytes()
        else:  # look-back anchored at chunk edges: same math up to rounding
            assert np.max(np.abs(got - whole)) / np.max(np.abs(whole)) <= 1e-6
        st.close()


def test_sharded_bidirectional_wide_sru_on_gpu(pg):
    import torch
    import dist_helpers as H
    from paper_1803_11389_b200 import partition
    fw, bw, X = H.make_bidir(H=64, d0=64, n_layers=3, seed=5)
    X = np.random.default_rng(3).standard_normal((300, 64))
    ref = H.bidir_reference(fw, bw, X)
    for mode, tol in (("f32", 1e-5), ("bf16", 2e-2)):
        make = partition.wide_sru_stage_factory(16, mode, 0)
        model = partition.ShardedBidirSRU(fw, bw, 0, 1, make)
        got = model.forward(torch.from_numpy(X.astype(np.float32)).cuda()).cpu().numpy()
        err = np.max(np.abs(got - ref)) / np.max(np.abs(ref))
        assert err <= tol, (mode, err)


def test_acoustic_cfg3_shape_matches_oracle(oracle):
    import torch
    from paper_1803_11389_b200 import workloads
    from paper_1803_11389_b200.acoustic import AcousticSRU
    w = workloads.make("cfg3", scale=1 / 16)  # L = 256 frames
    m = AcousticSRU(w.proj, w.layers, w.logits, mode="f32")
    got = m.forward(torch.from_numpy(w.X).cuda(), 32).cpu().numpy()
    h = (w.X.astype(np.float64) @ w.proj.T.astype(np.float64)).astype(np.float32)
    h = oracle.run_blocked("sru", [lay.mats() for lay in w.layers], h, 32)
    ref = h.astype(np.float64) @ w.logits.T.astype(np.float64)
    assert got.shape == (256, 2000)
    assert np.max(np.abs(got - ref)) / np.max(np.abs(ref)) <= 1e-5
    m.close()
