"""Multi-GPU partition host logic, covered on CPU with world_size-2 gloo
process groups and the oracle as the per-rank compute."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import dist_helpers as H
from paper_1803_11389_b200 import partition


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_partition_arithmetic():
    assert partition.layer_ranges(8, 1) == [(0, 8)]
    assert partition.layer_ranges(8, 4) == [(0, 2), (2, 4), (4, 6), (6, 8)]
    assert partition.layer_ranges(7, 3) == [(0, 3), (3, 5), (5, 7)]
    with pytest.raises(ValueError):
        partition.layer_ranges(2, 4)
    assert partition.unit_range(4096, 8, 3) == (1536, 2048)
    with pytest.raises(ValueError):
        partition.unit_range(100, 8, 0)
    assert partition.chunk_plan(100, 32, 16) == [(0, 32), (32, 32), (64, 32), (96, 4)]
    with pytest.raises(ValueError):
        partition.chunk_plan(100, 30, 16)


def test_layer_pipeline_two_ranks_bitwise_equals_single_process(tmp_path, oracle):
    out = str(tmp_path / "pipe.npy")
    mp.spawn(H.pipeline_worker, args=(2, _port(), out), nprocs=2, join=True)
    got = np.load(out)
    layers = oracle.generate_layers("qrnn", 32, 32, 4, 5, np.float32)
    X = np.random.default_rng(1).standard_normal((256, 32)).astype(np.float32)
    ref = oracle.run_blocked("qrnn", layers, X, 16)
    assert got.tobytes() == ref.tobytes()


def test_hidden_sharding_two_ranks_matches_unsharded(tmp_path):
    out = str(tmp_path / "shard.npy")
    mp.spawn(H.sharding_worker, args=(2, _port(), out), nprocs=2, join=True)
    got = np.load(out)
    fw, bw, X = H.make_bidir()
    ref = H.bidir_reference(fw, bw, X)
    assert got.shape == (40, 32)
    assert np.max(np.abs(got - ref)) <= 1e-12
