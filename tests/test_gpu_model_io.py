"""RNNW / RNNX straight to the device (rnnb_stack_load_rnnw,
rnnb_lstm_load_rnnw, rnnb_rnnx_load): bitwise the same results as the
array upload path, on reference-written files."""

import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


def test_stack_from_rnnw_matches_array_upload():
    import torch
    import paper_1803_11389_b200 as P
    from paper_1803_11389_b200 import model_io as M
    for name in ("sru2_f32.rnnw", "qrnn1_f64.rnnw"):
        path = os.path.join(GOLDEN, name)
        ws = M.load_weights(path)
        a = M.load_weights_device(path)
        b = P.DeviceStack(ws.kind, ws.layers, mode=ws.precision)
        dt = np.float32 if ws.precision == "f32" else np.float64
        X = torch.from_numpy(np.random.default_rng(1).standard_normal((45, ws.layers[0].d_in)).astype(dt)).cuda()
        for T in (1, 8, 45):
            assert a.forward(X, T).cpu().numpy().tobytes() == b.forward(X, T).cpu().numpy().tobytes()
        a.close()
        b.close()


def test_lstm_from_rnnw_matches_array_upload():
    import torch
    import paper_1803_11389_b200 as P
    from paper_1803_11389_b200 import model_io as M
    path = os.path.join(GOLDEN, "lstm1_f32.rnnw")
    ws = M.load_weights(path)
    a = M.load_weights_device(path)
    b = P.DeviceLstm(ws.layers[0])
    X = torch.from_numpy(np.random.default_rng(2).standard_normal((33, 10)).astype(np.float32)).cuda()
    assert a.forward(X, 4).cpu().numpy().tobytes() == b.forward(X, 4).cpu().numpy().tobytes()
    a.close()
    b.close()


@pytest.mark.parametrize("name", ["seq_f32.rnnx", "seq_f64.rnnx"])
def test_sequence_to_device(name):
    import torch
    from paper_1803_11389_b200 import model_io as M
    path = os.path.join(GOLDEN, name)
    host = M.load_sequence(path)
    dev = M.load_sequence_device(path)
    assert dev.is_cuda and np.array_equal(dev.cpu().numpy(), host)
    dev32 = M.load_sequence_device(path, dtype=torch.float32)
    assert np.array_equal(dev32.cpu().numpy(), host.astype(np.float32))
