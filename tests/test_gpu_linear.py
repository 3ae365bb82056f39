"""Dense-layer kernels (rnnb_linear_*: the cfg3 projection and logits) vs the
oracle's gemm (kernels.py:203-225 restated in oracle/), odd sizes included:
partial tiles in every dimension, K not a multiple of the k-tile, a bias."""

import numpy as np
import pytest

from parity_util import ROUND, assert_f32, normwise

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", ["f32", "f64", "bf16", "tf32", "f32x3"])
@pytest.mark.parametrize("L,d_in,d_out", [(4096, 120, 1024), (300, 1024, 2000), (77, 40, 130), (1, 8, 3),
                                         (5003, 200, 777)])
def test_linear_matches_oracle_gemm(oracle, mode, L, d_in, d_out):
    import torch
    from paper_1803_11389_b200.device import DeviceLinear
    rng = np.random.default_rng(L + d_in + d_out)
    dt = np.float64 if mode == "f64" else np.float32
    W = rng.uniform(-1, 1, (d_out, d_in)).astype(dt) / np.sqrt(d_in)
    b = rng.standard_normal(d_out).astype(dt)
    X = rng.standard_normal((L, d_in)).astype(dt)
    lin = DeviceLinear(W, b, mode=mode)
    Y = lin.forward(torch.from_numpy(X).cuda()).cpu().numpy()
    assert Y.shape == (L, d_out)
    # fp32 dense layers take the fp32-accurate 3xTF32 tcgen05 path when their
    # (384-column, 32-row) items fill the GPU, else the FFMA GEMM
    hpad = -(-(-(-d_out // 3)) // 128) * 128
    fills = (hpad // 128) * -(-L // 32) >= torch.cuda.get_device_properties(0).multi_processor_count
    assert lin.query(0) == (1 if mode in ("bf16", "tf32") or (mode in ("f32", "f32x3") and fills) else 0)
    if mode in ("bf16", "tf32"):
        rnd = ROUND[mode]
        ref = oracle.gemm(rnd(W), np.ascontiguousarray(rnd(X).T), kernel="fast").T + b
        # exact products of rounded operands, fp32 accumulation in another
        # order: the fp32 bound (tighter than the per-layer BOUND_VS_ROUNDED)
        assert normwise(Y, ref) <= 1e-5, normwise(Y, ref)
    else:
        ref = oracle.gemm(W, np.ascontiguousarray(X.T), kernel="fast").T + b
        if mode == "f64":
            assert np.max(np.abs(Y - ref)) <= 1e-12
        else:
            assert_f32(Y, ref)
    lin.close()


def test_linear_strided_input_and_output(oracle):
    import torch
    from paper_1803_11389_b200.device import DeviceLinear
    rng = np.random.default_rng(3)
    W = rng.uniform(-0.1, 0.1, (200, 64)).astype(np.float32)
    X = rng.standard_normal((50, 64)).astype(np.float32)
    for mode in ("f32", "bf16"):
        lin = DeviceLinear(W, mode=mode)
        big = torch.zeros((50, 96), device="cuda")
        big[:, :64] = torch.from_numpy(X).cuda()
        out = torch.full((50, 256), 7.0, device="cuda")
        lin.forward(big[:, :64], out=out[:, :200])
        dense = lin.forward(torch.from_numpy(X).cuda())
        assert torch.equal(out[:, :200], dense)
        assert bool((out[:, 200:] == 7.0).all())  # nothing written past d_out
        lin.close()


def test_linear_argument_errors():
    import torch
    from paper_1803_11389_b200.device import DeviceLinear
    lin = DeviceLinear(np.ones((4, 3), np.float32))
    with pytest.raises(ValueError):
        lin.forward(torch.zeros((5, 4), device="cuda"))
    with pytest.raises(ValueError):
        lin.forward(torch.zeros((5, 3), dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError):
        DeviceLinear(np.ones((4, 3), np.float32), bias=np.ones(5))
    lin.close()
