"""paper_1803_11389_b200.kernels: the drop-in for rnnblock kernels.py.

CPU part: the argument checks (same ValueError conditions as
kernels.py:34-47, 181-233, 312-322) fire before any device work.  GPU part
(`-m gpu`): the reference's kernel-level properties -- strict kernels are
bitwise the ascending-order chain (checked against the oracle's C
restatement and a scalar loop), fast/tiled within the reference's
tolerances, activation known answers, symmetry and dtype preservation."""

import math

import numpy as np
import pytest

from paper_1803_11389_b200 import kernels as K

F32, F64 = np.float32, np.float64


def rnd(shape, dtype, seed):
    return np.random.default_rng(seed).uniform(-1.0, 1.0, shape).astype(dtype)


@pytest.mark.parametrize("call", [
    lambda: K.gemv(np.ones((2, 3), F32), np.ones(2, F32)),                 # dimension mismatch
    lambda: K.gemv(np.ones((2, 2), F32), np.ones(2, F64)),                 # dtype mismatch
    lambda: K.gemv(np.ones((2, 2), F32), np.ones(2, F32), kernel="tiled"),  # gemv has no tiled kernel
    lambda: K.gemv(np.ones(4, F32), np.ones(4, F32)),                      # A not 2-d
    lambda: K.gemv(np.ones((2, 2), F32), np.ones((2, 1), F32)),            # x not 1-d
    lambda: K.gemv(np.ones((2, 0), F32), np.ones(0, F32)),                 # empty
    lambda: K.gemm(np.ones((2, 3), F32), np.ones((2, 3), F32)),            # dimension mismatch
    lambda: K.gemm(np.ones((2, 2), F32), np.ones((2, 2), F32), kernel="blas"),
    lambda: K.gemm(np.ones((2, 2), F32), np.ones((2, 2), F32), kernel="tiled", tile=(0, 4)),
    lambda: K.gemm(np.ones((4, 4), F32)[:, ::2], np.ones((2, 2), F32)),    # not C-contiguous
    lambda: K.set_compute_threads(0),
])
def test_argument_errors_match_reference(call):
    with pytest.raises(ValueError):
        call()


def test_dtype_mismatch_message():
    with pytest.raises(ValueError, match="dtype mismatch: float32 vs float64"):
        K.gemm(np.ones((2, 2), F32), np.ones((2, 2), F64))


def test_thread_control_round_trip():
    assert K.set_compute_threads(3) == 3
    assert K.get_compute_threads() == 3
    assert K.KERNELS == ("reference", "tiled", "fast")


gpu = pytest.mark.gpu


@gpu
@pytest.mark.parametrize("dtype", [F32, F64])
def test_gemm_strict_is_the_ascending_chain(oracle, dtype):
    for seed, (m, k, n) in enumerate([(1, 1, 1), (2, 5, 3), (33, 9, 65), (64, 63, 64), (128, 17, 256),
                                      (70, 1000, 40)]):
        A, B = rnd((m, k), dtype, seed), rnd((k, n), dtype, 100 + seed)
        ref = oracle.gemm(A, B, "reference")
        for kern in ("reference", "tiled"):
            assert K.gemm(A, B, kernel=kern).tobytes() == ref.tobytes(), (m, k, n, kern)
        tol = 5e-5 if dtype == F32 else 5e-12
        assert np.max(np.abs(K.gemm(A, B, kernel="fast") - ref)) <= tol


@gpu
def test_gemv_scalar_ascending_loop_and_gemm_column():
    A, x = rnd((13, 29), F32, 5), rnd(29, F32, 6)
    got = K.gemv(A, x)
    for i in range(13):
        acc = np.float32(0.0)
        for j in range(29):
            acc = np.float32(acc + np.float32(A[i, j] * x[j]))
        assert got[i] == acc
    B = rnd((31, 17), F32, 2)
    v = rnd(17, F32, 3)
    assert (K.gemm(B, v.reshape(-1, 1))[:, 0] == K.gemv(B, v)).all()
    assert K.gemv(np.eye(2, dtype=F64), np.array([3.0, -1.0])).tolist() == [3.0, -1.0]
    assert K.gemm(np.array([[1.0, 2.0], [3.0, 4.0]]), np.array([[0.0, 1.0], [1.0, 0.0]])).tolist() == \
        [[2.0, 1.0], [4.0, 3.0]]
    for seed, (m, k) in enumerate([(1, 1), (3, 17), (127, 255), (256, 256)]):
        M, y = rnd((m, k), F64, seed), rnd(k, F64, 50 + seed)
        assert np.max(np.abs(K.gemv(M, y, kernel="fast") - K.gemv(M, y))) <= 1e-12


@gpu
def test_activation_known_answers():
    assert K.sigmoid(0.0) == 0.5
    assert K.sigmoid(1000.0) == 1.0 and K.sigmoid(-1000.0) == 0.0
    assert abs(K.sigmoid(1.0) - 1.0 / (1.0 + math.exp(-1.0))) < 1e-15
    assert K.tanh_act(0.0) == 0.0
    assert abs(K.tanh_act(1.0) - math.tanh(1.0)) < 1e-15
    xs = np.random.default_rng(11).uniform(-50.0, 50.0, 500)
    assert np.max(np.abs(K.sigmoid(xs) + K.sigmoid(-xs) - 1.0)) <= np.finfo(F64).eps
    ts = np.random.default_rng(12).uniform(-20, 20, 200)
    assert (K.tanh_act(-ts) == -K.tanh_act(ts)).all()
    assert np.all(np.abs(K.tanh_act(ts)) <= 1.0)
    x32 = np.linspace(-8, 8, 1001, dtype=F32)
    assert K.sigmoid(x32).dtype == F32 and K.tanh_act(x32).dtype == F32
    assert np.max(np.abs(K.sigmoid(x32) - (0.5 * (1.0 + np.tanh(0.5 * x32))))) <= 2.4e-7
    assert np.max(np.abs(K.tanh_act(x32.reshape(7, 143)) - np.tanh(x32.reshape(7, 143)))) <= 2.4e-7
