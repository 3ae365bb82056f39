"""The C-ABI library loads and exports every symbol include/rnnb.h
declares; argument validation works without a GPU (no compute calls)."""

import ctypes
import os
import re

import pytest

from conftest import REPO
from paper_1803_11389_b200 import _lib


def _header_symbols():
    with open(os.path.join(REPO, "include", "rnnb.h")) as f:
        text = f.read()
    return sorted(set(re.findall(r"\b(rnnb_[a-z_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert sorted(_lib.SYMBOLS) == _header_symbols()


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in _header_symbols():
        assert hasattr(lib, name), name
    assert lib.rnnb_version().decode().startswith("rnnb-b200")


def test_plan_blocks_abi():
    lib = _lib.load()
    n, last = ctypes.c_int64(), ctypes.c_int64()
    assert lib.rnnb_plan_blocks(100, 32, ctypes.byref(n), ctypes.byref(last)) == _lib.OK
    assert (n.value, last.value) == (4, 4)
    assert lib.rnnb_plan_blocks(0, 4, None, None) == _lib.EINVAL
    assert b"seq_len" in lib.rnnb_last_error()
    assert lib.rnnb_plan_blocks(4, 0, None, None) == _lib.EINVAL


def test_create_rejects_bad_arguments_before_touching_cuda():
    lib = _lib.load()
    h = ctypes.c_void_p()
    one = (ctypes.c_int64 * 1)
    # LSTM is not a blocked kind (blocked.py:231-233)
    assert lib.rnnb_stack_create(ctypes.byref(h), 0, 1, one(8), one(8), 0, 0) == _lib.EINVAL
    assert b"SRU and QRNN" in lib.rnnb_last_error()
    # SRU needs d_in == d_h (cells.py:89)
    assert lib.rnnb_stack_create(ctypes.byref(h), _lib.SRU, 1, one(8), one(9), 0, 0) == _lib.EINVAL
    # stacked widths must chain
    two = (ctypes.c_int64 * 2)
    assert lib.rnnb_stack_create(ctypes.byref(h), _lib.QRNN, 2, two(8, 7), two(9, 9), 0, 0) == _lib.EINVAL
    assert lib.rnnb_stack_create(ctypes.byref(h), _lib.QRNN, 1, one(8), one(8), 9, 0) == _lib.EINVAL
    assert lib.rnnb_sweep(None, None, None, None, 1, 1, 0, None) == _lib.EINVAL
    assert lib.rnnb_finalize(_lib.SRU, ctypes.c_void_p(1), ctypes.c_void_p(1), None, ctypes.c_void_p(1),
                             1, 1, 0, None) == _lib.EINVAL


def test_status_mapping():
    with pytest.raises(ValueError):
        _lib.check(_lib.EINVAL)
    with pytest.raises(RuntimeError):
        _lib.check(_lib.ECUDA)
