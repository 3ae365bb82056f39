"""RNNW / RNNX files against files written by the
reference itself (tests/golden/*.rnnw|rnnx, make_golden.py model_files):
byte-identical saves, equal loads, the reference's exception classes for
every malformed-file case (model_io.py:209-308; pkg/tests/test_model_io.py
191-270), in the Python host path and in the native C-ABI parser (which
needs no GPU)."""

import json
import os
import struct

import numpy as np
import pytest

from conftest import GOLDEN


@pytest.fixture(scope="module")
def M():
    from paper_1803_11389_b200 import model_io
    return model_io


def _index():
    with open(os.path.join(GOLDEN, "model_files.json")) as f:
        return json.load(f)


def _generated(oracle, spec):
    from paper_1803_11389_b200 import cells
    kind = cells.CellKind.parse(spec["kind"])
    dt = np.float32 if spec["precision"] == "f32" else np.float64
    layers = oracle.generate_layers(spec["kind"], spec["d_in"], spec["d_h"], spec["n_layers"], spec["seed"], dt)
    cls = {"lstm": cells.LstmWeights, "sru": cells.SruWeights, "qrnn": cells.QrnnWeights}[spec["kind"]]
    return cells.WeightSet(kind, spec["precision"], [cls(*lay) for lay in layers])


@pytest.mark.parametrize("name", ["sru2_f32.rnnw", "qrnn1_f64.rnnw", "lstm1_f32.rnnw"])
def test_weights_round_trip_byte_identical(M, oracle, tmp_path, name):
    spec = _index()[name]
    ws = _generated(oracle, spec)
    out = tmp_path / name
    M.save_weights(ws, out)
    ref = open(os.path.join(GOLDEN, name), "rb").read()
    assert out.read_bytes() == ref
    back = M.load_weights(os.path.join(GOLDEN, name))
    assert back.kind is ws.kind and back.precision == ws.precision and len(back.layers) == len(ws.layers)
    for a, b in zip(back.layers, ws.layers):
        for x, y in zip(a.mats(), b.mats()):
            assert x.dtype == y.dtype and np.array_equal(x, y)
    kind, prec, dims = M.weights_info(os.path.join(GOLDEN, name))  # native parser
    assert kind is ws.kind and prec == ws.precision
    assert dims == [(lay.d_in, lay.d_h) for lay in ws.layers]


@pytest.mark.parametrize("name", ["seq_f32.rnnx", "seq_f64.rnnx"])
def test_sequence_round_trip(M, oracle, tmp_path, name):
    spec = _index()[name]
    dt = np.float32 if spec["precision"] == "f32" else np.float64
    X = oracle.generate_sequence(spec["seq_len"], spec["width"], spec["seed"], dt)
    out = tmp_path / name
    M.save_sequence(X, out)
    assert out.read_bytes() == open(os.path.join(GOLDEN, name), "rb").read()
    Y = M.load_sequence(os.path.join(GOLDEN, name))
    assert Y.dtype == dt and np.array_equal(X, Y)
    assert M.sequence_info(os.path.join(GOLDEN, name)) == (spec["precision"], spec["seq_len"], spec["width"])


def _both(M, path, exc, weights=True):
    """Python loader and native parser raise the same reference class."""
    with pytest.raises(exc):
        (M.load_weights if weights else M.load_sequence)(path)
    with pytest.raises(exc):
        (M.weights_info if weights else M.sequence_info)(path)


def test_weight_file_errors(M, tmp_path):
    good = open(os.path.join(GOLDEN, "sru2_f32.rnnw"), "rb").read()
    p = tmp_path / "w.rnnw"
    p.write_bytes(b"XXXX" + good[4:])
    _both(M, p, M.BadMagicError)
    p.write_bytes(good[:4] + struct.pack("<I", 2) + good[8:])
    _both(M, p, M.UnsupportedVersionError)
    p.write_bytes(good[:-5])
    _both(M, p, M.TruncatedFileError)
    p.write_bytes(good[:10])
    _both(M, p, M.TruncatedFileError)
    p.write_bytes(good + b"\0")
    _both(M, p, M.ShapeConsistencyError)
    p.write_bytes(good[:8] + bytes([7]) + good[9:])
    _both(M, p, M.ShapeConsistencyError)
    # lying header: a huge d_in must fail on size before allocating
    lie = bytearray(good)
    lie[16:20] = struct.pack("<I", 1 << 30)
    lie[20:24] = struct.pack("<I", 1 << 30)
    p.write_bytes(bytes(lie))
    with pytest.raises(M.FileFormatError):
        M.load_weights(p)
    with pytest.raises(M.FileFormatError):
        M.weights_info(p)
    for exc in (M.BadMagicError, M.TruncatedFileError, M.ShapeConsistencyError, M.UnsupportedVersionError):
        assert issubclass(exc, ValueError)


def test_sequence_file_errors(M, tmp_path):
    good = open(os.path.join(GOLDEN, "seq_f32.rnnx"), "rb").read()
    p = tmp_path / "x.rnnx"
    p.write_bytes(b"RNNW" + good[4:])
    _both(M, p, M.BadMagicError, weights=False)
    p.write_bytes(good[:4] + struct.pack("<I", 9) + good[8:])
    _both(M, p, M.UnsupportedVersionError, weights=False)
    p.write_bytes(good[:-4])
    _both(M, p, M.TruncatedFileError, weights=False)
    p.write_bytes(good + b"\0\0\0\0")
    _both(M, p, M.ShapeConsistencyError, weights=False)
    p.write_bytes(good[:12] + struct.pack("<I", 0) + good[16:])
    _both(M, p, M.ShapeConsistencyError, weights=False)


def test_presets_and_param_counts():
    from paper_1803_11389_b200 import model_io as M
    from paper_1803_11389_b200.cells import CellKind
    cfg = M.preset_config("qrnn-large")
    assert (cfg.kind, cfg.d_in, cfg.d_h) == (CellKind.QRNN, 1024, 1024)
    assert M.count_params(cfg) == 6 * 1024 * 1024  # BASELINE cfg2's 6,291,456 parameters
    assert M.count_params(M.preset_config("sru-small")) == 3 * 512 * 512 + 2 * 512
    with pytest.raises(ValueError, match="unknown preset"):
        M.preset_config("gru-small")
