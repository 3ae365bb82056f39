"""Deterministic generation on the GPU (rnnb_splitmix_uniform;
model_io.generate_weights / generate_sequence; bench_gpu gen-weights /
gen-seq): the SplitMix64 known answers and byte-identical RNNW / RNNX files
against files the reference itself wrote (tests/golden/, make_golden.py)."""

import ctypes
import json
import os
import subprocess
import sys

import numpy as np
import pytest

from conftest import GOLDEN, REPO
from paper_1803_11389_b200 import model_io


def test_generate_sequence_argument_errors():
    with pytest.raises(ValueError):
        model_io.generate_sequence(0, 4, 1)
    with pytest.raises(ValueError):
        model_io.generate_sequence(4, 4, 1, "f16")


gpu = pytest.mark.gpu


def _raw(seed, n):
    import torch
    from paper_1803_11389_b200 import _lib
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    _lib.check(_lib.load().rnnb_splitmix_uniform(ctypes.c_uint64(seed), ctypes.c_uint64(0), n,
                                                 ctypes.c_void_p(out.data_ptr()), _lib.DT_U64, None))
    return [int(v) & 0xFFFFFFFFFFFFFFFF for v in out.cpu().numpy()]


@gpu
def test_splitmix_known_answers():
    k = json.load(open(os.path.join(GOLDEN, "splitmix.json")))
    assert _raw(0, 4) == k["seed0_first4"]
    assert _raw(0, 1)[0] == 0xE220A8397B1DCDAF  # the generator's published first value
    assert _raw(42, 8) == k["seed42_first8"]
    u = model_io._splitmix_uniform(42, 8, np.float64)
    assert u.tolist() == k["uniform_seed42_first8"]


@gpu
@pytest.mark.parametrize("name", ["sru2_f32.rnnw", "qrnn1_f64.rnnw", "lstm1_f32.rnnw"])
def test_generate_weights_matches_reference_files(tmp_path, name):
    from paper_1803_11389_b200.cells import CellKind, RnnConfig
    m = json.load(open(os.path.join(GOLDEN, "model_files.json")))[name]
    cfg = RnnConfig(CellKind.parse(m["kind"]), m["d_in"], m["d_h"], n_layers=m["n_layers"],
                    precision=m["precision"])
    out = tmp_path / name
    model_io.save_weights(model_io.generate_weights(cfg, m["seed"]), str(out))
    assert out.read_bytes() == open(os.path.join(GOLDEN, name), "rb").read()


@gpu
@pytest.mark.parametrize("name", ["seq_f32.rnnx", "seq_f64.rnnx"])
def test_generate_sequence_matches_reference_files(tmp_path, name):
    m = json.load(open(os.path.join(GOLDEN, "model_files.json")))[name]
    out = tmp_path / name
    model_io.save_sequence(model_io.generate_sequence(m["seq_len"], m["width"], m["seed"], m["precision"]), str(out))
    assert out.read_bytes() == open(os.path.join(GOLDEN, name), "rb").read()


@gpu
def test_cli_gen_commands_match_reference_files(tmp_path):
    def cli(*args):
        r = subprocess.run([sys.executable, "-m", "paper_1803_11389_b200.bench_gpu", *args], capture_output=True,
                           text=True, cwd=REPO, timeout=300)
        assert r.returncode == 0, r.stderr
    w = tmp_path / "w.rnnw"
    cli("gen-weights", "--cell", "sru", "--width", "24", "--layers", "2", "--seed", "31", "--out", str(w))
    assert w.read_bytes() == open(os.path.join(GOLDEN, "sru2_f32.rnnw"), "rb").read()
    x = tmp_path / "x.rnnx"
    cli("gen-seq", "--seq-len", "37", "--width", "24", "--seed", "34", "--out", str(x))
    assert x.read_bytes() == open(os.path.join(GOLDEN, "seq_f32.rnnx"), "rb").read()
