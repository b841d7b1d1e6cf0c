"""The C-ABI library loads on a CPU-only host and exports every entry point
declared in include/flame_b200.h; argument validation runs before any device
work (status 1 -> ValueError)."""

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

import paper_2509_22681_b200 as fb
from paper_2509_22681_b200 import _lib

HEADER = Path(__file__).resolve().parent.parent / "include" / "flame_b200.h"


def declared_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(flame_[a-z0-9_]+)\s*\(", text)))


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    names = declared_functions()
    assert len(names) >= 14
    for name in names:
        assert hasattr(lib, name), name
    assert set(names) == set(_lib.EXPORTED)


def test_bad_descriptor_rejected_without_device():
    lib = _lib.load()
    desc = _lib.FlameModelDesc(16, 3, 2, 1, 24, 3, 64, 32, 0)  # head_dim does not divide
    out = ctypes.c_void_p()
    w = np.zeros(4)
    rc = lib.flame_create(ctypes.byref(desc), w.ctypes.data, 4, 0, 0, ctypes.byref(out))
    assert rc == 1
    assert b"head_dim" in lib.flame_last_error()
    with pytest.raises(ValueError):
        _lib.check(rc)


def test_bad_flmp_rejected_without_device():
    lib = _lib.load()
    out = ctypes.c_void_p()
    junk = b"NOPE" + b"\0" * 60
    assert lib.flame_create_flmp(junk, len(junk), 0, 0, ctypes.byref(out)) == 1
    assert b"magic" in lib.flame_last_error()


def test_list_capacity():
    assert _lib.load().flame_exec_list_capacity(8, 256, 512) == 2048
    assert _lib.load().flame_exec_list_capacity(4, 16, 512) == 512


def test_no_cpu_fallback_without_gpu(monkeypatch):
    import torch

    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    cfg = fb.ModelConfig(16, 4, 2, 1, 24, 3, 64, 32)
    with pytest.raises(RuntimeError):
        fb.model_forward(np.zeros((8, 16)), np.zeros((2, 16)), fb.init_params(cfg), cfg)


def test_sm100a_code_in_library():
    """The shipped .so carries sm_100a SASS with tcgen05 MMAs and TMA loads."""
    import shutil
    import subprocess

    if shutil.which("cuobjdump") is None:
        pytest.skip("cuobjdump not available")
    sass = subprocess.run(["cuobjdump", "-sass", str(_lib.LIB_PATH)], capture_output=True,
                          text=True, check=True).stdout
    assert "sm_100a" in sass
    assert "UTCHMMA" in sass and "UTMALDG" in sass and "LDTM" in sass


def test_pack_padded_host_staging():
    """flame_pack_padded (host-only): ragged records into fixed-stride slots,
    empty records skipped, an oversize record rejected (status 1)."""
    lib = _lib.load()
    recs = [np.arange(5, dtype=np.int64), np.zeros(0, dtype=np.int64), np.arange(100, 108, dtype=np.int64)]
    lens = np.array([len(r) for r in recs], dtype=np.int64)
    flat = np.concatenate(recs)
    dst = np.full((3, 8), -1, dtype=np.int64)
    assert lib.flame_pack_padded(dst.ctypes.data, 64, flat.ctypes.data, lens.ctypes.data, 3, 8) == 0
    np.testing.assert_array_equal(dst[0, :5], recs[0])
    assert (dst[0, 5:] == -1).all() and (dst[1] == -1).all()
    np.testing.assert_array_equal(dst[2], recs[2])
    rows = np.random.default_rng(0).standard_normal((6, 4)).astype(np.float32)
    out = np.zeros((2, 5, 4), dtype=np.float32)
    rl = np.array([2, 4], dtype=np.int64)
    assert lib.flame_pack_padded(out.ctypes.data, 80, rows.ctypes.data, rl.ctypes.data, 2, 16) == 0
    np.testing.assert_array_equal(out[0, :2], rows[:2])
    np.testing.assert_array_equal(out[1, :4], rows[2:])
    big = np.array([9], dtype=np.int64)
    assert lib.flame_pack_padded(dst.ctypes.data, 64, np.zeros(9, np.int64).ctypes.data, big.ctypes.data, 1, 8) == 1
