"""CPU-side checks of the drop-in boundary: libctcb.so loads and exports
every symbol include/ctcb.h declares; the host-side cutoff reproduces the
reference's blank-skip rule; argument validation happens before any CUDA call."""

import ctypes
import math
import os
import re

import numpy as np
import pytest

from paper_2310_17864_b200 import _lib, skip_cutoff

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "ctcb.h")).read()
    return sorted(set(re.findall(r"\b(ctcb_[a-z_]+)\s*\(", text)))


def test_header_matches_binding_list():
    assert declared_symbols() == sorted(_lib.SYMBOLS)


def test_library_exports_every_symbol():
    lib = _lib.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.ctcb_status_string(0) == b"ok"


def test_create_without_gpu_fails_cleanly():
    lib = _lib.load()
    h = ctypes.c_void_p()
    rc = lib.ctcb_create(32, 0, 10, 1, ctypes.c_float(-0.05), 50.0, 0, ctypes.byref(h))
    # no GPU here: a CUDA error, never a crash; with a GPU: OK
    assert rc in (_lib.CTCB_OK, _lib.CTCB_ERR_CUDA, _lib.CTCB_ERR_ARG)
    if rc == _lib.CTCB_OK:
        lib.ctcb_destroy(h)
    rc = lib.ctcb_create(32, 0, 0, 1, ctypes.c_float(0.0), 50.0, 0, ctypes.byref(h))
    assert rc == _lib.CTCB_ERR_ARG and b"beam_size" in lib.ctcb_last_error()


def reference_drop(x32, thr):
    # emissions.py:300-301 on the float64 upcast of an fp32 value
    return bool(np.exp(np.array([x32], dtype=np.float32).astype(np.float64))[0] >= thr - 1e-12)


@pytest.mark.parametrize("thr", [0.95, 0.9, 0.6, 0.5, 0.99, 0.999999, 1e-6])
def test_skip_cutoff_is_exact(thr):
    c = np.float32(skip_cutoff(thr))
    x = c
    for _ in range(2000):  # the 2000 fp32 values above the cutoff are dropped
        assert reference_drop(x, thr)
        x = np.nextafter(x, np.float32(np.inf))
    x = np.nextafter(c, np.float32(-np.inf))
    for _ in range(2000):  # and the 2000 below are kept
        assert not reference_drop(x, thr)
        x = np.nextafter(x, np.float32(-np.inf))


def test_skip_cutoff_known_values():
    # c(0.95) = 0xbd5218ea, one ulp above float32(log(0.95)); c(0.9) = 0xbdd7c741
    assert np.float32(skip_cutoff(0.95)).view(np.uint32) == 0xBD5218EA
    assert np.float32(skip_cutoff(0.9)).view(np.uint32) == 0xBDD7C741
    assert skip_cutoff(1.0) == math.inf
    with pytest.raises(ValueError):
        skip_cutoff(0.0)
    with pytest.raises(ValueError):
        skip_cutoff(1.5)


def test_c_cutoff_matches_python():
    lib = _lib.load()
    for thr in (0.95, 0.9, 0.5, 1.0):
        c = ctypes.c_float()
        assert lib.ctcb_skip_cutoff(thr, ctypes.byref(c)) == 0
        assert c.value == np.float32(skip_cutoff(thr))
