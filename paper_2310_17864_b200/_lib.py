"""ctypes binding of libctcb.so (the C ABI declared in include/ctcb.h).

The library is built in-tree by ``__graft_entry__.build()`` (nvcc, sm_100a).
There is no fallback: if the library is missing or fails to load, every entry
point raises.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("CTCB_LIB") or os.path.join(_HERE, "libctcb.so")

CTCB_OK, CTCB_ERR_ARG, CTCB_ERR_CUDA, CTCB_ERR_WORKSPACE, CTCB_ERR_UNSUPPORTED = 0, 1, 2, 3, 4
UTT_OK, UTT_EMPTY, UTT_BAD_LEN, UTT_BEAM_DIED, UTT_OVERFLOW = 0, 1, 2, 3, 4
UTT_NONFINITE, UTT_ABOVE_ZERO, UTT_NOT_NORMALIZED = 5, 6, 7

# every symbol include/ctcb.h declares (checked by tests/test_abi.py)
SYMBOLS = (
    "ctcb_create", "ctcb_destroy", "ctcb_skip_cutoff", "ctcb_topk_size", "ctcb_workspace_bytes",
    "ctcb_decode", "ctcb_decode_host", "ctcb_debug_frames", "ctcb_validate", "ctcb_set_validate", "ctcb_debug_counters", "ctcb_status_string",
    "ctcb_last_error", "ctcb_kernel_timing", "ctcb_kernel_time", "ctcb_launch_count", "ctcb_decode_host_async", "ctcb_decode_host_wait",
    "ctcb_set_merge_mode", "ctcb_set_beam_size_token", "ctcb_align", "ctcb_align_workspace_bytes",
    "ctcb_lm_create", "ctcb_lm_destroy", "ctcb_set_lm", "ctcb_set_silence", "ctcb_decode_lm",
)

_lib = None


class CtcbError(RuntimeError):
    """CUDA-side failure of the ctcb library."""


def build(force: bool = False) -> str:
    csrc = os.path.join(_HERE, "csrc")
    cmd = ["make", "-s", "-C", csrc]
    if force:
        cmd.insert(1, "-B")
    subprocess.run(cmd, check=True)
    return LIB_PATH


def load():
    """Load libctcb.so once and declare argument types."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise CtcbError(
            f"{LIB_PATH} is missing: the ctcb CUDA extension has not been built "
            "(run `python -c 'import __graft_entry__ as g; g.build()'`). There is no CPU fallback."
        )
    lib = ctypes.CDLL(LIB_PATH)
    c_int, c_int64, c_double, c_float, c_size_t, vp = (
        ctypes.c_int, ctypes.c_int64, ctypes.c_double, ctypes.c_float, ctypes.c_size_t, ctypes.c_void_p)
    lib.ctcb_create.argtypes = [c_int, c_int, c_int, c_int, c_float, c_double, c_int, ctypes.POINTER(vp)]
    lib.ctcb_destroy.argtypes = [vp]
    lib.ctcb_skip_cutoff.argtypes = [c_double, ctypes.POINTER(c_float)]
    lib.ctcb_topk_size.argtypes = [vp, ctypes.POINTER(c_int)]
    lib.ctcb_workspace_bytes.argtypes = [vp, c_int, c_int, ctypes.POINTER(c_size_t)]
    lib.ctcb_decode.argtypes = [vp, vp, c_int64, c_int64, vp, c_int, c_int, vp, c_size_t, vp,
                                vp, vp, vp, vp, vp, vp]
    lib.ctcb_decode_host.argtypes = [vp, vp, c_int64, c_int64, vp, c_int, c_int, vp, vp, vp, vp, vp, vp, vp]
    lib.ctcb_debug_frames.argtypes = [vp, vp, c_int64, c_int64, vp, c_int, c_int, vp, vp, vp, vp, vp, vp]
    lib.ctcb_validate.argtypes = [vp, vp, c_int64, c_int64, vp, c_int, c_int, c_int, vp, vp]
    lib.ctcb_set_validate.argtypes = [vp, c_int]
    lib.ctcb_debug_counters.argtypes = [vp, ctypes.POINTER(ctypes.c_uint64)]
    lib.ctcb_decode_host_async.argtypes = [vp, vp, c_int64, c_int64, vp, c_int, c_int, c_int, vp, vp, vp, vp, vp, vp,
                                           vp, ctypes.POINTER(c_int)]
    lib.ctcb_decode_host_wait.argtypes = [vp, c_int, ctypes.POINTER(c_int), ctypes.POINTER(c_int)]
    lib.ctcb_kernel_timing.argtypes = [vp, c_int]
    lib.ctcb_set_merge_mode.argtypes = [vp, c_int]
    lib.ctcb_align_workspace_bytes.argtypes = [c_int, c_int, c_int, ctypes.POINTER(c_size_t)]
    lib.ctcb_align.argtypes = [vp, c_int64, c_int64, vp, vp, vp, c_int, c_int, c_int, c_int, c_int, vp, c_size_t, vp,
                               vp, vp, vp, vp, vp]
    lib.ctcb_set_beam_size_token.argtypes = [vp, c_int]
    lib.ctcb_lm_create.argtypes = [c_int, c_int64, vp, vp, vp, vp, vp, c_int, c_int, c_int, ctypes.POINTER(vp)]
    lib.ctcb_lm_destroy.argtypes = [vp]
    lib.ctcb_set_lm.argtypes = [vp, vp, vp, c_double]
    lib.ctcb_set_silence.argtypes = [vp, c_int, c_double]
    lib.ctcb_decode_lm.argtypes = [vp, vp, c_int64, c_int64, vp, c_int, c_int, vp, c_size_t, vp,
                                   vp, vp, vp, vp, vp, vp, vp]
    lib.ctcb_launch_count.argtypes = [vp, ctypes.POINTER(ctypes.c_uint64)]
    lib.ctcb_kernel_time.argtypes = [vp, ctypes.POINTER(c_double), ctypes.POINTER(c_int), ctypes.POINTER(ctypes.c_char_p)]
    lib.ctcb_status_string.argtypes = [c_int]
    lib.ctcb_status_string.restype = ctypes.c_char_p
    lib.ctcb_last_error.argtypes = []
    lib.ctcb_last_error.restype = ctypes.c_char_p
    for name in SYMBOLS:
        if name not in ("ctcb_status_string", "ctcb_last_error"):
            getattr(lib, name).restype = c_int
    _lib = lib
    return lib


def check(rc: int, what: str) -> None:
    """Map a ctcb status to the Python exception the reference would raise."""
    if rc == CTCB_OK:
        return
    lib = load()
    msg = lib.ctcb_last_error().decode()
    if rc in (CTCB_ERR_ARG, CTCB_ERR_UNSUPPORTED, CTCB_ERR_WORKSPACE):
        raise ValueError(msg or lib.ctcb_status_string(rc).decode())
    raise CtcbError(f"{what}: {msg}")
