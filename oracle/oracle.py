"""ctypes front-end for the C oracle (test infrastructure only; see __init__)."""

from __future__ import annotations

import ctypes
import math
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

OK, ERR_EMPTY, ERR_ARG, ERR_TOKEN_K, ERR_BEAM_DIED = 0, 1, 2, 3, 4


class OracleError(ValueError):
    pass


class _Opts(ctypes.Structure):
    _fields_ = [
        ("beam", ctypes.c_int64),
        ("beam_size_token", ctypes.c_int64),
        ("n_best", ctypes.c_int64),
        ("blank", ctypes.c_int64),
        ("merge_max", ctypes.c_int32),
        ("beam_threshold", ctypes.c_double),
        ("skip_threshold", ctypes.c_double),
    ]


class _LM(ctypes.Structure):
    _fields_ = [
        ("order", ctypes.c_int32),
        ("n", ctypes.c_int64),
        ("words", ctypes.POINTER(ctypes.c_int32)),
        ("lengths", ctypes.POINTER(ctypes.c_int32)),
        ("logprob", ctypes.POINTER(ctypes.c_double)),
        ("backoff", ctypes.POINTER(ctypes.c_double)),
        ("start", ctypes.POINTER(ctypes.c_int32)),
        ("start_len", ctypes.c_int32),
        ("eos", ctypes.c_int32),
    ]


class _Fusion(ctypes.Structure):
    _fields_ = [
        ("lm_score", ctypes.POINTER(ctypes.c_double)),
        ("lm_next", ctypes.POINTER(ctypes.c_int32)),
        ("lm_fin", ctypes.POINTER(ctypes.c_double)),
        ("lm_start", ctypes.c_int32),
        ("lm_weight", ctypes.c_double),
        ("sil", ctypes.c_int64),
        ("sil_score", ctypes.c_double),
    ]


@dataclass
class LMTables:
    """Dense (context x token) fusion tables (ctc_lm.c; decoder.py:178-259)."""

    score: np.ndarray   # float64 [S, V]
    next: np.ndarray    # int32 [S, V]
    fin: np.ndarray     # float64 [S]
    start: int


def lm_tables(flat, token_word) -> LMTables:
    """Tables for a flattened model (paper_2310_17864_b200.lm.flatten) and a
    per-token word map (paper_2310_17864_b200.lm.token_words)."""
    tw = np.ascontiguousarray(token_word, dtype=np.int32)
    words = np.ascontiguousarray(flat.words, dtype=np.int32)
    lens = np.ascontiguousarray(flat.lengths, dtype=np.int32)
    lp = np.ascontiguousarray(flat.logprob, dtype=np.float64)
    bo = np.ascontiguousarray(flat.backoff, dtype=np.float64)
    st = np.ascontiguousarray(flat.start, dtype=np.int32)
    m = _LM(flat.order, len(lens), _ptr(words, ctypes.c_int32), _ptr(lens, ctypes.c_int32),
            _ptr(lp, ctypes.c_double), _ptr(bo, ctypes.c_double), _ptr(st, ctypes.c_int32), flat.start_len, flat.eos)
    ps, pn, pf = ctypes.POINTER(ctypes.c_double)(), ctypes.POINTER(ctypes.c_int32)(), ctypes.POINTER(ctypes.c_double)()
    S = ctypes.c_int64()
    start = ctypes.c_int32()
    rc = _lib().ctco_lm_tables(ctypes.byref(m), _ptr(tw, ctypes.c_int32), len(tw), ctypes.byref(ps),
                               ctypes.byref(pn), ctypes.byref(pf), ctypes.byref(S), ctypes.byref(start))
    if rc != OK:
        raise OracleError("LM too large for the oracle's exact tuple keys")
    V = len(tw)
    n = S.value
    out = LMTables(np.ctypeslib.as_array(ps, shape=(n * V,)).reshape(n, V).copy(),
                   np.ctypeslib.as_array(pn, shape=(n * V,)).reshape(n, V).copy(),
                   np.ctypeslib.as_array(pf, shape=(n,)).copy(), start.value)
    _lib().ctco_lm_free(ps, pn, pf)
    return out


def lib_path() -> str:
    return os.path.join(_HERE, "build", "libctc_oracle.so")


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (oracle/Makefile)."""
    path = lib_path()
    src = os.path.join(_HERE, "ctc_oracle.c")
    srcs = [src, os.path.join(_HERE, "ctc_align.c"), os.path.join(_HERE, "ctc_lm.c")]
    if force or not os.path.exists(path) or os.path.getmtime(path) < max(os.path.getmtime(x) for x in srcs):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return path


def _lib():
    global _LIB
    if _LIB is None:
        path = lib_path()
        if not os.path.exists(path):
            build()
        lib = ctypes.CDLL(path)
        p = ctypes.POINTER
        lib.ctco_decode.argtypes = [
            p(ctypes.c_double), ctypes.c_int64, ctypes.c_int64, p(_Opts),
            p(ctypes.c_int32), p(ctypes.c_int32), p(ctypes.c_int32), p(ctypes.c_int32),
            p(ctypes.c_double), p(ctypes.c_int32), p(ctypes.c_int64), p(ctypes.c_int64),
        ]
        lib.ctco_decode.restype = ctypes.c_int
        lib.ctco_blank_keep.argtypes = [
            p(ctypes.c_double), ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
            ctypes.c_double, p(ctypes.c_int32), p(ctypes.c_int64),
        ]
        lib.ctco_blank_keep.restype = ctypes.c_int
        lib.ctco_align.argtypes = [p(ctypes.c_double), ctypes.c_int64, ctypes.c_int64, ctypes.c_int64,
                                   p(ctypes.c_int32), ctypes.c_int64, p(ctypes.c_int32)]
        lib.ctco_align.restype = ctypes.c_int
        lib.ctco_decode_fused.argtypes = [
            p(ctypes.c_double), ctypes.c_int64, ctypes.c_int64, p(_Opts), p(_Fusion),
            p(ctypes.c_int32), p(ctypes.c_int32), p(ctypes.c_int32), p(ctypes.c_int32),
            p(ctypes.c_double), p(ctypes.c_double), p(ctypes.c_int32), p(ctypes.c_int64), p(ctypes.c_int64),
        ]
        lib.ctco_decode_fused.restype = ctypes.c_int
        lib.ctco_lm_tables.argtypes = [p(_LM), p(ctypes.c_int32), ctypes.c_int64, p(p(ctypes.c_double)),
                                       p(p(ctypes.c_int32)), p(p(ctypes.c_double)), p(ctypes.c_int64),
                                       p(ctypes.c_int32)]
        lib.ctco_lm_tables.restype = ctypes.c_int
        lib.ctco_lm_free.argtypes = [p(ctypes.c_double), p(ctypes.c_int32), p(ctypes.c_double)]
        lib.ctco_lm_free.restype = None
        _LIB = lib
    return _LIB


@dataclass
class OracleResult:
    """n-best of one utterance: like ctcforge's NBestList (decoder.py:69-99)."""

    tokens: list = field(default_factory=list)      # list[list[int]]
    scores: list = field(default_factory=list)      # list[float]
    timesteps: list = field(default_factory=list)   # list[list[int]]
    lm_scores: list = field(default_factory=list)   # list[float] (fusion only)
    frame_map: np.ndarray | None = None             # kept original frames

    def __len__(self):
        return len(self.tokens)


def _ptr(a, t):
    return a.ctypes.data_as(ctypes.POINTER(t))


def blank_keep(lp: np.ndarray, threshold: float, blank: int = 0) -> np.ndarray:
    """Kept-frame indices of blank_collapse (emissions.py:284-306)."""
    lp = np.ascontiguousarray(lp, dtype=np.float64)
    t, v = lp.shape
    fm = np.zeros(max(t, 1), dtype=np.int32)
    n = ctypes.c_int64(0)
    rc = _lib().ctco_blank_keep(_ptr(lp, ctypes.c_double), t, v, blank, float(threshold),
                                _ptr(fm, ctypes.c_int32), ctypes.byref(n))
    if rc != OK:
        raise OracleError(f"threshold must be in (0, 1], got {threshold}")
    return fm[: n.value].copy()


def decode(lp: np.ndarray, beam_size: int = 10, n_best: int = 1, blank_skip_threshold: float = 1.0,
           beam_threshold: float = 50.0, beam_size_token: int | None = None,
           merge_mode: str = "logadd", blank: int = 0, lm: LMTables | None = None, lm_weight: float = 0.0,
           sil: int | None = None, sil_score: float = 0.0) -> OracleResult:
    """Decode one utterance ``lp`` [T, V] (float32 is upcast exactly to float64,
    as EmissionMatrix does at emissions.py:129)."""
    lp = np.ascontiguousarray(lp, dtype=np.float64)
    if lp.ndim != 2:
        raise OracleError(f"log_probs must be 2-D, got shape {lp.shape}")
    t, v = lp.shape
    opts = _Opts(beam_size, 0 if beam_size_token is None else beam_size_token, n_best, blank,
                 1 if merge_mode == "max" else 0,
                 float(beam_threshold), float(blank_skip_threshold))
    cnt = ctypes.c_int32(0)
    nk = ctypes.c_int64(0)
    ef = ctypes.c_int64(-1)
    tmax = max(t, 1)
    out_len = np.zeros(max(n_best, 1), dtype=np.int32)
    out_tok = np.zeros((max(n_best, 1), tmax), dtype=np.int32)
    out_ts = np.zeros((max(n_best, 1), tmax), dtype=np.int32)
    out_sc = np.zeros(max(n_best, 1), dtype=np.float64)
    fm = np.zeros(tmax, dtype=np.int32)
    out_lm = np.zeros(max(n_best, 1), dtype=np.float64)
    if lm is None and sil is None:
        rc = _lib().ctco_decode(_ptr(lp, ctypes.c_double), t, v, ctypes.byref(opts), ctypes.byref(cnt),
                                _ptr(out_len, ctypes.c_int32), _ptr(out_tok, ctypes.c_int32),
                                _ptr(out_ts, ctypes.c_int32), _ptr(out_sc, ctypes.c_double),
                                _ptr(fm, ctypes.c_int32), ctypes.byref(nk), ctypes.byref(ef))
    else:
        fu = _Fusion(None, None, None, 0, float(lm_weight), -1 if sil is None else int(sil), float(sil_score))
        if lm is not None:
            fu.lm_score = _ptr(lm.score, ctypes.c_double)
            fu.lm_next = _ptr(lm.next, ctypes.c_int32)
            fu.lm_fin = _ptr(lm.fin, ctypes.c_double)
            fu.lm_start = lm.start
        rc = _lib().ctco_decode_fused(_ptr(lp, ctypes.c_double), t, v, ctypes.byref(opts), ctypes.byref(fu),
                                      ctypes.byref(cnt), _ptr(out_len, ctypes.c_int32),
                                      _ptr(out_tok, ctypes.c_int32), _ptr(out_ts, ctypes.c_int32),
                                      _ptr(out_sc, ctypes.c_double), _ptr(out_lm, ctypes.c_double),
                                      _ptr(fm, ctypes.c_int32), ctypes.byref(nk), ctypes.byref(ef))
    if rc == ERR_EMPTY:
        raise OracleError("empty emissions")
    if rc == ERR_ARG:
        raise OracleError("invalid decoder options")
    if rc == ERR_TOKEN_K:
        raise OracleError(f"beam_size_token {beam_size_token} exceeds vocabulary size {v}")
    if rc == ERR_BEAM_DIED:
        raise OracleError(f"beam died at frame {ef.value}: no extension survives "
                          f"(beam_size_token={beam_size_token if beam_size_token else v} may be too small)")
    res = OracleResult(frame_map=fm[: nk.value].copy())
    for r in range(cnt.value):
        n = int(out_len[r])
        res.tokens.append(out_tok[r, :n].tolist())
        res.timesteps.append(out_ts[r, :n].tolist())
        res.scores.append(float(out_sc[r]))
        res.lm_scores.append(float(out_lm[r]))
    return res


def decode_batch(log_probs: np.ndarray, lens, threads: int | None = None, **kw) -> list[OracleResult]:
    """Decode utterances ``log_probs[b, :lens[b]]`` on ``threads`` host threads
    (the C call releases the GIL).  Errors carry the utterance index, as
    decode_batch does at decoder.py:156-157."""
    threads = threads or os.cpu_count() or 1

    def one(b):
        try:
            return decode(log_probs[b, : int(lens[b])], **kw)
        except OracleError as exc:
            raise OracleError(f"utterance {b}: {exc}") from exc

    if threads <= 1 or len(lens) <= 1:
        return [one(b) for b in range(len(lens))]
    with ThreadPoolExecutor(max_workers=threads) as pool:
        return list(pool.map(one, range(len(lens))))


INF = math.inf


def align(lp: np.ndarray, targets, blank: int = 0) -> np.ndarray:
    """CTC forced alignment of one utterance (align.py:46-123): per-frame labels.
    Raises OracleError with the reference's messages."""
    lp = np.ascontiguousarray(lp, dtype=np.float64)
    T, V = lp.shape
    tg = np.ascontiguousarray(np.asarray(list(targets), dtype=np.int32))
    labels = np.zeros(max(T, 1), dtype=np.int32)
    rc = _lib().ctco_align(_ptr(lp, ctypes.c_double), T, V, blank, _ptr(tg, ctypes.c_int32), len(tg),
                           _ptr(labels, ctypes.c_int32))
    if rc == 11:
        raise OracleError("targets must be non-empty")
    if rc == 12:
        raise OracleError("targets must not contain the blank token")
    if rc == 13:
        bad = next(int(t) for t in tg if not 0 <= t < V)
        raise OracleError(f"target token {bad} out of range [0, {V})")
    if rc == 14:
        reps = int(sum(a == b for a, b in zip(tg[:-1], tg[1:])))
        raise OracleError(f"infeasible alignment: {T} frames cannot fit {len(tg)} targets "
                          f"with {reps} adjacent repeats (need at least {len(tg) + reps})")
    if rc == 15:
        raise OracleError("no feasible alignment path")
    return labels[:T]
