"""CTC forced alignment on the GPU (ctcforge align.py:46-165).

    forced_align(emissions, targets, tokens)          -> AlignmentResult   (align.py:46-123)
    forced_align_batch(emissions_list, targets_list, tokens) -> list[AlignmentResult]
    attribute_blanks(result)                          -> list[AlignmentSpan] (align.py:146-165)

The Viterbi pass runs in ``ctcb_align`` (one warp per utterance, fp64 path
scores, the reference's tie-breaking), so frame labels are bit-identical to
the reference's on float32-exact inputs (float64 emissions are rounded to
float32, the kernel's input dtype).  The kernel's backtrace also emits each
target's frame span (a feasible path holds target j's state in exactly one
run of frames), so the host only attaches scores: the mean frame
log-probability of a span, summed by numpy exactly as the reference does.
Tiling (attribute_blanks) and word grouping (align_words) work on span-start
arrays.  Errors are the reference's ``ValueError`` messages;
``forced_align_batch`` tags them ``utterance b: ...``.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib

ALIGN_OK, ALIGN_EMPTY, ALIGN_BLANK, ALIGN_RANGE, ALIGN_INFEASIBLE, ALIGN_NO_PATH, ALIGN_BAD_LEN = range(7)


@dataclass(frozen=True)
class AlignmentSpan:
    token: int
    start_frame: int
    end_frame: int  # exclusive
    score: float    # mean per-frame log-probability over the span


@dataclass
class AlignmentResult:
    frame_labels: np.ndarray  # [T] token per frame (blank allowed)
    frame_scores: np.ndarray  # [T] log-prob of the chosen label (float64)
    spans: list


def _span_score(frame_scores: np.ndarray, a: int, b: int) -> float:
    # mean of frames [a, b): numpy's pairwise summation, as align.py:137
    return float(frame_scores[a:b].mean())


def spans_from_runs(frame_labels: np.ndarray, frame_scores: np.ndarray, blank: int) -> list:
    """Token spans of a frame labelling computed on the host (for labellings
    that did not come from ctcb_align): maximal runs of one non-blank label,
    found from the label changes (align.py:126-143's result)."""
    labels = np.asarray(frame_labels)
    if labels.size == 0:
        return []
    cuts = np.flatnonzero(labels[1:] != labels[:-1]) + 1
    starts = np.concatenate(([0], cuts))
    ends = np.concatenate((cuts, [labels.size]))
    keep = labels[starts] != blank
    return [AlignmentSpan(int(labels[a]), int(a), int(b), _span_score(frame_scores, a, b))
            for a, b in zip(starts[keep], ends[keep])]


def attribute_blanks(result: AlignmentResult) -> list:
    """Widen spans so they tile [0, T): blank frames join the preceding span,
    leading blanks the first one (align.py:146-165).  Span i covers
    [start_i, start_{i+1}) with start_0 -> 0 and start_n -> T."""
    n = len(result.spans)
    if n == 0:
        return []
    bounds = [0] + [sp.start_frame for sp in result.spans[1:]] + [len(result.frame_labels)]
    return [AlignmentSpan(sp.token, bounds[i], bounds[i + 1], _span_score(result.frame_scores, bounds[i], bounds[i + 1]))
            for i, sp in enumerate(result.spans)]


def _blank_of(tokens) -> int:
    if tokens is None:
        return 0
    if isinstance(tokens, int):
        return tokens
    return int(getattr(tokens, "blank_index", 0))


def _log_probs(e) -> np.ndarray:
    lp = np.asarray(getattr(e, "log_probs", e))
    if lp.ndim != 2:
        raise ValueError(f"log_probs must be 2-D, got shape {lp.shape}")
    return lp


def forced_align_batch(emissions, targets, tokens=None, device: int = 0, raise_errors: bool = True) -> list:
    """Align a batch in one ``ctcb_align`` launch; ``tokens`` is a
    TokenDictionary-like object (``blank_index``), a blank index, or None (0).
    With ``raise_errors=False`` a failing utterance yields its error message
    (str) in place of an AlignmentResult."""
    blank = _blank_of(tokens)
    lps = [_log_probs(e) for e in emissions]
    tgs = [[int(t) for t in tg] for tg in targets]
    if len(lps) != len(tgs):
        raise ValueError("one target sequence per utterance is required")
    if not lps:
        return []
    V = lps[0].shape[1]
    for b, lp in enumerate(lps):
        if lp.shape[1] != V:
            raise ValueError(f"utterance {b}: emissions have {lp.shape[1]} columns, expected {V}")
    B = len(lps)
    T = max(max(lp.shape[0] for lp in lps), 1)
    s_max = 2 * max(max((len(t) for t in tgs), default=0), 1) + 1
    dev = torch.device("cuda", device)
    x = torch.zeros((B, T, V), dtype=torch.float32)
    for b, lp in enumerate(lps):
        x[b, : lp.shape[0]] = torch.from_numpy(np.array(lp, dtype=np.float32))
    x = x.to(dev)
    lens = torch.tensor([lp.shape[0] for lp in lps], dtype=torch.int32, device=dev)
    offs = np.zeros(B + 1, dtype=np.int32)
    offs[1:] = np.cumsum([len(t) for t in tgs])
    flat = torch.tensor([c for t in tgs for c in t] or [0], dtype=torch.int32, device=dev)
    toff = torch.from_numpy(offs).to(dev)
    lib = _lib.load()
    n = ctypes.c_size_t()
    _lib.check(lib.ctcb_align_workspace_bytes(B, T, s_max, ctypes.byref(n)), "ctcb_align_workspace_bytes")
    ws = torch.empty(max(n.value, 1), dtype=torch.uint8, device=dev)
    labels = torch.zeros((B, T), dtype=torch.int32, device=dev)
    scores = torch.zeros((B, T), dtype=torch.float32, device=dev)
    status = torch.full((B,), -1, dtype=torch.int32, device=dev)
    span_a = torch.zeros(max(int(offs[-1]), 1), dtype=torch.int32, device=dev)
    span_b = torch.zeros_like(span_a)
    vp = ctypes.c_void_p
    stream = torch.cuda.current_stream(dev).cuda_stream
    with torch.cuda.device(dev):
        _lib.check(lib.ctcb_align(vp(x.data_ptr()), x.stride(0), x.stride(1), vp(lens.data_ptr()),
                                  vp(flat.data_ptr()), vp(toff.data_ptr()), B, T, V, blank, s_max,
                                  vp(ws.data_ptr()), ws.numel(), vp(stream), vp(labels.data_ptr()),
                                  vp(scores.data_ptr()), vp(status.data_ptr()), vp(span_a.data_ptr()),
                                  vp(span_b.data_ptr())), "ctcb_align")
    st = status.cpu().numpy()
    lab = labels.cpu().numpy()
    sco = scores.cpu().numpy()
    sa, sb = span_a.cpu().numpy(), span_b.cpu().numpy()
    out = []
    for b in range(B):
        Tb = lps[b].shape[0]
        if st[b] != ALIGN_OK:
            msg = _message(int(st[b]), tgs[b], Tb, V)
            if raise_errors:
                raise ValueError(f"utterance {b}: " + msg)
            out.append(msg)
            continue
        fl = lab[b, :Tb].astype(np.int64)
        fs = sco[b, :Tb].astype(np.float64)
        o0 = int(offs[b])
        spans = [AlignmentSpan(tok, int(sa[o0 + j]), int(sb[o0 + j]), _span_score(fs, int(sa[o0 + j]), int(sb[o0 + j])))
                 for j, tok in enumerate(tgs[b])]
        out.append(AlignmentResult(frame_labels=fl, frame_scores=fs, spans=spans))
    return out


def _message(code: int, targets: list, T: int, V: int) -> str:
    # align.py:60-76, :108-110
    if code == ALIGN_EMPTY:
        return "targets must be non-empty"
    if code == ALIGN_BLANK:
        return "targets must not contain the blank token"
    if code == ALIGN_RANGE:
        bad = next(t for t in targets if not 0 <= t < V)
        return f"target token {bad} out of range [0, {V})"
    if code == ALIGN_INFEASIBLE:
        reps = sum(a == b for a, b in zip(targets, targets[1:]))
        return (f"infeasible alignment: {T} frames cannot fit {len(targets)} targets "
                f"with {reps} adjacent repeats (need at least {len(targets) + reps})")
    if code == ALIGN_NO_PATH:
        return "no feasible alignment path"
    if code < 0:
        raise _lib.CtcbError("ctcb_align left an utterance unprocessed (kernel did not run)")
    return "length out of range"


def forced_align(emissions, targets, tokens=None, device: int = 0) -> AlignmentResult:
    """Globally best frame-to-target alignment of one utterance (align.py:46-123)."""
    try:
        return forced_align_batch([emissions], [targets], tokens, device)[0]
    except ValueError as exc:
        msg = str(exc)
        raise ValueError(msg.split(": ", 1)[1] if msg.startswith("utterance 0: ") else msg) from None


@dataclass(frozen=True)
class WordSpan:
    word: str
    start_frame: int
    end_frame: int  # exclusive
    score: float


def align_words(result: AlignmentResult, tokens, transcript: list, lexicon) -> list:
    """Word spans (align.py:168-212): the transcript's first spellings
    (``lexicon.entries``: word -> spellings, tuples of token indices), laid
    end to end, must reproduce the aligned targets; word w owns the token
    spans [cut_w, cut_{w+1}) and scores the frame-weighted mean of its spans
    (span sums in span order over the frames they cover)."""
    first = []
    for word in transcript:
        variants = lexicon.entries.get(word)
        if not variants:
            raise ValueError(f"word {word!r} is not in the lexicon")
        first.append(tuple(variants[0]))
    if [t for sp in first for t in sp] != [sp.token for sp in result.spans]:
        raise ValueError("concatenated transcript spellings do not match the aligned targets")
    cuts = np.cumsum([0] + [len(sp) for sp in first])
    sums = [float(result.frame_scores[sp.start_frame: sp.end_frame].sum()) for sp in result.spans]
    widths = [sp.end_frame - sp.start_frame for sp in result.spans]
    words = []
    for w, word in enumerate(transcript):
        a, b = int(cuts[w]), int(cuts[w + 1])
        words.append(WordSpan(word, result.spans[a].start_frame, result.spans[b - 1].end_frame,
                              sum(sums[a:b]) / sum(widths[a:b])))
    return words
