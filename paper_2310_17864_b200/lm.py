"""Backoff n-gram LMs from ARPA text, for token-level shallow fusion.

Host side of the reference's ``lm.py`` (ctcforge lm.py:1-270): the ARPA
reader with the reference's validation and messages, the model type, and the
incremental scoring API.  Scores are natural-log (log10 × ln 10 at parse time,
lm.py:183-184).  The decoder does not score on the host: :func:`flatten` turns a
model into flat n-gram arrays for ``ctcb_lm_create``, and the device builds the
(context × token) score / successor tables from them (csrc/ctcb_lm.cu).

Models parsed by the reference itself (objects with ``order``, ``tables``,
``vocab``) are accepted wherever an :class:`NGramLM` is.
"""

from __future__ import annotations

import logging
import math
import re
from dataclasses import dataclass
from pathlib import Path

import numpy as np

LN10 = math.log(10.0)
OOV_PENALTY = -20.0  # lm.py:22-24

log = logging.getLogger(__name__)

_SECTION = re.compile(r"\\(\d+)-grams:")
_COUNT = re.compile(r"ngram\s+(\d+)\s*=\s*(\d+)")


class ArpaFormatError(ValueError):
    """The file is not well-formed ARPA text (lm.py:31-32)."""


@dataclass
class NGramLM:
    """``tables[n]``: n-tuple of word ids -> (logprob, backoff), natural log;
    ``vocab``: word -> id (lm.py:35-50)."""

    order: int
    tables: list
    vocab: dict

    @property
    def unk_id(self):
        return self.vocab.get("<unk>")


class LMState:
    """Context word ids plus a running total; equality by context (lm.py:53-74)."""

    __slots__ = ("context", "cumulative_score")

    def __init__(self, context=(), cumulative_score: float = 0.0):
        self.context = tuple(context)
        self.cumulative_score = cumulative_score

    def __eq__(self, other) -> bool:
        return isinstance(other, LMState) and self.context == other.context

    def __hash__(self) -> int:
        return hash(self.context)

    def __repr__(self) -> str:
        return f"LMState(context={self.context}, cumulative_score={self.cumulative_score})"


def parse_arpa(path, strict: bool = False) -> NGramLM:
    """Read an ARPA file (lm.py:77-226): header counts, one section per order,
    ``\\end\\``; errors name the file and line.  Missing lower-order prefixes
    warn (``strict=True``: raise)."""
    path = Path(path)
    lines = path.read_text(encoding="utf-8").splitlines()
    n_lines = len(lines)
    i = 0
    while i < n_lines and lines[i].strip() != "\\data\\":
        i += 1
    if i == n_lines:
        raise ArpaFormatError(f"{path}: missing \\data\\ header")
    i += 1
    counts: dict[int, int] = {}
    while i < n_lines:
        s = lines[i].strip()
        if s:
            m = _COUNT.fullmatch(s)
            if m is None:
                break
            counts[int(m.group(1))] = int(m.group(2))
        i += 1
    if not counts:
        raise ArpaFormatError(f"{path}: no 'ngram N=count' lines after \\data\\")
    order = max(counts)
    vocab: dict[str, int] = {}
    tables: list[dict] = [{} for _ in range(order + 1)]
    seen: set[int] = set()
    ended = False
    cur = None
    for ln in range(i, n_lines):
        s = lines[ln].strip()
        if not s:
            continue
        where = f"{path}: line {ln + 1}"
        if s == "\\end\\":
            ended = True
            cur = None
            continue
        if ended:
            raise ArpaFormatError(f"{where}: content after \\end\\")
        m = _SECTION.fullmatch(s)
        if m is not None:
            cur = int(m.group(1))
            if cur not in counts:
                raise ArpaFormatError(f"{where}: section \\{cur}-grams: was not declared in \\data\\")
            if cur in seen:
                raise ArpaFormatError(f"{where}: duplicate \\{cur}-grams: section")
            seen.add(cur)
            continue
        if cur is None:
            raise ArpaFormatError(f"{where}: unexpected content outside a section")
        n = cur
        f = s.split()
        if len(f) not in (n + 1, n + 2) or (len(f) == n + 2 and n == order):
            raise ArpaFormatError(f"{where}: malformed {n}-gram line")
        try:
            lp = float(f[0]) * LN10
            bo = float(f[n + 1]) * LN10 if len(f) == n + 2 else 0.0
        except ValueError:
            raise ArpaFormatError(f"{where}: malformed {n}-gram line") from None
        key = tuple(vocab.setdefault(word, len(vocab)) for word in f[1:n + 1])
        tables[n][key] = (lp, bo)
    if not ended:
        raise ArpaFormatError(f"{path}: missing \\end\\")
    for n, declared in sorted(counts.items()):
        if n not in seen and declared > 0:
            raise ArpaFormatError(f"{path}: missing \\{n}-grams: section")
        if len(tables[n]) != declared:
            raise ArpaFormatError(f"{path}: \\data\\ declares {declared} {n}-grams, file has {len(tables[n])}")
    missing = sum(1 for n in range(2, order + 1) for ng in tables[n] if ng[:-1] not in tables[n - 1])
    if missing:
        msg = f"{path}: {missing} n-grams have no lower-order context entry (pruned model?)"
        if strict:
            raise ArpaFormatError(msg)
        log.warning(msg)
    return NGramLM(order=order, tables=tables, vocab=vocab)


# ------------------------------------------------------------------ scoring (lm.py:229-270)
def _known(lm, ctx: tuple) -> tuple:
    while ctx and ctx not in lm.tables[len(ctx)]:
        ctx = ctx[1:]
    return ctx


def _backoff(lm, context: tuple, wid: int) -> float:
    ctx = context[-(lm.order - 1):] if lm.order > 1 else ()
    acc = 0.0
    while True:
        hit = lm.tables[len(ctx) + 1].get(ctx + (wid,))
        if hit is not None:
            return acc + hit[0]
        if not ctx:
            return acc + OOV_PENALTY
        c = lm.tables[len(ctx)].get(ctx)
        if c is not None:
            acc += c[1]
        ctx = ctx[1:]


def context_start(lm) -> tuple:
    sid = lm.vocab.get("<s>")
    return () if sid is None or lm.order == 1 else _known(lm, (sid,))


def context_score(lm, context: tuple, word: str):
    wid = lm.vocab.get(word)
    if wid is None:
        wid = lm.vocab.get("<unk>")
        if wid is None:
            return (), OOV_PENALTY
    score = _backoff(lm, context, wid)
    if lm.order == 1:
        return (), score
    return _known(lm, (context + (wid,))[-(lm.order - 1):]), score


def lm_start(lm) -> LMState:
    return LMState(context_start(lm), 0.0)


def lm_score(lm, state: LMState, word: str):
    nxt, score = context_score(lm, state.context, word)
    return LMState(nxt, state.cumulative_score + score), score


def lm_finish(lm, state: LMState) -> float:
    return context_score(lm, state.context, "</s>")[1]


# ------------------------------------------------------------------ device export
@dataclass
class FlatLM:
    """N-gram arrays for ``ctcb_lm_create``: row i is n-gram i (orders
    ascending), ``words[i, :n]`` its word ids (-1 padded)."""

    order: int
    words: np.ndarray     # int32 [N, order]
    lengths: np.ndarray   # int32 [N]
    logprob: np.ndarray   # float64 [N]
    backoff: np.ndarray   # float64 [N]
    start: np.ndarray     # int32 [order - 1] start context (-1 padded)
    start_len: int
    eos: int              # word id scored at the end ("</s>", else <unk>, else -1: OOV)
    unk: int


def flatten(lm) -> FlatLM:
    order = int(lm.order)
    rows = [(ng, v) for n in range(1, order + 1) for ng, v in lm.tables[n].items()]
    N = len(rows)
    words = np.full((N, order), -1, dtype=np.int32)
    lengths = np.empty(N, dtype=np.int32)
    lp = np.empty(N, dtype=np.float64)
    bo = np.empty(N, dtype=np.float64)
    for i, (ng, (a, b)) in enumerate(rows):
        words[i, :len(ng)] = ng
        lengths[i] = len(ng)
        lp[i] = a
        bo[i] = b
    st = context_start(lm)
    start = np.full(max(order - 1, 1), -1, dtype=np.int32)
    start[:len(st)] = st
    unk = lm.vocab.get("<unk>")
    eos = lm.vocab.get("</s>", unk)
    return FlatLM(order, words, lengths, lp, bo, start, len(st), -1 if eos is None else int(eos),
                  -1 if unk is None else int(unk))


def token_words(lm, tokens, blank: int, sil=None) -> np.ndarray:
    """Per token: its LM word id (``<unk>`` for unknown strings), -1 when the
    word is out of vocabulary with no ``<unk>`` (fixed OOV penalty, context
    reset), -2 for blank / silence (identity: no LM score, context kept;
    decoder.py:178-229)."""
    unk = lm.vocab.get("<unk>")
    out = np.empty(len(tokens), dtype=np.int32)
    for c, t in enumerate(tokens):
        if c == blank or (sil is not None and c == sil):
            out[c] = -2
            continue
        wid = lm.vocab.get(t, unk)
        out[c] = -1 if wid is None else wid
    return out
