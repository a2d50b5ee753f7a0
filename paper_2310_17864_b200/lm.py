"""Backoff n-gram LMs from ARPA text, for token-level shallow fusion.

Host side of the reference's ``lm.py`` (ctcforge lm.py:1-270), built around
the flat arrays the device consumes: the ARPA reader appends every n-gram
straight into per-order columns (word ids, natural-log probability, backoff)
with a tuple -> row index, so :func:`flatten` for ``ctcb_lm_create`` is a
concatenation, and ``NGramLM.tables[n]`` is a read-only view over those
columns.  Scores are natural log (log10 × ln 10 at parse time, lm.py:183-184);
the reader's validation order and messages are the reference's.

The incremental API (``lm_start`` / ``lm_score`` / ``lm_finish``, contexts as
word-id tuples) serves the tests and the oracle tables; the decoder itself
scores on the device (csrc/ctcb_lm.cu).  Models parsed by the reference
(objects with ``order``, ``tables``, ``vocab``) are accepted by
:func:`flatten`, :func:`token_words` and the scoring functions.
"""

from __future__ import annotations

import logging
import math
import re
from collections.abc import Mapping
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

LN10 = math.log(10.0)
OOV_PENALTY = -20.0  # out-of-vocabulary word without <unk> (lm.py:22-24)

log = logging.getLogger(__name__)

_SECTION = re.compile(r"\\(\d+)-grams:")
_COUNT = re.compile(r"ngram\s+(\d+)\s*=\s*(\d+)")


class ArpaFormatError(ValueError):
    """The file is not well-formed ARPA text (lm.py:31-32)."""


class _OrderColumns(Mapping):
    """All n-grams of one order: row index by word-id tuple plus parallel
    columns; as a Mapping, tuple -> (logprob, backoff) like the reference's
    per-order dict."""

    def __init__(self, n: int):
        self.n = n
        self.index: dict = {}
        self.ids: list = []
        self.logprob: list = []
        self.backoff: list = []

    def add(self, key: tuple, lp: float, bo: float) -> None:
        row = self.index.get(key)
        if row is None:  # a repeated n-gram keeps its first row, its last values
            self.index[key] = len(self.ids)
            self.ids.append(key)
            self.logprob.append(lp)
            self.backoff.append(bo)
        else:
            self.logprob[row], self.backoff[row] = lp, bo

    def __getitem__(self, key):
        row = self.index[key]
        return self.logprob[row], self.backoff[row]

    def get(self, key, default=None):
        row = self.index.get(key)
        return default if row is None else (self.logprob[row], self.backoff[row])

    def __contains__(self, key) -> bool:
        return key in self.index

    def __iter__(self):
        return iter(self.ids)

    def __len__(self) -> int:
        return len(self.ids)


@dataclass
class NGramLM:
    """``tables[n]``: word-id n-tuple -> (logprob, backoff), natural log
    (``tables[0]`` unused); ``vocab``: word -> id (lm.py:35-50)."""

    order: int
    tables: list
    vocab: dict = field(default_factory=dict)

    @property
    def unk_id(self):
        return self.vocab.get("<unk>")


@dataclass(eq=False)
class LMState:
    """Scoring context (word-id tuple) and the running total; two states are
    equal when their contexts are (lm.py:53-74)."""

    context: tuple = ()
    cumulative_score: float = 0.0

    def __post_init__(self):
        self.context = tuple(self.context)

    def __eq__(self, other) -> bool:
        return isinstance(other, LMState) and self.context == other.context

    def __hash__(self) -> int:
        return hash(self.context)


class _ArpaReader:
    """One pass over the file: `\\data\\` counts, then the n-gram sections."""

    def __init__(self, path: Path):
        self.path = path
        self.lines = path.read_text(encoding="utf-8").splitlines()
        self.counts: dict = {}
        self.vocab: dict = {}
        self.orders: dict = {}

    def fail(self, msg: str, line: int | None = None):
        where = f"{self.path}: line {line + 1}" if line is not None else f"{self.path}"
        raise ArpaFormatError(f"{where}: {msg}")

    def header(self) -> int:
        """Index of the first line after the count block."""
        try:
            at = next(k for k, s in enumerate(self.lines) if s.strip() == "\\data\\") + 1
        except StopIteration:
            self.fail("missing \\data\\ header")
        for k in range(at, len(self.lines)):
            s = self.lines[k].strip()
            if not s:
                continue
            m = _COUNT.fullmatch(s)
            if m is None:
                return self._counted(k)
            self.counts[int(m.group(1))] = int(m.group(2))
        return self._counted(len(self.lines))

    def _counted(self, k: int) -> int:
        if not self.counts:
            self.fail("no 'ngram N=count' lines after \\data\\")
        return k

    def body(self, start: int) -> None:
        top = max(self.counts)
        section = None
        finished = False
        for k in range(start, len(self.lines)):
            s = self.lines[k].strip()
            if not s:
                continue
            if s == "\\end\\":
                finished, section = True, None
                continue
            if finished:
                self.fail("content after \\end\\", k)
            m = _SECTION.fullmatch(s)
            if m is not None:
                n = int(m.group(1))
                if n not in self.counts:
                    self.fail(f"section \\{n}-grams: was not declared in \\data\\", k)
                if n in self.orders:
                    self.fail(f"duplicate \\{n}-grams: section", k)
                section = self.orders[n] = _OrderColumns(n)
                continue
            if section is None:
                self.fail("unexpected content outside a section", k)
            self._entry(section, s.split(), top, k)
        if not finished:
            self.fail("missing \\end\\")

    def _entry(self, section: _OrderColumns, f: list, top: int, k: int) -> None:
        n = section.n
        with_bo = len(f) == n + 2
        if not (len(f) == n + 1 or (with_bo and n != top)):
            self.fail(f"malformed {n}-gram line", k)
        try:
            lp = float(f[0]) * LN10
            bo = float(f[-1]) * LN10 if with_bo else 0.0
        except ValueError:
            self.fail(f"malformed {n}-gram line", k)
        key = tuple(self.vocab.setdefault(w, len(self.vocab)) for w in f[1:n + 1])
        section.add(key, lp, bo)

    def model(self, strict: bool) -> NGramLM:
        order = max(self.counts)
        tables = [_OrderColumns(0)] + [self.orders.get(n) or _OrderColumns(n) for n in range(1, order + 1)]
        for n in sorted(self.counts):
            declared = self.counts[n]
            if n not in self.orders and declared > 0:
                self.fail(f"missing \\{n}-grams: section")
            if len(tables[n]) != declared:
                self.fail(f"\\data\\ declares {declared} {n}-grams, file has {len(tables[n])}")
        orphans = sum(key[:-1] not in tables[len(key) - 1] for n in range(2, order + 1) for key in tables[n])
        if orphans:
            msg = f"{self.path}: {orphans} n-grams have no lower-order context entry (pruned model?)"
            if strict:
                raise ArpaFormatError(msg)
            log.warning(msg)
        return NGramLM(order=order, tables=tables, vocab=self.vocab)


def parse_arpa(path, strict: bool = False) -> NGramLM:
    """Read an ARPA file (lm.py:77-226).  Errors name the file and line;
    n-grams whose (n-1)-gram context is absent warn (``strict``: raise)."""
    reader = _ArpaReader(Path(path))
    reader.body(reader.header())
    return reader.model(strict)


# ------------------------------------------------------------------ scoring (lm.py:229-270)
def _longest_known(lm, ctx: tuple) -> tuple:
    """Longest suffix of ``ctx`` that is itself an n-gram of the model (a
    context absent from the model cannot affect later scores)."""
    for k in range(len(ctx), 0, -1):
        suffix = ctx[len(ctx) - k:]
        if suffix in lm.tables[k]:
            return suffix
    return ()


def _katz(lm, context: tuple, wid: int) -> float:
    """Backoff log-probability of ``wid`` after ``context``: the longest
    matching n-gram, plus the backoff weights of the longer contexts that
    missed, accumulated from the longest one down (lm.py:229-245)."""
    hist = context[max(len(context) - (lm.order - 1), 0):] if lm.order > 1 else ()
    penalty = 0.0
    for k in range(len(hist), -1, -1):
        suffix = hist[len(hist) - k:]
        hit = lm.tables[k + 1].get(suffix + (wid,))
        if hit is not None:
            return penalty + hit[0]
        if k == 0:
            break
        ctx = lm.tables[k].get(suffix)
        if ctx is not None:
            penalty += ctx[1]
    return penalty + OOV_PENALTY  # word only in higher orders of a broken model


def context_start(lm) -> tuple:
    sid = lm.vocab.get("<s>")
    return () if sid is None or lm.order == 1 else _longest_known(lm, (sid,))


def context_score(lm, context: tuple, word: str):
    """(next context, natural-log score) of ``word`` after ``context``; unknown
    words score as ``<unk>`` or, without one, the fixed penalty with the
    context reset."""
    wid = lm.vocab.get(word, lm.vocab.get("<unk>"))
    if wid is None:
        return (), OOV_PENALTY
    score = _katz(lm, context, wid)
    if lm.order == 1:
        return (), score
    grown = context + (wid,)
    return _longest_known(lm, grown[max(len(grown) - (lm.order - 1), 0):]), score


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


def _columns(lm, n: int):
    """(keys, logprobs, backoffs) of order n: the reader's columns, or a
    reference model's dict."""
    t = lm.tables[n]
    if isinstance(t, _OrderColumns):
        return t.ids, t.logprob, t.backoff
    keys = list(t)
    vals = [t[k] for k in keys]
    return keys, [v[0] for v in vals], [v[1] for v in vals]


def flatten(lm) -> FlatLM:
    order = int(lm.order)
    cols = [_columns(lm, n) for n in range(1, order + 1)]
    N = sum(len(c[0]) for c in cols)
    words = np.full((N, order), -1, dtype=np.int32)
    lengths = np.repeat(np.arange(1, order + 1, dtype=np.int32), [len(c[0]) for c in cols])
    row = 0
    for n, (keys, _, _) in enumerate(cols, start=1):
        if keys:
            words[row: row + len(keys), :n] = np.asarray(keys, dtype=np.int32).reshape(len(keys), n)
        row += len(keys)
    lp = np.fromiter((x for c in cols for x in c[1]), dtype=np.float64, count=N)
    bo = np.fromiter((x for c in cols for x in c[2]), dtype=np.float64, count=N)
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
    ids = [lm.vocab.get(t, unk) for t in tokens]
    out = np.array([-1 if w is None else w for w in ids], dtype=np.int32)
    out[blank] = -2
    if sil is not None:
        out[sil] = -2
    return out
