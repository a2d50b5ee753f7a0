"""ctcforge-shaped entry points on the GPU.

Drop-in counterparts of the reference's own API for the lexicon-free, LM-free
search:

    beam_search_decode(emissions, tokens, opts)       decoder.py:102-135
    decode_batch(emissions, tokens, opts, workers)     decoder.py:138-170

They take the reference's argument *shapes*: ``emissions`` is a [T, V] array
(or a list of them, or any object with ``log_probs`` / ``frame_map``
attributes like ctcforge's EmissionMatrix); ``tokens`` is a list of strings or
an object with ``tokens`` / ``blank_index``; ``opts`` carries
``beam_size, n_best, blank_skip_threshold, beam_threshold, beam_size_token,
merge_mode`` (a ``DecoderOptions`` here or ctcforge's own).  They return
``NBestList``s of ``Hypothesis(tokens, words=[], am_score, lm_score=0.0,
score, timesteps)`` exactly like decoder.py:69-99, decoded by libctcb.so.

What the CUDA path implements: the lexicon-free search with any
``beam_size_token`` (None / V: full vocabulary; K < V: per-frame top-K token
selection, decoder.py:440-458), ``merge_mode`` "logadd" or "max", token-level
shallow fusion with a backoff n-gram ``lm`` (decoder.py:178-259, :467-473,
:753-817; ``lm_weight``), and the silence token's ``sil_score`` bonus
(decoder.py:485-486).  A lexicon raises ``ValueError``.  fp64
emissions are rounded to fp32 (the decoder's input dtype) before decoding.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from .decoder import CUCTCDecoder

MERGE_MODES = ("logadd", "max")


@dataclass
class DecoderOptions:
    """Knob bundle with the reference's defaults and validation (decoder.py:34-66)."""

    beam_size: int = 10
    beam_size_token: int | None = None
    beam_threshold: float = 50.0
    lm_weight: float = 2.0
    word_score: float = 0.0
    sil_score: float = 0.0
    blank_skip_threshold: float = 1.0
    n_best: int = 1
    merge_mode: str = "logadd"

    def __post_init__(self):
        if self.beam_size < 1:
            raise ValueError("beam_size must be >= 1")
        if self.beam_size_token is not None and self.beam_size_token < 1:
            raise ValueError("beam_size_token must be >= 1")
        if not self.beam_threshold > 0:
            raise ValueError("beam_threshold must be positive")
        if not 0.0 < self.blank_skip_threshold <= 1.0:
            raise ValueError("blank_skip_threshold must be in (0, 1]")
        if not 1 <= self.n_best <= self.beam_size:
            raise ValueError("n_best must be in [1, beam_size]")
        if self.merge_mode not in MERGE_MODES:
            raise ValueError(f"merge_mode must be one of {MERGE_MODES}")


@dataclass
class Hypothesis:
    """One n-best entry (decoder.py:69-83)."""

    tokens: list
    words: list
    am_score: float
    lm_score: float
    score: float
    timesteps: list


@dataclass
class NBestList:
    """Hypotheses sorted by descending score (decoder.py:86-99)."""

    hypotheses: list = field(default_factory=list)

    def __iter__(self):
        return iter(self.hypotheses)

    def __len__(self):
        return len(self.hypotheses)

    def __getitem__(self, i):
        return self.hypotheses[i]


def _log_probs(e) -> np.ndarray:
    lp = getattr(e, "log_probs", e)
    lp = np.asarray(lp)
    if lp.ndim != 2:
        raise ValueError(f"log_probs must be 2-D, got shape {lp.shape}")
    fm = getattr(e, "frame_map", None)
    if fm is not None and not (len(fm) == lp.shape[0] and np.array_equal(fm, np.arange(lp.shape[0]))):
        raise ValueError("emissions were already collapsed (non-identity frame_map)")
    return lp


def _token_list(tokens):
    if hasattr(tokens, "tokens"):
        sil = getattr(tokens, "silence_index", None)
        return list(tokens.tokens), int(getattr(tokens, "blank_index", 0)), (None if sil is None else int(sil))
    return list(tokens), 0, None


_DECODERS: dict = {}


def _decoder(vocab, blank, opts, device, sil=None, lm=None) -> CUCTCDecoder:
    sil_score = float(getattr(opts, "sil_score", 0.0)) if sil is not None else 0.0
    key = (tuple(vocab), blank, opts.beam_size, opts.n_best, opts.blank_skip_threshold, opts.beam_threshold,
           opts.merge_mode, opts.beam_size_token, device, sil, sil_score, id(lm) if lm is not None else None,
           float(opts.lm_weight) if lm is not None else None)
    dec = _DECODERS.get(key)
    if dec is None:
        dec = CUCTCDecoder(vocab, blank_id=blank, beam_size=opts.beam_size, nbest=opts.n_best,
                           blank_skip_threshold=opts.blank_skip_threshold, beam_threshold=opts.beam_threshold,
                           device=device)
        dec.set_merge_mode(opts.merge_mode)
        if opts.beam_size_token is not None and opts.beam_size_token <= len(vocab):
            dec.set_beam_size_token(opts.beam_size_token)
        if sil is not None:
            dec.set_silence(sil, sil_score)
        if lm is not None:
            dec.set_lm(lm, float(opts.lm_weight))
            dec._lm_ref = lm  # keeps id(lm) in the cache key unique while cached
        _DECODERS[key] = dec
    return dec


def decode_batch(emissions, tokens, opts=None, lexicon=None, lm=None, workers: int = 1, device: int = 0):
    """GPU ``decode_batch`` (decoder.py:138-170): one launch for the batch;
    ``workers`` is accepted for signature compatibility (the GPU decodes all
    utterances concurrently).  Errors carry the utterance index."""
    if lexicon is not None:
        raise ValueError("the CUDA decoder has no lexicon mode")
    opts = opts if opts is not None else DecoderOptions()
    vocab, blank, sil = _token_list(tokens)
    lps = [_log_probs(e) for e in emissions]
    for i, lp in enumerate(lps):
        if lp.shape[1] != len(vocab):
            raise ValueError(f"utterance {i}: emissions have {lp.shape[1]} columns but the token "
                             f"dictionary has {len(vocab)} tokens")
    if not lps:
        return []
    if opts.beam_size_token is not None and opts.beam_size_token > len(vocab):  # decoder.py:124-128
        raise ValueError(f"utterance 0: beam_size_token {opts.beam_size_token} exceeds vocabulary size {len(vocab)}")
    dec = _decoder(vocab, blank, opts, device, sil, lm)
    T = max(lp.shape[0] for lp in lps)
    x = torch.zeros((len(lps), max(T, 1), len(vocab)), dtype=torch.float32)
    for b, lp in enumerate(lps):
        x[b, : lp.shape[0]] = torch.from_numpy(np.ascontiguousarray(lp, dtype=np.float32))
    lens = torch.tensor([lp.shape[0] for lp in lps], dtype=torch.int32)
    dev = torch.device("cuda", device)
    out = dec.decode(x.to(dev), lens.to(dev), timesteps=True)
    toks, ts, lengths, scores, counts = dec.to_host(out)
    lms = out.lm.cpu().numpy() if out.lm is not None else None
    sil_score = float(getattr(opts, "sil_score", 0.0))
    w = float(opts.lm_weight)
    result = []
    for b in range(len(lps)):
        hyps = []
        for j in range(int(counts[b])):
            n = int(lengths[b, j])
            sc = float(scores[b, j])
            tk = toks[b, j, :n].tolist()
            lm_v = float(lms[b, j]) if lms is not None else 0.0
            # decoder.py:805-812
            bonuses = float(opts.word_score) * 0 + sil_score * (tk.count(sil) if sil is not None else 0)
            lm_part = w * lm_v if lms is not None else 0.0
            hyps.append(Hypothesis(tokens=tk, words=[], am_score=sc - lm_part - bonuses, lm_score=lm_v, score=sc,
                                   timesteps=ts[b, j, :n].tolist()))
        result.append(NBestList(hyps))
    return result


def beam_search_decode(emissions, tokens, opts=None, lexicon=None, lm=None, device: int = 0) -> NBestList:
    """GPU ``beam_search_decode`` for one utterance (decoder.py:102-135)."""
    if _log_probs(emissions).shape[0] == 0:
        raise ValueError("empty emissions")
    try:
        return decode_batch([emissions], tokens, opts, lexicon, lm, device=device)[0]
    except ValueError as exc:
        msg = str(exc)
        raise ValueError(msg.split(": ", 1)[1] if msg.startswith("utterance 0: ") else msg) from None
