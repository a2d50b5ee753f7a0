"""Seeded synthetic CTC posteriors for the five BASELINE.json configurations.

The reference publishes no dataset for this path (LibriSpeech test-other and the
acoustic model behind the paper's Table 3, are not available),
so seeded inputs with the shapes and value distributions of BASELINE.json's
configs stand in for it.

Every utterance is generated from its own PCG64 stream
``default_rng([SEED, cfg, b])`` and lengths from ``default_rng([SEED, cfg, 10**6])``
so that any shard of a batch can be produced independently of how the batch is
split across GPUs.  Logits are float64, ``log_softmax`` is float64, and the
result is cast to float32 (the decoder's input dtype); rows beyond ``len_b`` are
zero.
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

SEED = 20261019


@dataclass(frozen=True)
class SynthConfig:
    name: str
    cfg: int
    batch: int
    vocab: int
    t_min: int
    t_max: int
    p_blank: float
    blank_peak: tuple[float, float]
    token_peak: tuple[float, float]
    sigma: float
    beam: int
    nbest: int
    threshold: float


CONFIGS = {
    0: SynthConfig("cfg0-tiny", 0, 4, 32, 200, 200, 0.6, (8.0, 8.0), (6.0, 6.0), 1.0, 10, 1, 0.95),
    1: SynthConfig("cfg1-asr", 1, 64, 500, 125, 875, 0.65, (5.0, 10.0), (4.0, 8.0), 1.5, 10, 1, 0.95),
    2: SynthConfig("cfg2-beam-sweep", 2, 256, 500, 125, 875, 0.65, (5.0, 10.0), (4.0, 8.0), 1.5, 10, 10, 0.95),
    3: SynthConfig("cfg3-large-vocab", 3, 128, 5000, 200, 1000, 0.5, (3.0, 7.0), (3.0, 7.0), 2.0, 10, 5, 0.9),
    4: SynthConfig("cfg4-whole-box", 4, 4096, 500, 125, 875, 0.65, (5.0, 10.0), (4.0, 8.0), 1.5, 10, 1, 0.95),
}


def lengths(cfg: SynthConfig) -> np.ndarray:
    """Per-utterance frame counts, uniform integers in [t_min, t_max]."""
    if cfg.t_min == cfg.t_max:
        return np.full(cfg.batch, cfg.t_max, dtype=np.int32)
    rng = np.random.default_rng([SEED, cfg.cfg, 10**6])
    return rng.integers(cfg.t_min, cfg.t_max + 1, size=cfg.batch).astype(np.int32)


def utterance(cfg: SynthConfig, b: int, n_frames: int) -> np.ndarray:
    """One utterance's float32 log-probabilities, shape [n_frames, V]."""
    rng = np.random.default_rng([SEED, cfg.cfg, b])
    v = cfg.vocab
    logits = rng.normal(0.0, cfg.sigma, size=(n_frames, v))
    is_blank = rng.random(n_frames) < cfg.p_blank
    blank_peak = rng.uniform(cfg.blank_peak[0], cfg.blank_peak[1], size=n_frames)
    token_peak = rng.uniform(cfg.token_peak[0], cfg.token_peak[1], size=n_frames)
    token = rng.integers(1, v, size=n_frames)
    rows = np.arange(n_frames)
    logits[rows[is_blank], 0] = blank_peak[is_blank]
    nb = ~is_blank
    logits[rows[nb], token[nb]] = token_peak[nb]
    m = logits.max(axis=1, keepdims=True)
    z = logits - m
    lp = z - np.log(np.exp(z).sum(axis=1, keepdims=True))
    return lp.astype(np.float32)


def batch(cfg: SynthConfig, indices=None, out=None, t_pad=None, threads: int = 8):
    """Generate utterances ``indices`` (default: all) into a padded [n, T, V] array.

    Returns ``(log_probs float32 [n, T, V], lens int32 [n])``.  ``out`` may be a
    preallocated (e.g. pinned) float32 array to fill in place.
    """
    all_lens = lengths(cfg)
    idx = np.arange(cfg.batch) if indices is None else np.asarray(indices, dtype=np.int64)
    lens = all_lens[idx]
    t = int(t_pad if t_pad is not None else (lens.max() if len(lens) else 0))
    if out is None:
        out = np.zeros((len(idx), t, cfg.vocab), dtype=np.float32)
    else:
        assert out.shape == (len(idx), t, cfg.vocab) and out.dtype == np.float32

    def fill(j):
        n = int(lens[j])
        out[j, :n] = utterance(cfg, int(idx[j]), n)
        out[j, n:] = 0.0

    if threads > 1 and len(idx) > 1:
        with ThreadPoolExecutor(max_workers=threads) as pool:
            list(pool.map(fill, range(len(idx))))
    else:
        for j in range(len(idx)):
            fill(j)
    return out, lens.astype(np.int32)


def simple_tokens(v: int) -> list[str]:
    """Token strings for a synthetic vocabulary: blank '-' at 0, then u1..u{V-1}."""
    return ["-"] + [f"u{i}" for i in range(1, v)]
