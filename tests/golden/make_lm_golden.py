"""Golden vectors for token-level LM fusion from the REFERENCE
(ctcforge.decoder.beam_search_decode with ``lm=``, decoder.py:178-259,
:467-473, :753-817; ctcforge.lm.parse_arpa, lm.py:77-226), imported in the
build container (it does not exist on the GPU box):

    python tests/golden/make_lm_golden.py

Writes ``tests/golden/lm/`` : the seeded synthetic ARPA models (our own
generator below: random backoff n-gram tables over token strings, orders 1-3,
with / without ``<unk>``, a pruned model with missing lower-order prefixes)
and ``lm_decode.json``: float32-exact emissions, decoder options, and the
reference's n-best (tokens, timesteps, score, am_score, lm_score), or its
error message.  Also the reference's ``lm_score`` / ``lm_finish`` values for
a few token sequences per model (the incremental API, lm.py:229-270).
"""

from __future__ import annotations

import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(HERE, "lm")
sys.path.insert(0, "/root/reference/pkg/src")

from ctcforge.decoder import DecoderOptions, beam_search_decode  # noqa: E402
from ctcforge.emissions import EmissionMatrix, TokenDictionary  # noqa: E402
from ctcforge.lm import lm_finish, lm_score, lm_start, parse_arpa  # noqa: E402


def write_arpa(path, tables, order):
    """tables[n]: {tuple of words: (log10 p, log10 backoff or None)}."""
    lines = ["\\data\\"] + [f"ngram {n}={len(tables[n])}" for n in range(1, order + 1)]
    for n in range(1, order + 1):
        lines += ["", f"\\{n}-grams:"]
        for ng in sorted(tables[n]):
            p, b = tables[n][ng]
            lines.append(f"{p:.6f}\t{' '.join(ng)}" + (f"\t{b:.6f}" if b is not None else ""))
    lines += ["", "\\end\\", ""]
    with open(path, "w", encoding="utf-8") as fh:
        fh.write("\n".join(lines))


def random_model(rng, words, order, unk=False, keep=0.5, prune=False):
    vocab = ["<s>", "</s>"] + list(words) + (["<unk>"] if unk else [])
    tables = {1: {}}
    for w in vocab:
        p = -99.0 if w == "<s>" else float(rng.uniform(-2.5, -0.3))
        tables[1][(w,)] = (p, float(rng.uniform(-1.0, 0.3)) if order > 1 else None)
    for n in range(2, order + 1):
        tables[n] = {}
        for ctx in list(tables[n - 1]):
            if ctx[-1] == "</s>":
                continue
            for w in vocab[1:]:
                if rng.random() < keep:
                    b = float(rng.uniform(-0.9, 0.2)) if n < order else None
                    tables[n][ctx + (w,)] = (float(rng.uniform(-2.2, -0.05)), b)
    if prune and order >= 3:
        # drop some bigrams that are prefixes of kept trigrams (pruned-model warning path)
        victims = sorted({ng[:-1] for ng in tables[3]})[:3]
        for v in victims:
            tables[2].pop(v, None)
    return tables


def logsoftmax32(x):
    x = x - x.max(1, keepdims=True)
    return (x - np.log(np.exp(x).sum(1, keepdims=True))).astype(np.float32)


def main():
    os.makedirs(OUT, exist_ok=True)
    rng = np.random.default_rng(31017)
    models = []
    specs = [  # (name, V, order, unk, keep, prune, oov_tokens)
        ("bigram_v6", 6, 2, False, 0.6, False, 0),
        ("trigram_v8", 8, 3, False, 0.4, False, 0),
        ("unigram_v5", 5, 1, False, 1.0, False, 0),
        ("bigram_unk_v9", 9, 2, True, 0.5, False, 2),
        ("bigram_oov_v7", 7, 2, False, 0.5, False, 2),
        ("trigram_pruned_v7", 7, 3, False, 0.5, True, 0),
        ("bigram_v30", 30, 2, False, 0.3, False, 3),
    ]
    for name, V, order, unk, keep, prune, n_oov in specs:
        toks = ["-"] + [f"{chr(97 + i % 26)}{i // 26 or ''}" for i in range(V - 1)]
        lm_words = toks[1: V - n_oov] if n_oov else toks[1:]
        tables = random_model(rng, lm_words, order, unk, keep, prune)
        path = os.path.join(OUT, f"{name}.arpa")
        write_arpa(path, tables, order)
        models.append({"name": name, "file": f"{name}.arpa", "tokens": toks})

    cases = []
    for m in models:
        lm = parse_arpa(os.path.join(OUT, m["file"]))
        toks = m["tokens"]
        V = len(toks)
        # incremental API values
        seqs = []
        for _ in range(3):
            n = int(rng.integers(1, 6))
            seq = [toks[int(c)] for c in rng.integers(1, V, size=n)]
            st = lm_start(lm)
            scores = []
            for w in seq:
                st, s = lm_score(lm, st, w)
                scores.append(s)
            seqs.append({"words": seq, "scores": scores, "total": st.cumulative_score,
                         "finish": lm_finish(lm, st)})
        m["api"] = seqs
        for variant in range(6):
            sil = None
            if variant == 4 and V > 5:
                sil = V - 1
            tokd = TokenDictionary(tuple(toks), blank_index=0, silence_index=sil)
            T = int(rng.integers(4, 40 if V > 10 else 14))
            peak = float(rng.choice([0.5, 1.0, 2.5]))
            lp = logsoftmax32(peak * rng.normal(size=(T, V)))
            beam = int(rng.choice([3, 5, 10, 16, 24]))
            kw = dict(beam_size=beam, n_best=min(beam, int(rng.integers(1, 6))),
                      lm_weight=float(rng.choice([0.0, 0.5, 1.7, 3.0, -0.4])),
                      beam_threshold=float(rng.choice([math.inf, 50.0, 8.0])),
                      blank_skip_threshold=float(rng.choice([1.0, 1.0, 0.9])),
                      merge_mode=str(rng.choice(["logadd", "logadd", "max"])))
            if variant == 5:
                kw["beam_size_token"] = int(rng.integers(2, V + 1))
            if sil is not None:
                kw["sil_score"] = float(rng.choice([0.0, 0.8, -1.2]))
            opts = DecoderOptions(**kw)
            case = {"model": m["name"], "lp": lp.astype(np.float64).tolist(), "sil": sil, "opts": kw}
            try:
                res = beam_search_decode(EmissionMatrix(lp.astype(np.float64)), tokd, opts, lm=lm)
                case["nbest"] = [{"tokens": h.tokens, "timesteps": h.timesteps, "score": h.score,
                                  "am_score": h.am_score, "lm_score": h.lm_score} for h in res]
            except ValueError as exc:
                case["error"] = str(exc)
            cases.append(case)
    with open(os.path.join(OUT, "lm_decode.json"), "w", encoding="utf-8") as fh:
        json.dump({"models": models, "cases": cases}, fh)
    print(len(models), "models,", len(cases), "cases,", sum("error" in c for c in cases), "errors")


if __name__ == "__main__":
    main()
