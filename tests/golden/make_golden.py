"""Generate golden vectors from the REFERENCE decoder (ctcforge, imported from
/root/reference in the build container; it does not exist on the GPU box).

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Writes ``tests/golden/golden.json`` with
  * known-answer cases mirroring the reference tests (test_decoder.py:45-51,
    :345-352; test_emissions.py:210-255),
  * seeded small random cases in the style of the reference's differential test
    (test_decoder.py:147-165), with their float64 inputs inline,
  * utterances of the BASELINE.json config shapes (regenerated on the fly from
    paper_2310_17864_b200.synth seeds; the fixture stores the SHA-256 of the
    float32 input bytes so a generator drift is detected).
Every case records ctcforge's n-best (tokens, timesteps, score) and frame map.
The CUDA parity tests use the fp32 cases; the oracle tests use all of them.
"""

from __future__ import annotations

import hashlib
import json
import math
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, "/root/reference/pkg/src")

from ctcforge import (  # noqa: E402
    DecoderOptions,
    EmissionMatrix,
    TokenDictionary,
    beam_search_decode,
    blank_collapse,
)

from paper_2310_17864_b200 import synth  # noqa: E402


def sha(x: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()


def toks(v):
    return TokenDictionary(tuple(["-"] + [f"t{i}" for i in range(1, v)]), blank_index=0)


def run(lp, beam, n_best, thr=1.0, beam_threshold=50.0, k=None, merge="logadd", strict=True):
    e = EmissionMatrix(lp, strict=strict)
    opts = DecoderOptions(beam_size=beam, n_best=n_best, blank_skip_threshold=thr,
                          beam_threshold=beam_threshold, beam_size_token=k, merge_mode=merge)
    nb = beam_search_decode(e, toks(lp.shape[1]), opts)
    fm = (blank_collapse(e, thr, 0).frame_map if thr < 1.0 else np.arange(lp.shape[0]))
    return {
        "tokens": [h.tokens for h in nb],
        "timesteps": [h.timesteps for h in nb],
        "scores": [h.score for h in nb],
        "frame_map": [int(x) for x in fm],
    }


def jf(x):
    """JSON-safe float (inf thresholds)."""
    return "inf" if x == math.inf else x


def log_softmax_rows(x):
    m = x.max(axis=1, keepdims=True)
    z = x - m
    return z - np.log(np.exp(z).sum(axis=1, keepdims=True))


def main():
    out = {"generator": "tests/golden/make_golden.py", "reference": "ctcforge 0.1.0 (/root/reference/pkg)",
           "known": [], "small": [], "configs": []}

    # -- known answers ------------------------------------------------------
    eps = 1e-13
    path = [1, 1, 0, 2, 3]
    probs = np.full((5, 4), eps)
    probs[np.arange(5), path] = 1.0 - 3 * eps
    lp = np.log(probs)
    out["known"].append({"name": "one_hot_greedy", "ref": "test_decoder.py:45-51", "lp": lp.tolist(),
                         "beam": 4, "n_best": 1, "thr": 1.0, **run(lp, 4, 1)})
    lp = np.log(np.full((4, 3), [0.98, 0.01, 0.01]))
    out["known"].append({"name": "collapse_to_nothing", "ref": "test_decoder.py:345-352", "lp": lp.tolist(),
                         "beam": 10, "n_best": 1, "thr": 0.9, **run(lp, 10, 1, thr=0.9)})
    lp = np.log(np.array([[0.99, 0.005, 0.005], [0.50, 0.25, 0.25], [0.99, 0.005, 0.005]]))
    out["known"].append({"name": "blank_collapse_drops", "ref": "test_emissions.py:218-229", "lp": lp.tolist(),
                         "beam": 10, "n_best": 1, "thr": 0.95, **run(lp, 10, 1, thr=0.95)})
    lp = np.log(np.array([[0.95, 0.03, 0.02], [0.2, 0.4, 0.4]]))
    out["known"].append({"name": "blank_collapse_exact_threshold", "ref": "test_emissions.py:251-255",
                         "lp": lp.tolist(), "beam": 10, "n_best": 1, "thr": 0.95, **run(lp, 10, 1, thr=0.95)})
    rng = np.random.default_rng(7)
    t, v = 400, 6
    dominated = rng.random(t) < 0.7
    pr = np.empty((t, v))
    for i in range(t):
        bp = rng.uniform(0.96, 0.995) if dominated[i] else rng.uniform(0.05, 0.90)
        rest = rng.random(v - 1)
        rest = (1 - bp) * rest / rest.sum()
        pr[i] = np.concatenate([[bp], rest])
    lp = np.log(pr)
    out["known"].append({"name": "blank_collapse_counting", "ref": "test_emissions.py:232-248", "lp": lp.tolist(),
                         "beam": 10, "n_best": 3, "thr": 0.95, **run(lp, 10, 3, thr=0.95)})
    # exact ties everywhere: uniform rows (tie-break by token sequence)
    lp = np.log(np.full((4, 4), 0.25))
    out["known"].append({"name": "uniform_rows_ties", "ref": "decoder.py:651-681", "lp": lp.tolist(),
                         "beam": 6, "n_best": 6, "thr": 1.0, **run(lp, 6, 6)})

    # -- seeded small random cases (differential-test style) ----------------
    for seed in range(24):
        rng = np.random.default_rng(1000 + seed)
        t, v = int(rng.integers(1, 10)), int(rng.integers(2, 8))
        lp64 = log_softmax_rows(rng.normal(size=(t, v)) * float(rng.uniform(0.5, 3.0)))
        lp32 = lp64.astype(np.float32)
        beam = int(rng.integers(1, 9))
        nb = int(rng.integers(1, beam + 1))
        thr = float(rng.choice([1.0, 0.9, 0.6]))
        bth = float(rng.choice([50.0, 3.0, math.inf]))
        for merge, k in (("logadd", None), ("max", None), ("logadd", 2)):
            out["small"].append({"seed": seed, "dtype": "float64", "lp": lp64.tolist(), "beam": beam,
                                 "n_best": nb, "thr": thr, "beam_threshold": jf(bth), "k": k, "merge": merge,
                                 **run(lp64, beam, nb, thr, bth, k, merge)})
        out["small"].append({"seed": seed, "dtype": "float32", "lp": lp32.astype(np.float64).tolist(),
                             "beam": beam, "n_best": nb, "thr": thr, "beam_threshold": jf(bth), "k": None,
                             "merge": "logadd", **run(lp32.astype(np.float64), beam, nb, thr, bth, strict=False)})

    # -- config-shaped utterances (inputs regenerated from seeds) -----------
    plan = [(0, range(4), [10]), (1, range(4), [10]), (2, range(2), [1, 10, 50, 100]), (3, range(2), [10]),
            (4, [0, 4095], [10])]
    for c, idx, beams in plan:
        cfg = synth.CONFIGS[c]
        lp, lens = synth.batch(cfg, indices=list(idx))
        for j, b in enumerate(idx):
            x = lp[j, : lens[j]]
            for beam in beams:
                nb = min(beam, 10) if c == 2 else cfg.nbest
                full = run(x.astype(np.float64), beam, beam, cfg.threshold, strict=True)
                res = run(x.astype(np.float64), beam, nb, cfg.threshold, strict=True)
                sc = full["scores"]
                out["configs"].append({
                    "cfg": c, "b": int(b), "len": int(lens[j]), "sha256": sha(x), "beam": beam, "n_best": nb,
                    "thr": cfg.threshold, **res,
                    "gap12": (sc[0] - sc[1]) if len(sc) > 1 else None,
                })
            print(f"cfg{c} b={b} len={lens[j]} done", flush=True)

    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(out, fh, separators=(",", ":"))
    print("wrote", os.path.join(HERE, "golden.json"))


if __name__ == "__main__":
    main()
