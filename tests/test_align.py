"""CTC forced alignment: the oracle and the host-side span
logic against the reference's golden outputs (CPU), and the CUDA Viterbi
kernel against both (GPU).  Golden vectors: tests/golden/make_align_golden.py."""

import json
import os

import numpy as np
import pytest

import oracle
from paper_2310_17864_b200 import align as galign

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "align.json")


def cases():
    with open(GOLD, encoding="utf-8") as fh:
        return json.load(fh)["cases"]


def spans_as_lists(spans):
    return [[s.token, s.start_frame, s.end_frame, s.score] for s in spans]


# ------------------------------------------------------------------ CPU
def test_oracle_matches_reference_golden():
    n_err = 0
    for c in cases():
        lp = np.array(c["lp"], dtype=np.float64)
        if "error" in c:
            with pytest.raises(oracle.OracleError) as exc:
                oracle.align(lp, c["targets"], c["blank"])
            assert str(exc.value) == c["error"], c["note"]
            n_err += 1
            continue
        labels = oracle.align(lp, c["targets"], c["blank"])
        assert labels.tolist() == c["labels"], c["note"]
    assert n_err == 4


def test_host_spans_match_reference_golden():
    # host spans (label runs) and tiling against the reference (align.py:126-165)
    for c in cases():
        if "error" in c:
            continue
        labels = np.array(c["labels"], dtype=np.int64)
        scores = np.array(c["scores"], dtype=np.float64)
        res = galign.AlignmentResult(labels, scores, galign.spans_from_runs(labels, scores, c["blank"]))
        assert spans_as_lists(res.spans) == c["spans"], c["note"]
        assert spans_as_lists(galign.attribute_blanks(res)) == c["tiled"], c["note"]


# ------------------------------------------------------------------ GPU
@pytest.mark.gpu
def test_kernel_matches_reference_golden():
    for c in cases():
        lp = np.array(c["lp"], dtype=np.float64)
        if "error" in c:
            with pytest.raises(ValueError) as exc:
                galign.forced_align(lp, c["targets"], c["blank"])
            assert str(exc.value) == c["error"], c["note"]
            continue
        r = galign.forced_align(lp, c["targets"], c["blank"])
        assert r.frame_labels.tolist() == c["labels"], c["note"]
        assert r.frame_scores.tolist() == c["scores"], c["note"]
        assert spans_as_lists(r.spans) == c["spans"], c["note"]


@pytest.mark.gpu
def test_kernel_batch_matches_oracle_on_long_utterances():
    """One launch over ragged utterances (T up to 900, up to ~300 targets)
    against the oracle; batch results equal single-utterance results."""
    rng = np.random.default_rng(7)
    lps, tgs = [], []
    for i in range(24):
        V = 60 if i % 2 else 500
        T = int(rng.integers(50, 900))
        L = int(rng.integers(1, T // 3))
        tg = rng.integers(1, V, size=L)
        logits = rng.normal(0, 1.5, size=(T, V))
        for t in range(T):
            logits[t, 0 if rng.random() < 0.5 else tg[min(L - 1, t * L // T)]] += rng.uniform(3, 8)
        x = logits - logits.max(1, keepdims=True)
        lp = (x - np.log(np.exp(x).sum(1, keepdims=True))).astype(np.float32)
        lps.append(lp)
        tgs.append(tg.tolist())
    for V in (60, 500):
        sel = [i for i in range(24) if lps[i].shape[1] == V]
        res = galign.forced_align_batch([lps[i] for i in sel], [tgs[i] for i in sel])
        for r, i in zip(res, sel):
            ref = oracle.align(lps[i].astype(np.float64), tgs[i])
            assert r.frame_labels.tolist() == ref.tolist(), i
            assert np.array_equal(r.frame_scores, lps[i][np.arange(len(ref)), ref].astype(np.float64))
        single = galign.forced_align(lps[sel[0]], tgs[sel[0]])
        assert single.frame_labels.tolist() == res[0].frame_labels.tolist()


@pytest.mark.gpu
def test_kernel_batch_error_names_utterance():
    lp = np.log(np.full((5, 4), 0.25))
    with pytest.raises(ValueError, match="utterance 1: infeasible alignment: 5 frames cannot fit 4 targets with "
                                         "2 adjacent repeats"):
        galign.forced_align_batch([lp, lp], [[1, 2], [1, 1, 2, 2]])
