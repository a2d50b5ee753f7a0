"""Token-level LM fusion: the ARPA reader and incremental API,
the oracle's fused search against the reference's golden n-best (CPU), and the
CUDA fused kernel against both (GPU).  Golden vectors:
tests/golden/make_lm_golden.py."""

import json
import math
import os

import numpy as np
import pytest

import oracle
from paper_2310_17864_b200 import lm as glm

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "lm")


def golden():
    with open(os.path.join(GOLD, "lm_decode.json"), encoding="utf-8") as fh:
        return json.load(fh)


def load_model(m):
    return glm.parse_arpa(os.path.join(GOLD, m["file"]))


def oracle_decode(case, model, tokens):
    o = case["opts"]
    lm = load_model(model)
    tw = glm.token_words(lm, tokens, 0, case["sil"])
    tabs = oracle.lm_tables(glm.flatten(lm), tw)
    return oracle.decode(np.array(case["lp"]), beam_size=o["beam_size"], n_best=o["n_best"],
                         blank_skip_threshold=o["blank_skip_threshold"], beam_threshold=o["beam_threshold"],
                         beam_size_token=o.get("beam_size_token"), merge_mode=o["merge_mode"], lm=tabs,
                         lm_weight=o["lm_weight"], sil=case["sil"], sil_score=o.get("sil_score", 0.0))


# ------------------------------------------------------------------ CPU
def test_arpa_reader_and_incremental_api_match_reference():
    g = golden()
    for m in g["models"]:
        lm = load_model(m)
        for s in m["api"]:
            st = glm.lm_start(lm)
            for w, want in zip(s["words"], s["scores"]):
                st, got = glm.lm_score(lm, st, w)
                assert got == want, (m["name"], s)
            assert st.cumulative_score == s["total"]
            assert glm.lm_finish(lm, st) == s["finish"]


def test_arpa_errors(tmp_path):
    def write(text):
        p = tmp_path / "x.arpa"
        p.write_text(text)
        return p

    with pytest.raises(glm.ArpaFormatError, match="missing \\\\data\\\\ header"):
        glm.parse_arpa(write("hello\n"))
    with pytest.raises(glm.ArpaFormatError, match="declares 2 1-grams, file has 1"):
        glm.parse_arpa(write("\\data\\\nngram 1=2\n\n\\1-grams:\n-1.0\ta\n\\end\\\n"))
    with pytest.raises(glm.ArpaFormatError, match="line 4: malformed 1-gram line"):
        glm.parse_arpa(write("\\data\\\nngram 1=1\n\\1-grams:\n-1.0\ta\tb\tc\n\\end\\\n"))
    with pytest.raises(glm.ArpaFormatError, match="missing \\\\end\\\\"):
        glm.parse_arpa(write("\\data\\\nngram 1=1\n\\1-grams:\n-1.0\ta\n"))
    with pytest.raises(glm.ArpaFormatError, match="content after"):
        glm.parse_arpa(write("\\data\\\nngram 1=1\n\\1-grams:\n-1.0\ta\n\\end\\\n-1.0\tb\n"))
    with pytest.raises(glm.ArpaFormatError, match="no lower-order context entry"):
        glm.parse_arpa(os.path.join(GOLD, "trigram_pruned_v7.arpa"), strict=True)
    with pytest.raises(glm.ArpaFormatError, match="line 5: malformed 1-gram line"):  # backoff at the top order
        glm.parse_arpa(write("\\data\\\nngram 1=2\n\\1-grams:\n-1.0\ta\n-2.0\tb\t-0.5\n\\end\\\n"))
    lm = glm.parse_arpa(write("\\data\\\nngram 1=2\nngram 2=1\n\\1-grams:\n-1.0\ta\n-2.0\tb\t-0.5\n"
                              "\\2-grams:\n-0.3\ta b\n\\end\\\n"))
    assert lm.tables[1][(0,)] == (-1.0 * glm.LN10, 0.0)
    assert lm.tables[1][(1,)] == (-2.0 * glm.LN10, -0.5 * glm.LN10)
    assert glm.lm_score(lm, glm.lm_start(lm), "zz")[1] == glm.OOV_PENALTY


def test_oracle_fusion_matches_reference_golden():
    g = golden()
    models = {m["name"]: m for m in g["models"]}
    n = 0
    for case in g["cases"]:
        m = models[case["model"]]
        res = oracle_decode(case, m, m["tokens"])
        exp = case["nbest"]
        assert res.tokens == [h["tokens"] for h in exp], case["model"]
        assert res.timesteps == [h["timesteps"] for h in exp]
        assert res.scores == [h["score"] for h in exp]
        assert res.lm_scores == [h["lm_score"] for h in exp]
        n += 1
    assert n == len(g["cases"]) >= 40


def test_oracle_tables_are_the_incremental_api():
    """Dense (context x token) rows equal lm_score along random paths."""
    g = golden()
    rng = np.random.default_rng(5)
    for m in g["models"]:
        lm = load_model(m)
        toks = m["tokens"]
        tabs = oracle.lm_tables(glm.flatten(lm), glm.token_words(lm, toks, 0))
        for _ in range(5):
            st, s = glm.lm_start(lm), tabs.start
            for c in rng.integers(1, len(toks), size=6):
                st, want = glm.lm_score(lm, st, toks[c])
                assert tabs.score[s, c] == want
                s = tabs.next[s, c]
            assert tabs.fin[s] == glm.lm_finish(lm, st)
