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


# ------------------------------------------------------------------ GPU
class _Tokens:
    def __init__(self, tokens, sil=None):
        self.tokens = tuple(tokens)
        self.blank_index = 0
        self.silence_index = sil


def _close(a, b):
    return abs(a - b) <= 1e-9 * (1.0 + abs(b))


@pytest.mark.gpu
def test_fused_kernel_matches_reference_golden():
    """ctcforge-shaped decode with lm= on the fused kernel == the reference's
    n-best (tokens, timesteps exact; score / am_score / lm_score to 1e-9)."""
    from paper_2310_17864_b200 import ctcforge_api as api
    g = golden()
    models = {m["name"]: m for m in g["models"]}
    for k, case in enumerate(g["cases"]):
        m = models[case["model"]]
        lm = load_model(m)
        opts = api.DecoderOptions(**case["opts"])
        res = api.beam_search_decode(np.array(case["lp"]), _Tokens(m["tokens"], case["sil"]), opts, lm=lm)
        exp = case["nbest"]
        assert [h.tokens for h in res] == [h["tokens"] for h in exp], (k, case["model"], case["opts"])
        assert [h.timesteps for h in res] == [h["timesteps"] for h in exp], k
        for h, e in zip(res, exp):
            assert _close(h.score, e["score"]) and _close(h.lm_score, e["lm_score"]), (k, h, e)
            assert _close(h.am_score, e["am_score"]), (k, h, e)


def random_arpa(path, rng, words, order, keep):
    """Seeded synthetic backoff model (our generator, like make_lm_golden.py)."""
    vocab = ["<s>", "</s>"] + list(words)
    tables = {1: {(w,): (-99.0 if w == "<s>" else float(rng.uniform(-2.5, -0.3)),
                         float(rng.uniform(-1.0, 0.3)) if order > 1 else None) for w in vocab}}
    for n in range(2, order + 1):
        tables[n] = {}
        for ctx in list(tables[n - 1]):
            if ctx[-1] == "</s>":
                continue
            for w in vocab[1:]:
                if rng.random() < keep:
                    tables[n][ctx + (w,)] = (float(rng.uniform(-2.2, -0.05)),
                                             float(rng.uniform(-0.9, 0.2)) if n < order else None)
    lines = ["\\data\\"] + [f"ngram {n}={len(tables[n])}" for n in range(1, order + 1)]
    for n in range(1, order + 1):
        lines += ["", f"\\{n}-grams:"]
        for ng, (p, b) in sorted(tables[n].items()):
            lines.append(f"{p:.5f}\t{' '.join(ng)}" + (f"\t{b:.5f}" if b is not None else ""))
    lines += ["", "\\end\\", ""]
    path.write_text("\n".join(lines))
    return glm.parse_arpa(path)


@pytest.mark.gpu
@pytest.mark.parametrize("V,order,beam,T", [(40, 2, 10, 120), (40, 3, 16, 90), (120, 2, 8, 200), (500, 2, 10, 150),
                                            (30, 2, 32, 60), (500, 1, 4, 80)])
def test_fused_kernel_matches_oracle_batches(tmp_path, V, order, beam, T):
    """Batches of ragged utterances through CUCTCDecoder.set_lm against the
    oracle's fused search (same fp32 inputs)."""
    import torch
    from paper_2310_17864_b200 import CUCTCDecoder
    rng = np.random.default_rng(V * 100 + order * 10 + beam)
    toks = ["-"] + [f"w{i}" for i in range(1, V)]
    lm = random_arpa(tmp_path / "m.arpa", rng, toks[1: V - 2], order, keep=min(0.5, 30.0 / V))  # 2 OOV tokens
    B = 12
    lens = rng.integers(1, T + 1, size=B).astype(np.int32)
    x = rng.normal(size=(B, T, V)) * float(rng.choice([1.0, 3.0]))
    x = x - x.max(2, keepdims=True)
    lp = (x - np.log(np.exp(x).sum(2, keepdims=True))).astype(np.float32)
    for w, thr, merge in ((1.3, 0.95, "logadd"), (0.4, 1.0, "max"), (2.5, 0.99, "logadd")):
        dec = CUCTCDecoder(toks, beam_size=beam, nbest=min(beam, 3), blank_skip_threshold=thr, beam_threshold=30.0)
        dec.set_merge_mode(merge)
        dec.set_lm(lm, w)
        out = dec.decode(torch.from_numpy(lp).cuda(), torch.from_numpy(lens).cuda())
        tokens, _, lengths, scores, counts = dec.to_host(out)
        lms = out.lm.cpu().numpy()
        tabs = oracle.lm_tables(glm.flatten(lm), glm.token_words(lm, toks, 0))
        for b in range(B):
            ref = oracle.decode(lp[b, : lens[b]], beam_size=beam, n_best=min(beam, 3), blank_skip_threshold=thr,
                                beam_threshold=30.0, merge_mode=merge, lm=tabs, lm_weight=w)
            got = [tokens[b, j, : lengths[b, j]].tolist() for j in range(counts[b])]
            assert got == ref.tokens, (b, w, thr, merge)
            for j in range(counts[b]):
                assert _close(scores[b, j], ref.scores[j]) and _close(lms[b, j], ref.lm_scores[j]), (b, j)


@pytest.mark.gpu
def test_silence_bonus_without_lm_matches_oracle():
    import torch
    from paper_2310_17864_b200 import CUCTCDecoder
    rng = np.random.default_rng(77)
    V, T, B = 24, 70, 8
    toks = ["-"] + [f"t{i}" for i in range(1, V)]
    lens = rng.integers(1, T + 1, size=B).astype(np.int32)
    x = rng.normal(size=(B, T, V)) * 2.0
    x = x - x.max(2, keepdims=True)
    lp = (x - np.log(np.exp(x).sum(2, keepdims=True))).astype(np.float32)
    for sil_score in (1.5, -0.7):
        dec = CUCTCDecoder(toks, beam_size=12, nbest=2)
        dec.set_silence(V - 1, sil_score)
        out = dec.decode(torch.from_numpy(lp).cuda(), torch.from_numpy(lens).cuda())
        tokens, _, lengths, scores, counts = dec.to_host(out)
        for b in range(B):
            ref = oracle.decode(lp[b, : lens[b]], beam_size=12, n_best=2, blank_skip_threshold=0.95,
                                sil=V - 1, sil_score=sil_score)
            assert [tokens[b, j, : lengths[b, j]].tolist() for j in range(counts[b])] == ref.tokens
            assert all(_close(scores[b, j], ref.scores[j]) for j in range(counts[b]))


@pytest.mark.gpu
def test_fused_errors(tmp_path):
    from paper_2310_17864_b200 import CUCTCDecoder
    rng = np.random.default_rng(3)
    toks = ["-", "a", "b", "c"]
    lm = random_arpa(tmp_path / "e.arpa", rng, toks[1:], 2, 0.5)
    dec = CUCTCDecoder(toks, beam_size=200)
    with pytest.raises(ValueError, match="beam_size <= 128"):
        dec.set_lm(lm, 1.0)
    dec = CUCTCDecoder(toks, beam_size=4)
    with pytest.raises(ValueError, match="silence_index must differ"):
        dec.set_silence(0, 1.0)
    dec.set_lm(lm, 1.0)
    dec.set_lm(None)
    assert dec._lm is None


@pytest.mark.gpu
def test_fused_host_buffer_path_matches_device_path(tmp_path):
    """__call__ with a pinned CPU tensor (ctcb_decode_host_async, chunked) and
    with CUDA tensors give the same LM-fused hypotheses."""
    import torch
    from paper_2310_17864_b200 import CUCTCDecoder
    rng = np.random.default_rng(12)
    V, T, B = 50, 80, 600
    toks = ["-"] + [f"w{i}" for i in range(1, V)]
    lm = random_arpa(tmp_path / "h.arpa", rng, toks[1:], 2, 0.3)
    lens = rng.integers(1, T + 1, size=B).astype(np.int32)
    x = rng.normal(size=(B, T, V)) * 2.0
    x = x - x.max(2, keepdims=True)
    lp = (x - np.log(np.exp(x).sum(2, keepdims=True))).astype(np.float32)
    dec = CUCTCDecoder(toks, beam_size=8, nbest=2)
    dec.set_lm(lm, 1.2)
    dev = dec(torch.from_numpy(lp).cuda(), torch.from_numpy(lens).cuda())
    host = dec(torch.from_numpy(lp).pin_memory(), torch.from_numpy(lens))
    assert dev == host and len(dev) == B


def test_flatten_and_token_words(tmp_path):
    """Device export: n-grams in ascending order with -1 padding, the start
    context, the end word, and the token -> word map (identity for blank and
    silence, <unk> for unknown strings, -1 without <unk>)."""
    p = tmp_path / "f.arpa"
    p.write_text("\\data\\\nngram 1=4\nngram 2=2\n\n\\1-grams:\n-1.0\t<s>\t-0.2\n-0.5\t</s>\n-0.7\ta\t-0.1\n"
                 "-0.9\tb\n\n\\2-grams:\n-0.3\t<s> a\n-0.4\ta b\n\n\\end\\\n")
    lm = glm.parse_arpa(p)
    f = glm.flatten(lm)
    assert f.order == 2 and f.words.shape == (6, 2) and f.lengths.tolist() == [1, 1, 1, 1, 2, 2]
    assert (f.words[:4, 1] == -1).all()
    assert f.start_len == 1 and f.start[0] == lm.vocab["<s>"] and f.eos == lm.vocab["</s>"] and f.unk == -1
    assert f.logprob[4] == -0.3 * glm.LN10 and f.backoff[2] == -0.1 * glm.LN10
    tw = glm.token_words(lm, ["-", "a", "b", "zz", "|"], 0, sil=4)
    assert tw.tolist() == [-2, lm.vocab["a"], lm.vocab["b"], -1, -2]
    p.write_text(p.read_text().replace("ngram 1=4", "ngram 1=5").replace("-0.9\tb\n", "-0.9\tb\n-2.0\t<unk>\n"))
    lm2 = glm.parse_arpa(p)
    assert glm.token_words(lm2, ["-", "zz"], 0).tolist() == [-2, lm2.vocab["<unk>"]]
    assert glm.flatten(lm2).unk == lm2.vocab["<unk>"]
    # a unigram model has the empty start context
    q = tmp_path / "u.arpa"
    q.write_text("\\data\\\nngram 1=2\n\n\\1-grams:\n-1.0\t<s>\n-0.5\ta\n\n\\end\\\n")
    assert glm.flatten(glm.parse_arpa(q)).start_len == 0


@pytest.mark.gpu
def test_fused_kernel_four_gram_model(tmp_path):
    """Order 4 (contexts of three words, deeper backoff chains) against the oracle."""
    import torch
    from paper_2310_17864_b200 import CUCTCDecoder
    rng = np.random.default_rng(404)
    V, T, B = 9, 40, 10
    toks = ["-"] + [f"w{i}" for i in range(1, V)]
    lm = random_arpa(tmp_path / "q.arpa", rng, toks[1:], 4, 0.35)
    assert lm.order == 4
    lens = rng.integers(1, T + 1, size=B).astype(np.int32)
    x = rng.normal(size=(B, T, V)) * 2.0
    x = x - x.max(2, keepdims=True)
    lp = (x - np.log(np.exp(x).sum(2, keepdims=True))).astype(np.float32)
    dec = CUCTCDecoder(toks, beam_size=12, nbest=3, blank_skip_threshold=1.0)
    dec.set_lm(lm, 1.4)
    out = dec.decode(torch.from_numpy(lp).cuda(), torch.from_numpy(lens).cuda())
    tokens, _, lengths, scores, counts = dec.to_host(out)
    lms = out.lm.cpu().numpy()
    tabs = oracle.lm_tables(glm.flatten(lm), glm.token_words(lm, toks, 0))
    for b in range(B):
        ref = oracle.decode(lp[b, : lens[b]], beam_size=12, n_best=3, lm=tabs, lm_weight=1.4)
        assert [tokens[b, j, : lengths[b, j]].tolist() for j in range(counts[b])] == ref.tokens, b
        for j in range(counts[b]):
            assert _close(scores[b, j], ref.scores[j]) and _close(lms[b, j], ref.lm_scores[j])


def test_reader_and_scorer_match_reference_implementation():
    """The ARPA reader / Katz scorer are this repo's own code: cross-check
    them against ctcforge's (from baseline/_ref or /root/reference, when
    present) on every golden model: tables, contexts, scores, bit for bit."""
    import glob
    import sys
    here = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for p in (os.path.join(here, "baseline", "_ref"), "/root/reference/pkg/src"):
        if os.path.isdir(os.path.join(p, "ctcforge")) and p not in sys.path:
            sys.path.append(p)
    rlm = pytest.importorskip("ctcforge.lm")
    files = sorted(glob.glob(os.path.join(GOLD, "*.arpa")))
    assert files
    rng = np.random.default_rng(3)
    for f in files:
        a, b = rlm.parse_arpa(f), glm.parse_arpa(f)
        assert a.order == b.order and a.vocab == b.vocab
        for n in range(1, a.order + 1):
            assert dict(a.tables[n]) == dict(b.tables[n].items())
        words = list(a.vocab) + ["zz-oov"]
        for _ in range(100):
            sa, sb = rlm.lm_start(a), glm.lm_start(b)
            for w in rng.choice(words, size=6):
                sa, x = rlm.lm_score(a, sa, str(w))
                sb, y = glm.lm_score(b, sb, str(w))
                assert x == y and sa.context == sb.context
            assert rlm.lm_finish(a, sa) == glm.lm_finish(b, sb)


@pytest.mark.gpu
@pytest.mark.parametrize("V,beam", [(12, 10), (40, 16), (500, 10)])
def test_fused_kernel_invalid_rows_raise(tmp_path, V, beam):
    """NaN / +inf / positive rows through the LM-fused kernel: the decode
    raises the reference's validation message for the first offender and the
    same decoder then decodes a clean batch (no out-of-range indices)."""
    import torch
    from paper_2310_17864_b200 import cuda_ctc_decoder
    rng = np.random.default_rng(V + beam)
    toks = ["-"] + [f"w{i}" for i in range(1, V)]
    lm = random_arpa(tmp_path / "m.arpa", rng, toks[1:], 2, keep=min(0.5, 30.0 / V))
    B, T = 6, 40
    x = rng.normal(size=(B, T, V)) * 2.0
    lp = (x - np.log(np.exp(x).sum(2, keepdims=True))).astype(np.float32)
    lens = torch.tensor([40, 31, 40, 7, 40, 22], dtype=torch.int32).cuda()
    dec = cuda_ctc_decoder(toks, beam_size=beam, nbest=2, blank_skip_threshold=1.0)
    dec.set_lm(lm, 1.2)
    clean = dec(torch.from_numpy(lp).cuda(), lens)
    bad = lp.copy()
    for b in range(1, B):
        for t in rng.choice(int(lens[b]), size=2, replace=False):
            bad[b, t, rng.integers(0, V, size=3)] = [np.nan, np.inf, 3.0]
    t1 = min(t for t in range(40) if not np.isfinite(bad[1, t]).all())
    with pytest.raises(ValueError, match=f"utterance 1: non-finite log-probability at frame {t1}, token "):
        dec(torch.from_numpy(bad).cuda(), lens)
    again = dec(torch.from_numpy(lp).cuda(), lens)
    assert [[h.tokens for h in g] for g in again] == [[h.tokens for h in g] for g in clean]
