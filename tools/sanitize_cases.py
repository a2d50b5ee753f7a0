"""Small decodes through every device kernel, for compute-sanitizer
(memcheck / racecheck / synccheck; tools/gpu_sanitize.sh).

    python tools/sanitize_cases.py [case ...]

Cases: fast_fused (ctcb_decode_fast_small_kernel, cfg0 + 12 cfg1 utterances),
fast_pre (framemap / rowoff / topk / fast_pre_small), fast_general (V=700, the
non-SMALL layout), generic (CTCB_FORCE_GENERIC), block (beam 50: topk_wide +
block kernel), block_inline, lm (fused LM kernel), align, validate (a row that
fails EmissionMatrix's checks).  Every decode is compared with the C oracle
(tokens exact, scores 1e-6) so a sanitizer run also checks the results.
"""
import os
import sys
import tempfile

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402
from paper_2310_17864_b200 import CUCTCDecoder, synth  # noqa: E402
from paper_2310_17864_b200 import align as galign  # noqa: E402
from paper_2310_17864_b200 import lm as glm  # noqa: E402


def small_batch(cfg_id, n, t_cap):
    cfg = synth.CONFIGS[cfg_id]
    lens = np.minimum(synth.lengths(cfg)[:n], t_cap).astype(np.int32)
    T = int(lens.max())
    lp = np.zeros((n, T, cfg.vocab), np.float32)
    for b in range(n):
        lp[b, : lens[b]] = synth.utterance(cfg, b, int(lens[b]))
    return cfg, lp, lens


def rand_batch(seed, B, T, V, scale=2.0):
    rng = np.random.default_rng(seed)
    lens = rng.integers(1, T + 1, size=B).astype(np.int32)
    x = rng.normal(size=(B, T, V)) * scale
    x = x - x.max(2, keepdims=True)
    return (x - np.log(np.exp(x).sum(2, keepdims=True))).astype(np.float32), lens


def check(name, dec, lp, lens, beam, nbest, thr, **okw):
    out = dec.decode(torch.from_numpy(lp).cuda(), torch.from_numpy(lens).cuda())
    tokens, _, lengths, scores, counts = dec.to_host(out)
    ref = oracle.decode_batch(lp, lens, beam_size=beam, n_best=nbest, blank_skip_threshold=thr, **okw)
    for b, r in enumerate(ref):
        got = [tokens[b, j, : lengths[b, j]].tolist() for j in range(counts[b])]
        assert got == r.tokens, (name, b)
        assert np.allclose(scores[b, : counts[b]], r.scores, rtol=0, atol=1e-6), (name, b)
    print(f"{name}: {len(ref)} utterances match the oracle", flush=True)


def case_fast_fused():
    os.environ["CTCB_TOPK_MODE"] = "fused"
    for cid, n, cap in ((0, 4, 200), (1, 12, 160)):
        cfg, lp, lens = small_batch(cid, n, cap)
        dec = CUCTCDecoder(synth.simple_tokens(cfg.vocab), beam_size=cfg.beam, nbest=2,
                           blank_skip_threshold=cfg.threshold)
        check(f"fast_fused cfg{cid}", dec, lp, lens, cfg.beam, 2, cfg.threshold)
    del os.environ["CTCB_TOPK_MODE"]


def case_fast_pre():
    os.environ["CTCB_TOPK_MODE"] = "precomp"
    cfg, lp, lens = small_batch(1, 12, 160)
    dec = CUCTCDecoder(synth.simple_tokens(cfg.vocab), beam_size=10, nbest=3, blank_skip_threshold=0.95)
    check("fast_pre cfg1", dec, lp, lens, 10, 3, 0.95)
    del os.environ["CTCB_TOPK_MODE"]


def case_fast_general():
    lp, lens = rand_batch(5, 6, 60, 700)
    dec = CUCTCDecoder(["-"] + [f"t{i}" for i in range(1, 700)], beam_size=8, nbest=2, blank_skip_threshold=0.9)
    check("fast_general V=700", dec, lp, lens, 8, 2, 0.9)


def case_generic():
    os.environ["CTCB_FORCE_GENERIC"] = "1"
    lp, lens = rand_batch(6, 6, 60, 40)
    dec = CUCTCDecoder(["-"] + [f"t{i}" for i in range(1, 40)], beam_size=24, nbest=3)
    check("generic beam 24", dec, lp, lens, 24, 3, 1.0)
    del os.environ["CTCB_FORCE_GENERIC"]


def case_block(inline=False):
    if inline:
        os.environ["CTCB_BLOCK_TOPK"] = "inline"
    cfg, lp, lens = small_batch(2, 6, 120)
    dec = CUCTCDecoder(synth.simple_tokens(cfg.vocab), beam_size=50, nbest=5, blank_skip_threshold=0.95)
    check("block beam 50" + (" inline" if inline else ""), dec, lp, lens, 50, 5, 0.95)
    os.environ.pop("CTCB_BLOCK_TOPK", None)


def case_lm():
    V = 40
    toks = ["-"] + [f"w{i}" for i in range(1, V)]
    p = tempfile.mktemp(suffix=".arpa")
    with open(p, "w") as f:
        f.write("\\data\\\nngram 1=6\nngram 2=3\n\n\\1-grams:\n-99\t<s>\t-0.3\n-1.0\t</s>\n-0.7\tw1\t-0.2\n"
                "-1.2\tw2\t-0.4\n-1.5\tw3\t-0.1\n-0.9\tw4\n\n\\2-grams:\n-0.3\t<s> w1\n-0.5\tw1 w2\n-0.4\tw2 w3\n\n"
                "\\end\\\n")
    lm = glm.parse_arpa(p)
    lp, lens = rand_batch(7, 6, 50, V)
    dec = CUCTCDecoder(toks, beam_size=10, nbest=2, beam_threshold=30.0)
    dec.set_lm(lm, 1.3)
    out = dec.decode(torch.from_numpy(lp).cuda(), torch.from_numpy(lens).cuda())
    tokens, _, lengths, scores, counts = dec.to_host(out)
    tabs = oracle.lm_tables(glm.flatten(lm), glm.token_words(lm, toks, 0))
    for b in range(len(lens)):
        ref = oracle.decode(lp[b, : lens[b]], beam_size=10, n_best=2, beam_threshold=30.0, lm=tabs, lm_weight=1.3)
        got = [tokens[b, j, : lengths[b, j]].tolist() for j in range(counts[b])]
        assert got == ref.tokens, ("lm", b)
    print("lm: 6 utterances match the oracle", flush=True)


def case_align():
    rng = np.random.default_rng(9)
    lps, tgs = [], []
    for _ in range(5):
        T = int(rng.integers(20, 60))
        x = rng.normal(size=(T, 30)) * 2.0
        lps.append((x - np.log(np.exp(x).sum(1, keepdims=True))).astype(np.float32))
        tgs.append(rng.integers(1, 30, size=int(rng.integers(1, T // 3))).tolist())
    res = galign.forced_align_batch(lps, tgs)
    for r, lp, tg in zip(res, lps, tgs):
        assert list(r.frame_labels) == list(oracle.align(lp.astype(np.float64), tg)), "align"
    print("align: 5 utterances match the oracle", flush=True)


def case_validate():
    cfg, lp, lens = small_batch(0, 4, 200)
    lp[1, 7, 3] = np.nan
    dec = CUCTCDecoder(synth.simple_tokens(cfg.vocab), beam_size=10, nbest=1, blank_skip_threshold=0.95)
    try:
        dec(torch.from_numpy(lp).cuda(), torch.from_numpy(lens).cuda())
    except ValueError as e:
        print(f"validate: raised {e}", flush=True)
    else:
        raise AssertionError("validate: NaN row decoded")


CASES = {"fast_fused": case_fast_fused, "fast_pre": case_fast_pre, "fast_general": case_fast_general,
         "generic": case_generic, "block": case_block, "block_inline": lambda: case_block(True), "lm": case_lm,
         "align": case_align, "validate": case_validate}

if __name__ == "__main__":
    for name in sys.argv[1:] or list(CASES):
        CASES[name]()
    torch.cuda.synchronize()
    print("all cases done")
