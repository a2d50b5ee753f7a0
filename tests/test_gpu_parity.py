"""CUDA decoder parity against the reference outputs (golden vectors) and the
C oracle, through the C ABI (paper_2310_17864_b200 -> libctcb.so).

Tolerances (north star): best-path tokens bit-exact on inputs whose final
top-1/top-2 gap exceeds 1e-3; scores within 1e-4 absolute (fp64 device math
typically agrees to ~1e-12); blank-skip frame maps bit-exact.
"""

import dataclasses
import math
import json
import os
import hashlib

import numpy as np
import pytest

torch = pytest.importorskip("torch")

import oracle  # noqa: E402
from paper_2310_17864_b200 import CUCTCDecoder, cuda_ctc_decoder, synth  # noqa: E402

pytestmark = pytest.mark.gpu

SCORE_TOL = 1e-4
NEAR_TIE = 1e-3


def vocab(v):
    return ["-"] + [f"t{i}" for i in range(1, v)]


def run(lp, lens, beam, nbest=1, thr=1.0, bthr=50.0, timesteps=False, merge="logadd", K=None):
    dec = CUCTCDecoder(vocab(lp.shape[2]), beam_size=beam, nbest=nbest, blank_skip_threshold=thr,
                       beam_threshold=bthr)
    dec.set_merge_mode(merge)
    dec.set_beam_size_token(K)
    out = dec.decode(torch.from_numpy(np.ascontiguousarray(lp)).cuda(), torch.from_numpy(np.asarray(lens, np.int32)).cuda(),
                     timesteps=timesteps)
    tokens, ts, lengths, scores, counts = dec.to_host(out)
    res = []
    for b in range(lp.shape[0]):
        n = int(counts[b])
        res.append({
            "tokens": [tokens[b, j, : lengths[b, j]].tolist() for j in range(n)],
            "timesteps": [ts[b, j, : lengths[b, j]].tolist() for j in range(n)] if ts is not None else None,
            "scores": [float(scores[b, j]) for j in range(n)],
        })
    return res


def assert_same(got, exp_tokens, exp_scores, exp_ts=None, gap=None, ctx=""):
    assert len(got["scores"]) == len(exp_scores), ctx
    for a, b in zip(got["scores"], exp_scores):
        assert abs(a - b) <= SCORE_TOL, f"{ctx}: score {a} vs {b}"
    if gap is None or gap > NEAR_TIE:
        assert got["tokens"] == exp_tokens, ctx
        if exp_ts is not None and got["timesteps"] is not None:
            assert got["timesteps"] == exp_ts, ctx


def test_known_answers(golden):
    for case in golden["known"]:
        lp = np.array(case["lp"], dtype=np.float32)[None]
        got = run(lp, [lp.shape[1]], case["beam"], case["n_best"], case["thr"], timesteps=True)[0]
        ref = oracle.decode(lp[0], beam_size=case["beam"], n_best=case["n_best"], blank_skip_threshold=case["thr"])
        assert_same(got, ref.tokens, ref.scores, ref.timesteps, ctx=case["name"])
        # the reference's own answers survive the fp32 cast for these inputs
        assert got["tokens"] == case["tokens"], case["name"]
    one_hot = golden["known"][0]
    lp = np.array(one_hot["lp"], dtype=np.float32)[None]
    got = run(lp, [5], 4, timesteps=True)[0]
    assert got["tokens"][0] == [1, 2, 3] and got["timesteps"][0] == [0, 3, 4] and abs(got["scores"][0]) < 1e-5


def test_small_random_fp32_against_reference(golden):
    for case in golden["small"]:
        if case["merge"] != "logadd" or case["k"] is not None:
            continue
        lp = np.array(case["lp"], dtype=np.float32)[None]
        got = run(lp, [lp.shape[1]], case["beam"], case["n_best"], case["thr"], case["beam_threshold"],
                  timesteps=True)[0]
        if case["dtype"] == "float32":  # golden = ctcforge on these exact fp32 values
            assert_same(got, case["tokens"], case["scores"], case["timesteps"], ctx=f"seed {case['seed']}")
            for a, b in zip(got["scores"], case["scores"]):
                assert abs(a - b) <= 1e-9
        ref = oracle.decode(lp[0], beam_size=case["beam"], n_best=case["n_best"], blank_skip_threshold=case["thr"],
                            beam_threshold=case["beam_threshold"])
        assert_same(got, ref.tokens, ref.scores, ref.timesteps, ctx=f"seed {case['seed']} oracle")


def test_config_shapes_against_reference(golden):
    for case in golden["configs"]:
        cfg = synth.CONFIGS[case["cfg"]]
        n = int(synth.lengths(cfg)[case["b"]])
        x = synth.utterance(cfg, case["b"], n)
        assert hashlib.sha256(x.tobytes()).hexdigest() == case["sha256"], "generator drift"
        got = run(x[None], [n], case["beam"], case["n_best"], case["thr"], timesteps=True)[0]
        assert_same(got, case["tokens"], case["scores"], case["timesteps"], gap=case["gap12"],
                    ctx=f"cfg{case['cfg']} b{case['b']} beam{case['beam']}")


def _batch_vs_oracle(cfg_id, indices=None, beam=None, nbest=None):
    cfg = synth.CONFIGS[cfg_id]
    beam = beam or cfg.beam
    nbest = nbest or (min(beam, 10) if cfg_id == 2 else cfg.nbest)
    lp, lens = synth.batch(cfg, indices=indices)
    got = run(lp, lens, beam, nbest, cfg.threshold)
    full = oracle.decode_batch(lp, lens, beam_size=beam, n_best=min(beam, max(nbest, 2)), blank_skip_threshold=cfg.threshold)
    mism = 0
    for b, (g, r) in enumerate(zip(got, full)):
        gap = r.scores[0] - r.scores[1] if len(r.scores) > 1 else None
        exp_tokens, exp_scores = r.tokens[:nbest], r.scores[:nbest]
        assert len(g["scores"]) == len(exp_scores)
        for a, e in zip(g["scores"], exp_scores):
            assert abs(a - e) <= SCORE_TOL, f"cfg{cfg_id} utt {b}: {a} vs {e}"
        if g["tokens"][0] != exp_tokens[0]:
            assert gap is not None and gap <= NEAR_TIE, f"cfg{cfg_id} utt {b}: top-1 tokens differ (gap {gap})"
            mism += 1
    return mism


def test_cfg0_full_batch():
    assert _batch_vs_oracle(0) == 0


def test_cfg1_full_batch():
    _batch_vs_oracle(1)


@pytest.mark.parametrize("beam", [1, 10, 50, 100])
def test_cfg2_beam_sweep(beam):
    _batch_vs_oracle(2, indices=range(8 if beam >= 50 else 32), beam=beam)


def test_cfg3_large_vocab():
    _batch_vs_oracle(3, indices=range(6))


def test_cfg4_sample():
    _batch_vs_oracle(4, indices=[0, 1, 2, 4093, 4094, 4095])


def test_debug_frames_match_blank_collapse_and_topk():
    for cfg_id in (0, 1, 3):
        cfg = synth.CONFIGS[cfg_id]
        lp, lens = synth.batch(cfg, indices=range(3))
        dec = cuda_ctc_decoder(vocab(cfg.vocab), beam_size=cfg.beam, blank_skip_threshold=cfg.threshold)
        fm, kept, tt, tv, bl = dec.debug_frames(torch.from_numpy(lp).cuda(), torch.from_numpy(lens).cuda())
        fm, kept, tt, tv, bl = (x.cpu().numpy() for x in (fm, kept, tt, tv, bl))
        k = dec.topk
        for b in range(3):
            x = lp[b, : lens[b]]
            ref_fm = oracle.blank_keep(x, cfg.threshold)
            assert kept[b] == len(ref_fm)
            assert fm[b, : kept[b]].tolist() == ref_fm.tolist()
            for i in range(0, kept[b], max(1, kept[b] // 40)):
                row = x[ref_fm[i]]
                order = np.lexsort((np.arange(cfg.vocab), -row.astype(np.float64)))
                order = order[order != 0][:k]
                assert tt[b, i].tolist() == order.tolist()
                assert np.array_equal(tv[b, i], row[order])
                assert bl[b, i] == row[0]


# -- edge cases --------------------------------------------------------------


def test_empty_utterance_raises():
    cfg = synth.CONFIGS[0]
    lp, lens = synth.batch(cfg, indices=range(3))
    lens[1] = 0
    dec = cuda_ctc_decoder(vocab(32))
    with pytest.raises(ValueError, match="utterance 1: empty emissions"):
        dec(torch.from_numpy(lp).cuda(), torch.from_numpy(lens).cuda())


def test_ragged_and_single_frame_lengths():
    cfg = synth.CONFIGS[1]
    lp, lens = synth.batch(cfg, indices=range(6))
    lens = np.array([1, 2, 3, 31, 32, 33], dtype=np.int32)
    got = run(lp, lens, 10, 3, 0.95)
    ref = oracle.decode_batch(lp, lens, beam_size=10, n_best=3, blank_skip_threshold=0.95)
    for g, r in zip(got, ref):
        assert g["tokens"] == r.tokens
        assert np.allclose(g["scores"], r.scores, atol=1e-9, rtol=0)


def test_all_frames_skipped_gives_empty_hypothesis():
    lp = np.log(np.full((1, 4, 3), [0.98, 0.01, 0.01])).astype(np.float32)
    got = run(lp, [4], 10, 1, 0.9)[0]
    assert got["tokens"] == [[]] and got["scores"] == [0.0]


def test_threshold_one_is_identity_and_no_skip():
    cfg = synth.CONFIGS[0]
    lp, lens = synth.batch(cfg, indices=range(2))
    got = run(lp, lens, 10, 2, 1.0)
    ref = oracle.decode_batch(lp, lens, beam_size=10, n_best=2, blank_skip_threshold=1.0)
    for g, r in zip(got, ref):
        assert g["tokens"] == r.tokens and np.allclose(g["scores"], r.scores, atol=1e-9, rtol=0)


def test_batch_permutation_and_determinism():
    cfg = synth.CONFIGS[1]
    lp, lens = synth.batch(cfg, indices=range(12))
    a = run(lp, lens, 10, 2, 0.95)
    b = run(lp, lens, 10, 2, 0.95)
    assert a == b
    perm = np.array([5, 3, 11, 0, 1, 2, 4, 6, 7, 8, 9, 10])
    c = run(lp[perm], lens[perm], 10, 2, 0.95)
    for i, j in enumerate(perm):
        assert c[i] == a[j]


def test_large_beam_exhaustive_small():
    rng = np.random.default_rng(22)
    for _ in range(10):
        t, v = int(rng.integers(1, 5)), int(rng.integers(2, 4))
        x = rng.normal(size=(t, v))
        lp = (x - np.log(np.exp(x).sum(1, keepdims=True))).astype(np.float32)[None]
        got = run(lp, [t], 512, 1, 1.0, float("inf"))[0]
        ref = oracle.decode(lp[0], beam_size=512, n_best=1, beam_threshold=float("inf"))
        assert got["tokens"] == ref.tokens and abs(got["scores"][0] - ref.scores[0]) < 1e-9


def test_uniform_rows_exact_ties():
    lp = np.log(np.full((1, 5, 4), 0.25)).astype(np.float32)
    got = run(lp, [5], 6, 6, 1.0, timesteps=True)[0]
    ref = oracle.decode(lp[0], beam_size=6, n_best=6)
    assert got["tokens"] == ref.tokens and got["timesteps"] == ref.timesteps
    assert np.allclose(got["scores"], ref.scores, atol=1e-12, rtol=0)


def test_argument_errors():
    with pytest.raises(ValueError, match="beam_size must be >= 1"):
        cuda_ctc_decoder(vocab(4), beam_size=0)
    with pytest.raises(ValueError, match="n_best"):
        cuda_ctc_decoder(vocab(4), beam_size=2, nbest=3)
    with pytest.raises(ValueError, match="blank_skip_threshold"):
        cuda_ctc_decoder(vocab(4), blank_skip_threshold=0.0)
    with pytest.raises(ValueError, match="unique"):
        cuda_ctc_decoder(["-", "a", "a"])
    dec = cuda_ctc_decoder(vocab(4))
    with pytest.raises(ValueError, match="columns"):
        dec(torch.zeros((1, 3, 5), device="cuda"), torch.tensor([3], dtype=torch.int32, device="cuda"))
    with pytest.raises(ValueError, match="length out of range"):
        dec(torch.full((1, 3, 4), -1.3862944, device="cuda"), torch.tensor([7], dtype=torch.int32, device="cuda"))


def test_validate_mode_messages():
    lp = np.log(np.full((2, 3, 4), 0.25)).astype(np.float32)
    lp[1, 2, 3] = np.nan
    dec = cuda_ctc_decoder(vocab(4), validate=True)
    with pytest.raises(ValueError, match="utterance 1: non-finite log-probability at frame 2, token 3"):
        dec(torch.from_numpy(lp).cuda(), torch.tensor([3, 3], dtype=torch.int32).cuda())
    lp[1, 2, 3] = np.log(0.25)
    lp[0, 1, 2] = 0.5
    with pytest.raises(ValueError, match="utterance 0: log-probability above 0 at frame 1, token 2"):
        dec(torch.from_numpy(lp).cuda(), torch.tensor([3, 3], dtype=torch.int32).cuda())
    lp[0, 1, 2] = -3.0
    with pytest.raises(ValueError, match="utterance 0: frame 1 is not normalized"):
        dec(torch.from_numpy(lp).cuda(), torch.tensor([3, 3], dtype=torch.int32).cuda())


def test_strided_input_view():
    cfg = synth.CONFIGS[0]
    lp, lens = synth.batch(cfg, indices=range(2))
    big = torch.zeros((2, lp.shape[1] * 2, 32), device="cuda")
    big[:, ::2] = torch.from_numpy(lp).cuda()
    view = big[:, ::2]  # stride_t = 64 elements
    dec = cuda_ctc_decoder(vocab(32))
    got = dec(view, torch.from_numpy(lens).cuda())
    ref = oracle.decode_batch(lp, lens, beam_size=10, n_best=1, blank_skip_threshold=0.95)
    assert [[h.tokens for h in g] for g in got] == [r.tokens for r in ref]


def test_fast_and_generic_kernels_agree(monkeypatch):
    """beam <= 16 runs the register-resident fast kernel; CTCB_FORCE_GENERIC=1
    forces the generic one.  Both must give identical results."""
    cases = []
    for cfg_id, idx in ((0, range(4)), (1, range(24)), (3, range(3))):
        cfg = synth.CONFIGS[cfg_id]
        lp, lens = synth.batch(cfg, indices=idx)
        for beam, nb in ((cfg.beam, cfg.nbest), (1, 1), (16, 16)):
            cases.append((lp, lens, beam, nb, cfg.threshold))
    fast = [run(lp, lens, beam, nb, thr, timesteps=True) for lp, lens, beam, nb, thr in cases]
    monkeypatch.setenv("CTCB_FORCE_GENERIC", "1")
    gen = [run(lp, lens, beam, nb, thr, timesteps=True) for lp, lens, beam, nb, thr in cases]
    for a, b in zip(fast, gen):
        for x, y in zip(a, b):
            assert x["tokens"] == y["tokens"] and x["timesteps"] == y["timesteps"]
            assert np.allclose(x["scores"], y["scores"], atol=1e-9, rtol=0)


def test_fused_and_precomputed_topk_modes_agree(monkeypatch):
    """Small batches precompute the top-k of every frame in a frame-parallel
    kernel; large batches fuse it into the beam walk.  Both must agree."""
    cases = []
    for cfg_id, idx in ((0, range(4)), (1, range(16)), (3, range(2))):
        cfg = synth.CONFIGS[cfg_id]
        lp, lens = synth.batch(cfg, indices=idx)
        cases.append((lp, lens, cfg.beam, cfg.nbest, cfg.threshold))
    # V > 512: rows read from global memory (V % 4 == 0) or staged (odd V);
    # a column of exact ties exercises the radix fallback
    rng = np.random.default_rng(52)
    for V in (1000, 1001):
        x = rng.normal(size=(3, 60, V)) * 2.0
        x[:, 7, :] = 0.0
        x = x - x.max(2, keepdims=True)
        lp = (x - np.log(np.exp(x).sum(2, keepdims=True))).astype(np.float32)
        cases.append((lp, np.array([60, 41, 9], dtype=np.int32), 10, 3, 0.95))
    monkeypatch.setenv("CTCB_TOPK_MODE", "precomp")
    pre = [run(lp, lens, beam, nb, thr, timesteps=True) for lp, lens, beam, nb, thr in cases]
    monkeypatch.setenv("CTCB_TOPK_STAGED", "1")
    staged = [run(lp, lens, beam, nb, thr, timesteps=True) for lp, lens, beam, nb, thr in cases]
    monkeypatch.delenv("CTCB_TOPK_STAGED")
    monkeypatch.setenv("CTCB_TOPK_MODE", "fused")
    fus = [run(lp, lens, beam, nb, thr, timesteps=True) for lp, lens, beam, nb, thr in cases]
    assert pre == fus and staged == fus
    for (lp, lens, beam, nb, thr), got in zip(cases[-2:], pre[-2:]):
        for b in range(lp.shape[0]):
            ref = oracle.decode(lp[b, : lens[b]], beam_size=beam, n_best=nb, blank_skip_threshold=thr)
            assert [g for g in got[b]["tokens"]] == ref.tokens


def test_host_buffer_path_matches_device_path():
    """ctcb_decode_host (CPU tensors, valid frames copied) == device path."""
    cfg = synth.CONFIGS[1]
    lp, lens = synth.batch(cfg, indices=range(12))
    dec = cuda_ctc_decoder(vocab(cfg.vocab), nbest=3, beam_size=10, blank_skip_threshold=cfg.threshold)
    dev = dec(torch.from_numpy(lp).cuda(), torch.from_numpy(lens).cuda())
    host = dec(torch.from_numpy(lp).pin_memory(), torch.from_numpy(lens))
    assert dev == host
    lens2 = lens.copy()
    lens2[3] = 0
    with pytest.raises(ValueError, match="utterance 3: empty emissions"):
        dec(torch.from_numpy(lp), torch.from_numpy(lens2))


def test_host_buffer_chunked_pipeline():
    """The pipelined host path (ctcb_decode_host_async, several utterance ranges)
    == device path, and an error in a later range names the right utterance."""
    cfg = dataclasses.replace(synth.CONFIGS[0], batch=600)
    lp, lens = synth.batch(cfg)
    dec = cuda_ctc_decoder(vocab(cfg.vocab), nbest=2, beam_size=10, blank_skip_threshold=cfg.threshold)
    dev = dec(torch.from_numpy(lp).cuda(), torch.from_numpy(lens).cuda())
    host = dec(torch.from_numpy(lp).pin_memory(), torch.from_numpy(lens))
    assert len(host) == 600 and dev == host
    lens2 = lens.copy()
    lens2[450] = 0
    with pytest.raises(ValueError, match="utterance 450: empty emissions"):
        dec(torch.from_numpy(lp), torch.from_numpy(lens2))
    # the handle is reusable after the error
    assert dec(torch.from_numpy(lp).pin_memory(), torch.from_numpy(lens)) == dev


def test_multi_device_decoder_matches_single():
    """MultiDeviceDecoder (consecutive length-balanced ranges, one decoder and
    stream per entry of ``devices``; [0, 0, 0] runs three on one GPU) ==
    the single-device decoder for CPU (pinned and pageable) and CUDA inputs;
    errors name the utterance's index in the whole batch."""
    from paper_2310_17864_b200 import MultiDeviceDecoder
    cfg = dataclasses.replace(synth.CONFIGS[0], batch=700)
    lp, lens = synth.batch(cfg)
    single = cuda_ctc_decoder(vocab(cfg.vocab), nbest=2, beam_size=10, blank_skip_threshold=cfg.threshold)
    ref = single(torch.from_numpy(lp).cuda(), torch.from_numpy(lens).cuda())
    multi = MultiDeviceDecoder(vocab(cfg.vocab), devices=[0, 0, 0], nbest=2, beam_size=10,
                               blank_skip_threshold=cfg.threshold)
    assert multi(torch.from_numpy(lp).pin_memory(), torch.from_numpy(lens)) == ref
    assert len(multi.last_ranges) == 3 and all(b1 > b0 for b0, b1 in multi.last_ranges)
    assert multi(torch.from_numpy(lp), torch.from_numpy(lens)) == ref
    assert multi(torch.from_numpy(lp).cuda(), torch.from_numpy(lens).cuda()) == ref
    lens2 = lens.copy()
    b_err = multi.last_ranges[2][0] + 5
    lens2[b_err] = 0
    for x in (torch.from_numpy(lp), torch.from_numpy(lp).cuda()):
        with pytest.raises(ValueError, match=f"utterance {b_err}: empty emissions"):
            multi(x, torch.from_numpy(lens2))
    assert multi(torch.from_numpy(lp).pin_memory(), torch.from_numpy(lens)) == ref
    # options reach every device's decoder
    multi.set_merge_mode("max")
    single.set_merge_mode("max")
    assert multi(torch.from_numpy(lp).cuda(), torch.from_numpy(lens).cuda()) == \
        single(torch.from_numpy(lp).cuda(), torch.from_numpy(lens).cuda())
    multi.set_silence(cfg.vocab - 1, 0.5)
    single.set_silence(cfg.vocab - 1, 0.5)
    assert multi(torch.from_numpy(lp).pin_memory(), torch.from_numpy(lens)) == \
        single(torch.from_numpy(lp).cuda(), torch.from_numpy(lens).cuda())


def test_multi_device_decoder_side_stream_producer():
    """Input produced on a side stream (delayed by a device-side sleep) and
    decoded from that stream: every range's decoder -- including those run
    on worker threads, whose current stream is the default one -- must wait
    for the producer (thread-local current streams)."""
    from paper_2310_17864_b200 import MultiDeviceDecoder
    cfg = dataclasses.replace(synth.CONFIGS[0], batch=300)
    lp, lens = synth.batch(cfg)
    src = torch.from_numpy(lp).cuda()
    lens_d = torch.from_numpy(lens).cuda()
    single = cuda_ctc_decoder(vocab(cfg.vocab), nbest=2, beam_size=10, blank_skip_threshold=cfg.threshold)
    ref = single(src, lens_d)
    multi = MultiDeviceDecoder(vocab(cfg.vocab), devices=[0, 0, 0], nbest=2, beam_size=10,
                               blank_skip_threshold=cfg.threshold)
    side = torch.cuda.Stream()
    for _ in range(3):
        with torch.cuda.stream(side):
            dst = torch.zeros_like(src)
            torch.cuda._sleep(20_000_000)
            dst.copy_(src)
            got = multi(dst, lens_d)
        assert got == ref


@pytest.mark.parametrize("force_generic", ["0", "1"])
def test_merge_mode_max_matches_oracle(monkeypatch, force_generic):
    """merge_mode="max" (decoder.py:610-613, :789-791) on both kernels against the
    oracle (fp32 inputs): the golden fp64 max-merge cases rounded to fp32, and
    config-shaped batches."""
    monkeypatch.setenv("CTCB_FORCE_GENERIC", force_generic)
    g = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "golden.json")))
    for c in [c for c in g["small"] if c["merge"] == "max"]:
        lp = np.array(c["lp"], dtype=np.float32)[None]
        thr = c["beam_threshold"]
        thr = np.inf if thr == "inf" else thr
        ref = oracle.decode(lp[0], beam_size=c["beam"], n_best=c["n_best"], blank_skip_threshold=c["thr"],
                            beam_threshold=thr, merge_mode="max")
        got = run(lp, [lp.shape[1]], c["beam"], c["n_best"], c["thr"], thr, timesteps=True, merge="max")[0]
        assert_same(got, ref.tokens, ref.scores, ref.timesteps, ctx=f"seed {c['seed']}")
    for cfg_id, idx in ((0, range(4)), (1, range(8))):
        cfg = synth.CONFIGS[cfg_id]
        lp, lens = synth.batch(cfg, indices=idx)
        got = run(lp, lens, cfg.beam, 3, cfg.threshold, merge="max")
        for b in range(len(lens)):
            ref = oracle.decode(lp[b, : lens[b]], beam_size=cfg.beam, n_best=3, blank_skip_threshold=cfg.threshold,
                                merge_mode="max")
            assert_same(got[b], ref.tokens, ref.scores, ctx=f"cfg{cfg_id} utt {b}")


@pytest.mark.parametrize("force_generic", ["0", "1"])
def test_beam_size_token_matches_oracle(monkeypatch, force_generic):
    """beam_size_token = K < V (decoder.py:440-458) on both kernels against the
    oracle: K below, at and above the kept top-k size (k = 2 beam), so the
    selected tokens are a prefix of the top-k list or need the K-th key of the
    whole row; blank selected or not; a repeat's token selected or not."""
    monkeypatch.setenv("CTCB_FORCE_GENERIC", force_generic)
    plans = ((0, range(4), 10, (1, 2, 5, 19, 20, 21, 25, 31, 32)), (1, range(6), 10, (3, 15, 21, 60, 499)),
             (1, range(3), 16, (7, 31, 32, 33, 40)), (3, range(2), 10, (4, 20, 22, 200)))
    for cfg_id, idx, beam, Ks in plans:
        cfg = synth.CONFIGS[cfg_id]
        lp, lens = synth.batch(cfg, indices=idx)
        nb = min(3, beam)
        for K in Ks:
            got = run(lp, lens, beam, nb, cfg.threshold, timesteps=True, K=K)
            for b in range(len(lens)):
                ref = oracle.decode(lp[b, : lens[b]], beam_size=beam, n_best=nb, blank_skip_threshold=cfg.threshold,
                                    beam_size_token=K)
                assert_same(got[b], ref.tokens, ref.scores, ref.timesteps, ctx=f"cfg{cfg_id} beam {beam} K {K} utt {b}")
    # K == V is the full vocabulary
    cfg = synth.CONFIGS[0]
    lp, lens = synth.batch(cfg)
    assert run(lp, lens, 10, 2, cfg.threshold, K=cfg.vocab) == run(lp, lens, 10, 2, cfg.threshold)


@pytest.mark.parametrize("force_generic", ["0", "1"])
def test_regression_short_append_lists(monkeypatch, force_generic):
    """Found by tools/fuzz_parity.py: V=5, beam 8, beam_size_token 3 leaves
    append lists shorter than the beam, where the one-shot selection's
    dominance count does not hold; the kernel must fall back to the exact
    merge (the candidate [2, 1] was dropped at the second kept frame)."""
    monkeypatch.setenv("CTCB_FORCE_GENERIC", force_generic)
    u = np.load(os.path.join(os.path.dirname(__file__), "golden", "regress_short_lists.npy"))
    for T in (7, u.shape[0]):
        for K in (3, None):
            got = run(u[None, :T], [T], 8, 8, 0.8, timesteps=True, K=K)[0]
            ref = oracle.decode(u[:T], beam_size=8, n_best=8, blank_skip_threshold=0.8, beam_size_token=K)
            assert_same(got, ref.tokens, ref.scores, ref.timesteps, ctx=f"T {T} K {K}")


def test_regression_threshold_tie_libm_rounding():
    """Quantized logits put a candidate exactly at best - beam_threshold; the
    generic kernel's logaddexp reproduces libm's rounding (guarded
    double-double), so its keep / drop decision matches the reference."""
    lp = np.load(os.path.join(os.path.dirname(__file__), "golden", "regress_threshold_688.npy"))
    u = lp[1, :10]
    got = run(u[None], [10], 62, 31, 0.8, 2.0, timesteps=True)[0]
    ref = oracle.decode(u, beam_size=62, n_best=31, blank_skip_threshold=0.8, beam_threshold=2.0)
    assert got["tokens"] == ref.tokens
    assert got["scores"] == ref.scores


# ---------------------------------------------------------------- headline path
# The bench decodes B = 4096 > 10 x SMs utterances, which selects the fused
# one-warp-per-utterance kernel (top-k inside the beam walk); the small-batch
# tests above run the precomputed-top-k kernels.  These decode full batches
# through the exact kernel and mode the headline number comes from and compare
# every utterance with the oracle (decoder.py:102-170 restated).

def _full_vs_oracle(lp, lens, beam, nbest, thr, expect_kernel=None):
    dec = CUCTCDecoder(vocab(lp.shape[2]), beam_size=beam, nbest=nbest, blank_skip_threshold=thr)
    dec.kernel_timing(True)
    out = dec.decode(torch.from_numpy(np.ascontiguousarray(lp)).cuda(), torch.from_numpy(lens).cuda())
    tokens, _, lengths, scores, counts = dec.to_host(out)
    _, _, kname = dec.kernel_time()
    if expect_kernel is not None:
        assert kname == expect_kernel, kname
    ref = oracle.decode_batch(lp, lens, beam_size=beam, n_best=min(beam, max(nbest, 2)), blank_skip_threshold=thr)
    near = 0
    for b, r in enumerate(ref):
        n = int(counts[b])
        exp_t, exp_s = r.tokens[:nbest], r.scores[:nbest]
        assert n == len(exp_s), f"utt {b}: {n} hypotheses vs {len(exp_s)}"
        for j in range(n):
            assert abs(float(scores[b, j]) - exp_s[j]) <= SCORE_TOL, f"utt {b} rank {j}"
        got_t = [tokens[b, j, : lengths[b, j]].tolist() for j in range(n)]
        if got_t != exp_t:
            gap = r.scores[0] - r.scores[1] if len(r.scores) > 1 else None
            assert gap is not None and gap <= NEAR_TIE, f"utt {b}: tokens differ (top-1/top-2 gap {gap})"
            near += 1
    return near


def test_cfg4_headline_kernel_512(monkeypatch):
    """512 cfg4 utterances (every 8th of the 4096, all lengths) in one call
    through ctcb_decode_fast_small_kernel, the benchmarked kernel (selected
    for B > 10 x SMs; forced here so the test stays small)."""
    monkeypatch.setenv("CTCB_TOPK_MODE", "fused")
    cfg = synth.CONFIGS[4]
    lp, lens = synth.batch(cfg, indices=range(0, 4096, 8))
    near = _full_vs_oracle(lp, lens, cfg.beam, cfg.nbest, cfg.threshold, "ctcb_decode_fast_small_kernel")
    assert near <= 5


@pytest.mark.parametrize("beam", [1, 10])
def test_cfg2_full_batch(beam):
    cfg = synth.CONFIGS[2]
    lp, lens = synth.batch(cfg)
    _full_vs_oracle(lp, lens, beam, min(beam, 10), cfg.threshold)


def test_cfg3_full_batch():
    cfg = synth.CONFIGS[3]
    lp, lens = synth.batch(cfg)
    _full_vs_oracle(lp, lens, cfg.beam, cfg.nbest, cfg.threshold)


# ---------------------------------------------------------------- known ulp-level cases
# Both cases need exactly tied scores in quantized inputs.  The kernels'
# logaddexp rounds log1p(exp(-d)) with a polynomial (ctcb_common.cuh), glibc
# (numpy, the reference) with its own rounding, so an exact fp64 tie can land
# one ulp apart and reorder hypotheses INSIDE the tie.  Within the north-star
# tolerances (tokens exact only where adjacent gaps exceed 1e-3, scores 1e-4)
# both decodes agree; the bitwise ranking checks are expected failures.

def _rank_ok(got, ref, nb):
    """north-star comparison: scores 1e-4, tokens exact where both adjacent
    final gaps of the reference exceed 1e-3"""
    if len(got["scores"]) != len(ref.scores[:nb]):
        return False
    for a, e in zip(got["scores"], ref.scores[:nb]):
        if abs(a - e) > SCORE_TOL:
            return False
    allsc = ref.scores
    for j in range(len(got["tokens"])):
        lo = allsc[j - 1] - allsc[j] if j > 0 else 1.0
        hi = allsc[j] - allsc[j + 1] if j + 1 < len(allsc) else 1.0
        if lo > NEAR_TIE and hi > NEAR_TIE and got["tokens"][j] != ref.tokens[j]:
            return False
    return True


def _beam39_case():
    u = np.load(os.path.join(os.path.dirname(__file__), "golden", "regress_ties_beam39.npy"))
    got = run(u[None], [u.shape[0]], 39, 39, 1.0, 5.0)[0]
    ref = oracle.decode(u, beam_size=39, n_best=39, blank_skip_threshold=1.0, beam_threshold=5.0)
    return got, ref


def test_regression_ties_beam39_tolerant():
    got, ref = _beam39_case()
    assert _rank_ok(got, ref, 39)


@pytest.mark.xfail(reason="3-way exact fp64 tie at ranks 27-29: device logaddexp lands one ulp from glibc's",
                   strict=False)
def test_regression_ties_beam39_bitwise():
    got, ref = _beam39_case()
    assert got["tokens"] == ref.tokens and got["scores"] == ref.scores


def _token_k_ties_case():
    """fuzz_parity seed 202 iteration 461 (utterance 6): V = 3 quantized rows
    with exact ties, beam_size_token = 2, skip threshold 0.8, no beam
    threshold.  At frame 9 two hypotheses tie to ~1e-15; the device
    logaddexp orders them one ulp differently from glibc, and the beams
    diverge afterwards (best path tokens equal, score -11.25 vs -10.42)."""
    x = np.load(os.path.join(os.path.dirname(__file__), "golden", "regress_token_k_ties.npy"))
    got = run(x[None], [x.shape[0]], 10, 10, 0.8, math.inf, K=2)[0]
    ref = oracle.decode(x, beam_size=10, n_best=10, blank_skip_threshold=0.8, beam_threshold=math.inf,
                        beam_size_token=2)
    return got, ref


def test_regression_token_k_ties_best_path():
    got, ref = _token_k_ties_case()
    assert got["tokens"][0] == ref.tokens[0]


@pytest.mark.xfail(reason="exact score tie at frame 9 ordered one ulp apart; the beams diverge later",
                   strict=False)
def test_regression_token_k_ties_bitwise():
    got, ref = _token_k_ties_case()
    assert got["tokens"] == ref.tokens and got["scores"] == ref.scores


def _lm602_case():
    import json
    from paper_2310_17864_b200 import lm as glm
    base = os.path.join(os.path.dirname(__file__), "golden", "regress_lm_s62_602")
    meta = json.load(open(base + ".json"))
    lp = np.load(base + ".npy")
    lens = np.array(meta["lens"], np.int32)
    toks = ["-"] + [f"t{i}" for i in range(1, meta["V"])]
    lm = glm.parse_arpa(base + ".arpa")
    bthr = math.inf if meta["bthr"] == "inf" else meta["bthr"]
    dec = CUCTCDecoder(toks, beam_size=meta["beam"], nbest=meta["nb"], blank_skip_threshold=meta["thr"],
                       beam_threshold=bthr)
    dec.set_lm(lm, meta["w"])
    out = dec.decode(torch.from_numpy(lp).cuda(), torch.from_numpy(lens).cuda())
    tok, _, ln, sc, cnt = dec.to_host(out)
    tabs = oracle.lm_tables(glm.flatten(lm), glm.token_words(lm, toks, 0, None))
    res = []
    for b in range(len(lens)):
        ref = oracle.decode(lp[b, : lens[b]], beam_size=meta["beam"], n_best=meta["nb"],
                            blank_skip_threshold=meta["thr"], beam_threshold=bthr, lm=tabs, lm_weight=meta["w"])
        got = {"tokens": [tok[b, j, : ln[b, j]].tolist() for j in range(cnt[b])],
               "scores": [float(sc[b, j]) for j in range(cnt[b])]}
        res.append((got, ref))
    return res, meta["nb"]


def test_regression_lm_fuzz_s62_602_tolerant():
    """tools/fuzz_lm.py seed 62 iteration 602 (V=3, beam 25, quantized rows,
    bigram-free unigram model with weight 0.3), replayed with FUZZ_DUMP."""
    res, nb = _lm602_case()
    bad = [b for b, (g, r) in enumerate(res) if not _rank_ok(g, r, nb)]
    assert not bad, bad


@pytest.mark.xfail(reason="exact score ties in quantized rows: one-ulp logaddexp differences reorder tied ranks",
                   strict=False)
def test_regression_lm_fuzz_s62_602_bitwise():
    res, nb = _lm602_case()
    for g, r in res:
        assert g["tokens"] == r.tokens[:nb] and g["scores"] == r.scores[:nb]


# ---------------------------------------------------------------- large-beam block kernel
# 16 < beam <= 128 (no token cap, no LM) runs one 256-thread CTA per
# utterance (ctcb_block.cu).  Quantized logits give exact in-frame score ties,
# and small vocabularies give fewer live candidates than beam slots: both
# exercise the tie-run resolution and the serial exact fallback.
@pytest.mark.parametrize("V,beam,quant", [(5, 17, 1.0), (5, 62, 0.5), (12, 40, 1.0), (12, 100, 0.5),
                                          (30, 128, 1.0), (64, 50, 0.0)])
def test_block_kernel_ties_small_vocab(V, beam, quant, monkeypatch):
    """Block kernel vs the oracle (north-star tolerance: scores 1e-4, ranks
    exact outside 1e-3 near-ties) and vs the one-warp generic kernel (bitwise:
    both fold scores with the same fp64 helpers)."""
    rng = np.random.default_rng(V * 1000 + beam)
    B, T = 6, 24
    x = rng.normal(size=(B, T, V)) * 2.0
    if quant:
        x = np.round(x / quant) * quant
    lp = (x - np.log(np.exp(x).sum(-1, keepdims=True))).astype(np.float32)
    lens = rng.integers(1, T + 1, size=B).astype(np.int32)
    nb = min(beam, 8)

    def dec_run():
        dec = CUCTCDecoder(vocab(V), beam_size=beam, nbest=nb, blank_skip_threshold=0.9, beam_threshold=8.0)
        dec.kernel_timing(True)
        out = dec.decode(torch.from_numpy(lp).cuda(), torch.from_numpy(lens).cuda(), timesteps=True)
        return dec.to_host(out), dec.kernel_time()[2]

    (tok, ts, ln, sc, cnt), name = dec_run()
    assert name == "ctcb_decode_block_kernel"
    monkeypatch.setenv("CTCB_BLOCK", "0")
    (tok2, ts2, ln2, sc2, cnt2), name2 = dec_run()
    assert name2 != "ctcb_decode_block_kernel"
    assert np.array_equal(cnt, cnt2)
    for b in range(B):
        ref = oracle.decode(lp[b, : lens[b]], beam_size=beam, n_best=nb, blank_skip_threshold=0.9, beam_threshold=8.0)
        n = int(cnt[b])
        got = {"tokens": [tok[b, j, : ln[b, j]].tolist() for j in range(n)],
               "scores": [float(sc[b, j]) for j in range(n)]}
        assert _rank_ok(got, ref, nb), (b, got, ref.tokens, ref.scores)
        for j in range(n):
            assert sc[b, j] == sc2[b, j] and ln[b, j] == ln2[b, j], (b, j)
            assert np.array_equal(tok[b, j, : ln[b, j]], tok2[b, j, : ln[b, j]]), (b, j)
            assert np.array_equal(ts[b, j, : ln[b, j]], ts2[b, j, : ln[b, j]]), (b, j)


# ---------------------------------------------------------------- fused input validation
def _val_batch(V=12, B=4, T=20, seed=5):
    rng = np.random.default_rng(seed)
    x = rng.normal(size=(B, T, V))
    return (x - np.log(np.exp(x).sum(-1, keepdims=True))).astype(np.float32)


@pytest.mark.parametrize("beam,env", [(10, None), (32, None), (10, "CTCB_FORCE_GENERIC"), (4, "CTCB_TOPK_MODE")])
def test_fused_validation_default(beam, env, monkeypatch):
    """Validation is on by default and fused into the decode kernels (fast,
    block) or done after them (generic); each case raises the reference's
    message for the first invalid utterance (emissions.py:128-150 run by
    decode_batch in utterance order)."""
    if env == "CTCB_TOPK_MODE":
        monkeypatch.setenv(env, "fused")
    elif env:
        monkeypatch.setenv(env, "1")
    V = 12
    dec = cuda_ctc_decoder(vocab(V), beam_size=beam, nbest=1, blank_skip_threshold=0.9)
    lens = torch.tensor([20, 20, 15, 20], dtype=torch.int32).cuda()
    lp = _val_batch(V)
    got = dec(torch.from_numpy(lp).cuda(), lens)  # clean batch decodes
    assert len(got) == 4
    bad = lp.copy()
    bad[2, 14, 5] = np.nan
    bad[1, 3, 7] = 0.5
    bad[3, 17, 2] = np.nan
    with pytest.raises(ValueError, match=r"utterance 1: log-probability above 0 at frame 3, token 7: 0\.5"):
        dec(torch.from_numpy(bad).cuda(), lens)
    bad[1, 3, 7] = np.log(0.01)  # utterance 1 now unnormalized (strict)
    with pytest.raises(ValueError, match=r"utterance 1: frame 3 is not normalized"):
        dec(torch.from_numpy(bad).cuda(), lens)
    bad[1, 3] = lp[1, 3]
    with pytest.raises(ValueError, match=r"utterance 2: non-finite log-probability at frame 14, token 5"):
        dec(torch.from_numpy(bad).cuda(), lens)
    bad[2, 14] = lp[2, 14]
    bad[2, 16, 4] = np.nan  # beyond lens[2] = 15: not checked (frames t >= len are padding)
    with pytest.raises(ValueError, match=r"utterance 3: non-finite log-probability at frame 17, token 2"):
        dec(torch.from_numpy(bad).cuda(), lens)
    bad[3, 17] = lp[3, 17]
    # a blank-skipped frame (blank prob 0.95 >= 0.9) is never staged by the
    # decode kernel: the follow-up pass checks it
    row = np.full(V, np.log(0.05 / (V - 1)), dtype=np.float32)
    row[0] = np.log(0.95)
    bad[0, 9] = row
    bad[0, 9, 6] = -np.inf
    with pytest.raises(ValueError, match=r"utterance 0: non-finite log-probability at frame 9, token 6"):
        dec(torch.from_numpy(bad).cuda(), lens)
    dec.set_validate(False)
    dec(torch.from_numpy(bad).cuda(), lens)  # decodes (garbage in, no error)
    dec.set_validate("nonstrict")
    bad[0, 9] = row
    bad[0, 9, 6] = np.log(0.5)  # unnormalized only: passes without the norm check
    dec(torch.from_numpy(bad).cuda(), lens)


def test_fused_validation_host_path():
    V = 12
    dec = cuda_ctc_decoder(vocab(V), beam_size=10, nbest=1)
    lp = _val_batch(V)
    lp[2, 4, 1] = np.inf
    with pytest.raises(ValueError, match=r"utterance 2: non-finite log-probability at frame 4, token 1"):
        dec(torch.from_numpy(lp), torch.tensor([20, 20, 20, 20], dtype=torch.int32))


# ---------------------------------------------------------------- overlapped precomputed top-k
# Precomputed mode runs ctcb_topk_kernel either before the walk or beside it
# (frame-major lists published through per-list ready flags, the walk launched
# as its programmatic dependent; CTCB_OVERLAP=1 forces it, 0 disables it).
# Both schedules must give bit-identical decodes, equal to the oracle.

def _overlap_cases():
    cases = []
    cfg = synth.CONFIGS[1]
    lp, lens = synth.batch(cfg)  # V = 500: staged rows
    cases.append(("cfg1", lp, lens, cfg.beam, cfg.nbest, cfg.threshold, 64))
    cfg = synth.CONFIGS[3]
    lp, lens = synth.batch(cfg, indices=range(24))  # V = 5000: rows from global memory
    cases.append(("cfg3", lp, lens, cfg.beam, cfg.nbest, cfg.threshold, 6))
    rng = np.random.default_rng(77)  # odd V > 512: staged, unaligned rows
    x = rng.normal(size=(5, 90, 1001)) * 2.0
    x = x - x.max(2, keepdims=True)
    lp = (x - np.log(np.exp(x).sum(2, keepdims=True))).astype(np.float32)
    cases.append(("v1001", lp, np.array([90, 3, 47, 1, 88], dtype=np.int32), 10, 3, 0.95, 5))
    return cases


@pytest.mark.parametrize("case", [0, 1, 2])
def test_overlapped_topk_matches_sequential_and_oracle(monkeypatch, case):
    name, lp, lens, beam, nb, thr, n_oracle = _overlap_cases()[case]
    monkeypatch.setenv("CTCB_TOPK_MODE", "precomp")
    monkeypatch.setenv("CTCB_OVERLAP", "1")
    ov = run(lp, lens, beam, nb, thr, timesteps=True)
    ov2 = run(lp, lens, beam, nb, thr, timesteps=True)
    monkeypatch.setenv("CTCB_OVERLAP", "0")
    seq = run(lp, lens, beam, nb, thr, timesteps=True)
    assert ov == seq, name
    assert ov2 == seq, f"{name}: overlapped decode not deterministic"
    ref = oracle.decode_batch(lp[:n_oracle], lens[:n_oracle], beam_size=beam, n_best=max(nb, 2),
                              blank_skip_threshold=thr)
    for b, r in enumerate(ref):
        gap = r.scores[0] - r.scores[1] if len(r.scores) > 1 else None
        assert_same(ov[b], r.tokens[:nb], r.scores[:nb], gap=gap, ctx=f"{name} utt {b}")


def test_overlapped_topk_validation_messages(monkeypatch):
    """validation keys written by the overlapped top-k reach the host check"""
    monkeypatch.setenv("CTCB_TOPK_MODE", "precomp")
    monkeypatch.setenv("CTCB_OVERLAP", "1")
    cfg = synth.CONFIGS[3]
    lp, lens = synth.batch(cfg, indices=range(8))
    lp[5, 11, 123] = np.nan
    dec = cuda_ctc_decoder(vocab(cfg.vocab), beam_size=cfg.beam, blank_skip_threshold=1.0, validate=True)
    with pytest.raises(ValueError, match="utterance 5: non-finite log-probability at frame 11, token 123"):
        dec(torch.from_numpy(lp).cuda(), torch.from_numpy(lens).cuda())


@pytest.mark.parametrize("beam", [50, 100])
def test_overlapped_block_topk_matches_sequential_and_oracle(monkeypatch, beam):
    """block kernel (16 < beam <= 128): ctcb_topk_wide_kernel beside the walk"""
    cfg = synth.CONFIGS[2]
    lp, lens = synth.batch(cfg, indices=range(12))
    monkeypatch.setenv("CTCB_OVERLAP", "1")
    ov = run(lp, lens, beam, 10, cfg.threshold, timesteps=True)
    monkeypatch.setenv("CTCB_OVERLAP", "0")
    seq = run(lp, lens, beam, 10, cfg.threshold, timesteps=True)
    assert ov == seq
    ref = oracle.decode_batch(lp[:3], lens[:3], beam_size=beam, n_best=10, blank_skip_threshold=cfg.threshold)
    for b, r in enumerate(ref):
        gap = r.scores[0] - r.scores[1] if len(r.scores) > 1 else None
        assert_same(ov[b], r.tokens[:10], r.scores[:10], gap=gap, ctx=f"beam {beam} utt {b}")


@pytest.mark.parametrize("beam,V,overlap", [(10, 12, "0"), (10, 12, "1"), (10, 1000, "1"), (32, 12, "0"),
                                            (32, 12, "1"), (50, 500, "1"), (10, 12, "fused"), (10, 500, "fused"),
                                            (10, 1000, "fused"), (10, 12, "generic"), (24, 12, "inline")])
def test_precomputed_modes_never_walk_invalid_rows(monkeypatch, beam, V, overlap):
    """Rows with NaN / +inf / positive log-probs in every utterance: the
    precomputed-mode walks (fast and block kernels, lists before or beside the
    walk) stop at the top-k kernel's offender key instead of walking non-finite
    scores; the decode raises the reference's message for the first invalid
    utterance, and the same decoder then decodes a clean batch."""
    # (also the in-kernel top-k schedules: fused fast kernel, generic kernel,
    # block kernel with its inline top-k)
    if overlap == "fused":
        monkeypatch.setenv("CTCB_TOPK_MODE", "fused")
    elif overlap == "generic":
        monkeypatch.setenv("CTCB_FORCE_GENERIC", "1")
    elif overlap == "inline":
        monkeypatch.setenv("CTCB_BLOCK_TOPK", "inline")
    else:
        monkeypatch.setenv("CTCB_TOPK_MODE", "precomp")
        monkeypatch.setenv("CTCB_OVERLAP", overlap)
    rng = np.random.default_rng(beam * 7 + V)
    B, T = 8, 40
    x = rng.normal(size=(B, T, V)) * 2.0
    lp = (x - np.log(np.exp(x).sum(-1, keepdims=True))).astype(np.float32)
    lens = torch.tensor([40, 33, 40, 5, 40, 21, 40, 40], dtype=torch.int32).cuda()
    dec = cuda_ctc_decoder(vocab(V), beam_size=beam, nbest=1, blank_skip_threshold=1.0)
    clean = dec(torch.from_numpy(lp).cuda(), lens)
    bad = lp.copy()
    for b in range(B):
        for t in rng.choice(min(int(lens[b]), 40), size=2, replace=False):
            bad[b, t, rng.integers(0, V, size=3)] = [np.nan, np.inf, 3.0]
    bad[0, :, :] = lp[0]  # utterance 0 clean: utterance 1 is the first offender
    t1 = min(t for t in range(40) if not np.isfinite(bad[1, t]).all() or (bad[1, t] > 1e-4).any())
    with pytest.raises(ValueError, match=f"utterance 1: non-finite log-probability at frame {t1}, token "):
        dec(torch.from_numpy(bad).cuda(), lens)
    again = dec(torch.from_numpy(lp).cuda(), lens)
    assert [[h.tokens for h in g] for g in again] == [[h.tokens for h in g] for g in clean]
