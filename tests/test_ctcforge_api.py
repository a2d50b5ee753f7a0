"""The ctcforge-shaped GPU entry points against the reference's
own outputs (golden vectors), with full Hypothesis fields incl. timesteps."""

import numpy as np
import pytest

from paper_2310_17864_b200.ctcforge_api import DecoderOptions


def test_options_validation_matches_reference():
    # decoder.py:54-66 (test_decoder.py:314-324)
    for kw, msg in (({"beam_size": 0}, "beam_size"), ({"n_best": 5, "beam_size": 2}, "n_best"),
                    ({"blank_skip_threshold": 0.0}, "blank_skip_threshold"), ({"merge_mode": "sum"}, "merge_mode"),
                    ({"beam_threshold": 0.0}, "beam_threshold")):
        with pytest.raises(ValueError, match=msg):
            DecoderOptions(**kw)


@pytest.mark.gpu
def test_shim_matches_reference_golden(golden):
    from paper_2310_17864_b200.ctcforge_api import beam_search_decode, decode_batch

    cases = [c for c in golden["small"] if c["dtype"] == "float32" and c["k"] is None]
    assert cases
    for c in cases:
        lp = np.array(c["lp"], dtype=np.float64)
        v = lp.shape[1]
        tokens = ["-"] + [f"t{i}" for i in range(1, v)]
        opts = DecoderOptions(beam_size=c["beam"], n_best=c["n_best"], blank_skip_threshold=c["thr"],
                              beam_threshold=c["beam_threshold"], merge_mode=c["merge"])
        nb = beam_search_decode(lp, tokens, opts)
        assert [h.tokens for h in nb] == c["tokens"]
        assert [h.timesteps for h in nb] == c["timesteps"]
        for h, s in zip(nb, c["scores"]):
            assert h.score == pytest.approx(s, abs=1e-9)
            assert h.am_score == h.score and h.lm_score == 0.0 and h.words == []
    # batch == per-utterance, order preserved
    lps = [np.array(c["lp"], dtype=np.float64) for c in cases if len(c["lp"][0]) == 5][:6]
    if lps:
        tokens = ["-"] + [f"t{i}" for i in range(1, 5)]
        opts = DecoderOptions(beam_size=4, n_best=2)
        batch = decode_batch(lps, tokens, opts)
        single = [beam_search_decode(lp, tokens, opts) for lp in lps]
        assert [[h.tokens for h in x] for x in batch] == [[h.tokens for h in x] for x in single]


@pytest.mark.gpu
def test_shim_merge_max_matches_oracle(golden):
    """merge_mode="max" through the shim against the oracle on fp32-rounded inputs
    (the golden max-merge cases are fp64; the decoder's input dtype is fp32)."""
    import oracle
    from paper_2310_17864_b200.ctcforge_api import beam_search_decode

    for c in [c for c in golden["small"] if c["merge"] == "max"][:12]:
        lp = np.array(c["lp"], dtype=np.float32).astype(np.float64)
        tokens = ["-"] + [f"t{i}" for i in range(1, lp.shape[1])]
        opts = DecoderOptions(beam_size=c["beam"], n_best=c["n_best"], blank_skip_threshold=c["thr"],
                              beam_threshold=c["beam_threshold"], merge_mode="max")
        nb = beam_search_decode(lp, tokens, opts)
        ref = oracle.decode(lp, beam_size=c["beam"], n_best=c["n_best"], blank_skip_threshold=c["thr"],
                            beam_threshold=c["beam_threshold"], merge_mode="max")
        assert [h.tokens for h in nb] == ref.tokens and [h.timesteps for h in nb] == ref.timesteps
        assert np.allclose([h.score for h in nb], ref.scores, atol=1e-9, rtol=0)


@pytest.mark.gpu
def test_shim_beam_size_token_matches_reference_golden(golden):
    """beam_size_token < V through the shim against the oracle on fp32-rounded
    golden inputs (the golden K=2 cases are fp64)."""
    import oracle
    from paper_2310_17864_b200.ctcforge_api import beam_search_decode

    cases = [c for c in golden["small"] if c["k"] is not None]
    assert cases
    for c in cases:
        lp = np.array(c["lp"], dtype=np.float32).astype(np.float64)
        tokens = ["-"] + [f"t{i}" for i in range(1, lp.shape[1])]
        opts = DecoderOptions(beam_size=c["beam"], n_best=c["n_best"], blank_skip_threshold=c["thr"],
                              beam_threshold=c["beam_threshold"], beam_size_token=c["k"], merge_mode=c["merge"])
        try:
            ref = oracle.decode(lp, beam_size=c["beam"], n_best=c["n_best"], blank_skip_threshold=c["thr"],
                                beam_threshold=c["beam_threshold"], beam_size_token=c["k"], merge_mode=c["merge"])
        except oracle.OracleError as exc:
            with pytest.raises(ValueError, match="beam died"):
                beam_search_decode(lp, tokens, opts)
            assert "beam died" in str(exc)
            continue
        nb = beam_search_decode(lp, tokens, opts)
        assert [h.tokens for h in nb] == ref.tokens and [h.timesteps for h in nb] == ref.timesteps
        assert np.allclose([h.score for h in nb], ref.scores, atol=1e-9, rtol=0)


@pytest.mark.gpu
def test_shim_errors():
    from paper_2310_17864_b200.ctcforge_api import beam_search_decode, decode_batch

    tokens = ["-", "a", "b"]
    with pytest.raises(ValueError, match="empty"):
        beam_search_decode(np.zeros((0, 3)), tokens)
    with pytest.raises(ValueError, match="columns"):
        beam_search_decode(np.log(np.full((2, 4), 0.25)), tokens)
    with pytest.raises(ValueError, match="^beam_size_token 4 exceeds vocabulary size 3$"):
        beam_search_decode(np.log(np.full((2, 3), 1 / 3)), tokens, DecoderOptions(beam_size_token=4))
    good = np.log(np.full((3, 3), 1 / 3))
    with pytest.raises(ValueError, match="utterance 1: empty emissions"):
        decode_batch([good, np.zeros((0, 3))], tokens)
