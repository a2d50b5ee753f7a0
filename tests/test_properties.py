"""Size-independent properties of the CUDA decoder, mirroring the reference's
own behavioural tests (ctcforge tests/test_decoder.py: greedy equivalence at
beam 1 with max merge, the exhaustive CTC path-sum at unbounded beam, n-best
ordering, max-merge beam monotonicity, batch-of-one and permutation
invariance) with independent checkers written here (greedy collapse and an
exhaustive enumeration of all frame paths).  The last test covers the edge
sizes (V = 2, T = 4000) against the oracle."""

import itertools

import numpy as np
import pytest

torch = pytest.importorskip("torch")

from paper_2310_17864_b200 import CUCTCDecoder  # noqa: E402

pytestmark = pytest.mark.gpu


def vocab(v):
    return ["-"] + [f"t{i}" for i in range(1, v)]


def logsoftmax32(x):
    x = x - x.max(-1, keepdims=True)
    return (x - np.log(np.exp(x).sum(-1, keepdims=True))).astype(np.float32)


def decode(lp, beam, nbest=1, merge="logadd", thr=1.0, bthr=50.0):
    dec = CUCTCDecoder(vocab(lp.shape[-1]), beam_size=beam, nbest=nbest, blank_skip_threshold=thr,
                       beam_threshold=bthr)
    dec.set_merge_mode(merge)
    x = torch.from_numpy(np.ascontiguousarray(lp[None])).cuda()
    out = dec.decode(x, torch.tensor([lp.shape[0]], dtype=torch.int32).cuda(), timesteps=True)
    tok, ts, ln, sc, cnt = dec.to_host(out)
    return [(tok[0, j, : ln[0, j]].tolist(), float(sc[0, j]), ts[0, j, : ln[0, j]].tolist()) for j in range(cnt[0])]


def greedy(lp):
    best = lp.argmax(1)
    out, prev = [], -1
    for c in best:
        if c != prev and c != 0:
            out.append(int(c))
        prev = c
    return out


def collapse(path):
    out, prev = [], -1
    for c in path:
        if c != prev and c != 0:
            out.append(c)
        prev = c
    return tuple(out)


def exhaustive_totals(lp):
    """log Σ over frame paths of exp(Σ lp) per collapsed label sequence."""
    T, V = lp.shape
    acc = {}
    lp64 = lp.astype(np.float64)
    for path in itertools.product(range(V), repeat=T):
        s = float(sum(lp64[t, c] for t, c in enumerate(path)))
        k = collapse(path)
        acc[k] = np.logaddexp(acc[k], s) if k in acc else s
    return acc


def test_beam1_max_merge_is_greedy():
    rng = np.random.default_rng(21)
    for _ in range(60):
        T, V = int(rng.integers(1, 15)), int(rng.choice([3, 5, 40]))
        lp = logsoftmax32(rng.normal(size=(T, V)))
        assert decode(lp, 1, merge="max")[0][0] == greedy(lp)


def test_unbounded_beam_is_the_exhaustive_path_sum():
    rng = np.random.default_rng(22)
    for _ in range(25):
        T, V = int(rng.integers(1, 6)), int(rng.integers(2, 4))
        lp = logsoftmax32(rng.normal(size=(T, V)))
        totals = exhaustive_totals(lp)
        best = max(totals.values())
        toks, score, _ = decode(lp, 512, bthr=float("inf"))[0]
        assert score == pytest.approx(best, abs=1e-9)
        assert totals[tuple(toks)] == pytest.approx(best, abs=1e-9)


def test_nbest_sorted_distinct_and_bounded():
    rng = np.random.default_rng(23)
    for _ in range(20):
        lp = logsoftmax32(rng.normal(size=(int(rng.integers(2, 30)), 6)))
        res = decode(lp, 8, nbest=5)
        assert 1 <= len(res) <= 5
        scores = [s for _, s, _ in res]
        assert all(a >= b for a, b in zip(scores, scores[1:]))
        assert len({tuple(t) for t, _, _ in res}) == len(res)
        for toks, _, ts in res:
            assert len(ts) == len(toks) and ts == sorted(ts) and len(set(ts)) == len(ts)


def test_max_merge_top_score_monotone_in_beam():
    rng = np.random.default_rng(34)
    for _ in range(25):
        lp = logsoftmax32(rng.normal(size=(8, 4)))
        prev = -np.inf
        for beam in (1, 2, 4, 8, 16):
            top = decode(lp, beam, merge="max", bthr=float("inf"))[0][1]
            assert top >= prev - 1e-12
            prev = top


def test_timesteps_are_original_frames_after_skipping():
    """Timesteps index the original frames (frame_map), not kept frames."""
    T, V = 9, 4
    p = np.full((T, V), 0.01)
    path = [0, 0, 1, 0, 0, 2, 2, 0, 3]
    p[np.arange(T), path] = 0.97
    lp = np.log(p / p.sum(1, keepdims=True)).astype(np.float32)
    toks, _, ts = decode(lp, 4, thr=0.95)[0]
    assert toks == [1, 2, 3] and ts == [2, 5, 8]


def test_batch_of_one_equals_batch_member():
    rng = np.random.default_rng(9)
    lp = logsoftmax32(rng.normal(size=(5, 40, 12)) * 2)
    lens = np.array([40, 17, 1, 33, 25], dtype=np.int32)
    dec = CUCTCDecoder(vocab(12), beam_size=6, nbest=3)
    out = dec.decode(torch.from_numpy(lp).cuda(), torch.from_numpy(lens).cuda())
    tok, _, ln, sc, cnt = dec.to_host(out)
    for b in range(5):
        single = decode(lp[b, : lens[b]], 6, nbest=3, thr=0.95)
        assert [t for t, _, _ in single] == [tok[b, j, : ln[b, j]].tolist() for j in range(cnt[b])]
        assert [s for _, s, _ in single] == [float(sc[b, j]) for j in range(cnt[b])]


def test_two_token_vocabulary_and_long_utterances():
    """V = 2 (blank + one token; top-k of 1) on both kernels, and T = 4000
    frames (long trellis walks) against the oracle."""
    import oracle
    rng = np.random.default_rng(41)
    for beam in (1, 2, 4, 20):
        lp = logsoftmax32(rng.normal(size=(30, 2)) * 2)
        got = decode(lp, beam, nbest=min(beam, 2), thr=0.95)
        ref = oracle.decode(lp, beam_size=beam, n_best=min(beam, 2), blank_skip_threshold=0.95)
        assert [t for t, _, _ in got] == ref.tokens and np.allclose([s for _, s, _ in got], ref.scores, atol=1e-9)
    lp = logsoftmax32(rng.normal(size=(4000, 24)) * 3)
    for beam in (10, 24):
        got = decode(lp, beam, nbest=3, thr=0.95)
        ref = oracle.decode(lp, beam_size=beam, n_best=3, blank_skip_threshold=0.95)
        assert [t for t, _, _ in got] == ref.tokens
        assert np.allclose([s for _, s, _ in got], ref.scores, rtol=0, atol=1e-6)
        assert [ts for _, _, ts in got] == ref.timesteps
