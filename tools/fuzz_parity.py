"""Randomised parity sweep (GPU): random small batches with random options
(beam 1-24, V 3-700, skip threshold, beam threshold incl. small/inf, merge
mode, beam_size_token, peaky/flat/tied rows, ragged lengths) decoded by the
CUDA kernels and by the oracle; reports every mismatch beyond the north-star
tolerances (tokens exact unless the final top-1/top-2 gap <= 1e-3, scores 1e-4).

    python tools/fuzz_parity.py [n_batches] [seed]
"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from paper_2310_17864_b200 import CUCTCDecoder

n_batches = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
only = int(sys.argv[3]) if len(sys.argv) > 3 else None  # replay one iteration (inputs saved to gpurun_out/)
bad = checked = ties = 0
for it in range(n_batches):
    V = int(rng.choice([3, 5, 8, 16, 32, 61, 100, 257, 500, 700]))
    beam = int(rng.integers(1, 25)) if rng.random() < 0.8 else int(rng.integers(17, 70))
    nb = int(rng.integers(1, beam + 1))
    thr = float(rng.choice([1.0, 0.95, 0.8, 0.5]))
    bthr = float(rng.choice([50.0, 5.0, 2.0, np.inf]))
    merge = str(rng.choice(["logadd", "max"]))
    K = None if rng.random() < 0.6 else int(rng.integers(1, V + 1))
    B = int(rng.integers(1, 12))
    T = int(rng.integers(1, 60))
    kind = rng.choice(["peaky", "flat", "ties"])
    lp = np.zeros((B, T, V), np.float32)
    lens = rng.integers(1, T + 1, size=B).astype(np.int32)
    for b in range(B):
        x = rng.normal(0, 1.0 if kind != "flat" else 0.1, size=(T, V))
        if kind == "peaky":
            for t in range(T):
                x[t, 0 if rng.random() < 0.5 else rng.integers(0, V)] += rng.uniform(2, 8)
        if kind == "ties":
            x = np.round(x * 2) / 2
        x = x - x.max(1, keepdims=True)
        lp[b] = (x - np.log(np.exp(x).sum(1, keepdims=True))).astype(np.float32)
    if only is not None:
        if it != only:
            continue
        os.makedirs("gpurun_out", exist_ok=True)
        np.save(f"gpurun_out/fuzz_case_{it}.npy", lp)
        print(dict(V=V, beam=beam, nb=nb, thr=thr, bthr=bthr, merge=merge, K=K, lens=lens.tolist()))
    for force in ("0", "1"):
        os.environ["CTCB_FORCE_GENERIC"] = force  # read when the handle is created
        dec = CUCTCDecoder(["-"] + [f"t{i}" for i in range(1, V)], beam_size=beam, nbest=nb,
                           blank_skip_threshold=thr, beam_threshold=bthr)
        dec.set_merge_mode(merge)
        dec.set_beam_size_token(K)
        try:
            out = dec.decode(torch.from_numpy(lp).cuda(), torch.from_numpy(lens).cuda())
            tok, _, ln, sc, cnt = dec.to_host(out)
            err = None
        except ValueError as e:
            err = str(e)
        for b in range(B):
            try:
                ref = oracle.decode(lp[b, : lens[b]], beam_size=beam, n_best=max(nb, 2) if beam > 1 else 1,
                                    blank_skip_threshold=thr, beam_threshold=bthr, merge_mode=merge, beam_size_token=K)
            except oracle.OracleError as e:
                if err is None or "beam died" not in err:
                    print("MISMATCH died", it, force, b, e, err); bad += 1
                break
            if err is not None:
                print("MISMATCH err", it, force, b, err); bad += 1
                break
            checked += 1
            got_t = [tok[b, j, : ln[b, j]].tolist() for j in range(cnt[b])]
            got_s = [float(sc[b, j]) for j in range(cnt[b])]
            exp_t, exp_s = ref.tokens[:nb], ref.scores[:nb]
            ok = len(got_s) == len(exp_s) and all(abs(a - e) <= 1e-4 for a, e in zip(got_s, exp_s))
            # north-star screen: ranks whose adjacent final gaps are all > 1e-3
            # must carry bit-identical token sequences
            allsc = ref.scores
            for j in range(len(exp_t)):
                if not ok:
                    break
                lo = allsc[j - 1] - allsc[j] if j > 0 else 1.0
                hi = allsc[j] - allsc[j + 1] if j + 1 < len(allsc) else 1.0
                if lo > 1e-3 and hi > 1e-3 and j < len(got_t):
                    ok = got_t[j] == exp_t[j]
            if ok and got_t != exp_t:
                ties += 1
            if not ok:
                bad += 1
                print("MISMATCH", dict(it=it, force=force, b=b, V=V, beam=beam, nb=nb, thr=thr, bthr=bthr, merge=merge,
                                      K=K, kind=str(kind), T=int(lens[b])), got_t[:2], exp_t[:2], got_s[:2], exp_s[:2])
    os.environ.pop("CTCB_FORCE_GENERIC", None)
print(f"checked {checked} utterance decodes, {bad} mismatches, {ties} differ only inside near-tie runs")
