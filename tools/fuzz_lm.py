"""Randomised parity sweep of the fused search (GPU): random token-level LMs
(orders 1-3, <unk> / OOV tokens, random backoffs) and random options (beam
1-128, V 3-600, lm_weight incl. 0 and negative, silence bonus, skip threshold,
beam threshold, merge mode, beam_size_token, peaky / flat / tied rows) decoded
by the fused CUDA kernel and by the oracle; reports every mismatch beyond the
north-star tolerances (tokens exact unless an adjacent final gap <= 1e-3,
scores 1e-4).

    python tools/fuzz_lm.py [n_batches] [seed]
"""
import os
import sys
import tempfile
from pathlib import Path

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_2310_17864_b200 import CUCTCDecoder  # noqa: E402
from paper_2310_17864_b200 import lm as glm  # noqa: E402


def random_model(path, rng, words, order, keep, unk):
    vocab = ["<s>", "</s>"] + list(words) + (["<unk>"] if unk else [])
    tables = {1: {(w,): (-99.0 if w == "<s>" else float(rng.uniform(-3.0, -0.2)),
                         float(rng.uniform(-1.0, 0.4)) if order > 1 else None) for w in vocab}}
    for n in range(2, order + 1):
        tables[n] = {}
        for ctx in list(tables[n - 1]):
            if ctx[-1] == "</s>":
                continue
            for w in vocab[1:]:
                if rng.random() < keep:
                    tables[n][ctx + (w,)] = (float(rng.uniform(-2.5, -0.02)),
                                             float(rng.uniform(-0.9, 0.3)) if n < order else None)
    lines = ["\\data\\"] + [f"ngram {n}={len(tables[n])}" for n in range(1, order + 1)]
    for n in range(1, order + 1):
        lines += ["", f"\\{n}-grams:"]
        for ng, (p, b) in sorted(tables[n].items()):
            lines.append(f"{p:.4f}\t{' '.join(ng)}" + (f"\t{b:.4f}" if b is not None else ""))
    lines += ["", "\\end\\", ""]
    Path(path).write_text("\n".join(lines))
    return glm.parse_arpa(path)


def main():
    n_batches = int(sys.argv[1]) if len(sys.argv) > 1 else 100
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 1)
    only = int(sys.argv[3]) if len(sys.argv) > 3 else None  # replay one iteration
    tmp = tempfile.mkdtemp()
    bad = checked = ties = 0
    for it in range(n_batches):
        V = int(rng.choice([3, 5, 8, 16, 40, 100, 257, 600]))
        order = int(rng.choice([1, 2, 2, 3]))
        beam = int(rng.integers(1, 20)) if rng.random() < 0.8 else int(rng.integers(20, 129))
        nb = int(rng.integers(1, beam + 1))
        thr = float(rng.choice([1.0, 0.95, 0.8]))
        bthr = float(rng.choice([50.0, 8.0, 2.0, np.inf]))
        merge = str(rng.choice(["logadd", "max"]))
        K = None if rng.random() < 0.7 else int(rng.integers(1, V + 1))
        w = float(rng.choice([0.0, 0.3, 1.0, 2.0, 4.0, -0.5]))
        sil = V - 1 if (V > 3 and rng.random() < 0.3) else None
        sil_score = float(rng.choice([0.0, 1.0, -2.0])) if sil is not None else 0.0
        toks = ["-"] + [f"t{i}" for i in range(1, V)]
        n_oov = int(rng.integers(0, 3)) if V > 4 else 0
        words = toks[1: V - n_oov]
        keep = min(0.6, 12.0 / V) if order == 3 else min(0.6, 40.0 / V)
        lm = random_model(os.path.join(tmp, f"m{it}.arpa"), rng, words, order, keep, unk=rng.random() < 0.3)
        B = int(rng.integers(1, 10))
        T = int(rng.integers(1, 50))
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
        if only is not None and it != only:
            continue
        dump = os.environ.get("FUZZ_DUMP")
        if dump and only is not None:  # write the replayed case as a regression fixture and stop
            import json
            import shutil
            shutil.copy(os.path.join(tmp, f"m{it}.arpa"), dump + ".arpa")
            np.save(dump + ".npy", lp)
            Path(dump + ".json").write_text(json.dumps(dict(
                it=it, lens=lens.tolist(), V=V, beam=beam, nb=nb, thr=thr, bthr=bthr if np.isfinite(bthr) else "inf",
                merge=merge, K=K, w=w, sil=sil, sil_score=sil_score, kind=str(kind)), indent=1) + "\n")
            print("dumped", dump)
            return
        dec = CUCTCDecoder(toks, beam_size=beam, nbest=nb, blank_skip_threshold=thr, beam_threshold=bthr)
        dec.set_merge_mode(merge)
        dec.set_beam_size_token(K)
        dec.set_silence(sil, sil_score)
        dec.set_lm(lm, w)
        try:
            out = dec.decode(torch.from_numpy(lp).cuda(), torch.from_numpy(lens).cuda())
            tok, _, ln, sc, cnt = dec.to_host(out)
            lms = out.lm.cpu().numpy()
            err = None
        except (ValueError, RuntimeError) as e:
            err = str(e)
        tabs = oracle.lm_tables(glm.flatten(lm), glm.token_words(lm, toks, 0, sil))
        for b in range(B):
            try:
                ref = oracle.decode(lp[b, : lens[b]], beam_size=beam, n_best=max(nb, 2) if beam > 1 else 1,
                                    blank_skip_threshold=thr, beam_threshold=bthr, merge_mode=merge,
                                    beam_size_token=K, lm=tabs, lm_weight=w, sil=sil, sil_score=sil_score)
            except oracle.OracleError as e:
                if err is None or "beam died" not in err:
                    print("MISMATCH died", it, b, e, err)
                    bad += 1
                break
            if err is not None:
                print("MISMATCH err", it, b, err)
                bad += 1
                break
            checked += 1
            got_t = [tok[b, j, : ln[b, j]].tolist() for j in range(cnt[b])]
            got_s = [float(sc[b, j]) for j in range(cnt[b])]
            got_l = [float(lms[b, j]) for j in range(cnt[b])]
            exp_t, exp_s, exp_l = ref.tokens[:nb], ref.scores[:nb], ref.lm_scores[:nb]
            ok = len(got_s) == len(exp_s) and all(abs(a - e) <= 1e-4 for a, e in zip(got_s, exp_s))
            allsc = ref.scores
            for j in range(len(exp_t)):
                if not ok:
                    break
                lo = allsc[j - 1] - allsc[j] if j > 0 else 1.0
                hi = allsc[j] - allsc[j + 1] if j + 1 < len(allsc) else 1.0
                if lo > 1e-3 and hi > 1e-3 and j < len(got_t):
                    ok = got_t[j] == exp_t[j] and abs(got_l[j] - exp_l[j]) <= 1e-4
            if ok and got_t != exp_t:
                ties += 1
            if not ok:
                bad += 1
                print("MISMATCH", dict(it=it, b=b, V=V, order=order, beam=beam, nb=nb, thr=thr, bthr=bthr,
                                      merge=merge, K=K, w=w, sil=sil, sil_score=sil_score, kind=str(kind),
                                      T=int(lens[b])), got_t[:2], exp_t[:2], got_s[:2], exp_s[:2])
    print(f"checked {checked} utterance decodes, {bad} mismatches, {ties} differ only inside near-tie runs")


if __name__ == "__main__":
    main()
