"""Token-level LM fusion throughput on the cfg4 / cfg1 workloads.

A seeded synthetic backoff model over the V=500 token strings (orders 2 and 3,
``--keep`` successors per context) is attached with ``CUCTCDecoder.set_lm``;
the fused kernel decodes the resident batch (CUDA events), and the oracle's
fused search (C restatement of ctcforge decoder.py with lm=) decodes a bounded
sample on all host cores.  One JSON line per (order, lm_weight).

    python tools/bench_lm.py [--workload cfg4] [--steps 5] [--orders 2,3] [--weights 0.5,2.0]
"""
import argparse
import json
import os
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2310_17864_b200 import lm as glm  # noqa: E402
from paper_2310_17864_b200 import synth  # noqa: E402


def synthetic_lm(path, tokens, order, per_ctx, seed=7):
    """Backoff model: every token a unigram; `per_ctx` successors per context."""
    rng = np.random.default_rng(seed)
    vocab = ["<s>", "</s>"] + list(tokens)
    tables = {1: {(w,): (-99.0 if w == "<s>" else float(rng.uniform(-3.5, -1.5)),
                         float(rng.uniform(-0.8, 0.0)) if order > 1 else None) for w in vocab}}
    for n in range(2, order + 1):
        tables[n] = {}
        ctxs = [c for c in tables[n - 1] if c[-1] != "</s>"]
        if n == 3:
            ctxs = [ctxs[i] for i in rng.permutation(len(ctxs))[: len(ctxs) // 4]]
        for ctx in ctxs:
            for j in rng.choice(len(vocab) - 1, size=per_ctx, replace=False):
                w = vocab[1 + j]
                tables[n][ctx + (w,)] = (float(rng.uniform(-2.5, -0.1)),
                                         float(rng.uniform(-0.6, 0.0)) if n < order else None)
    lines = ["\\data\\"] + [f"ngram {n}={len(tables[n])}" for n in range(1, order + 1)]
    for n in range(1, order + 1):
        lines += ["", f"\\{n}-grams:"]
        for ng, (p, b) in tables[n].items():
            lines.append(f"{p:.4f}\t{' '.join(ng)}" + (f"\t{b:.4f}" if b is not None else ""))
    lines += ["", "\\end\\", ""]
    with open(path, "w") as fh:
        fh.write("\n".join(lines))
    return glm.parse_arpa(path)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg4", choices=["cfg4", "cfg1", "cfg3"])
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--orders", default="2,3")
    ap.add_argument("--weights", default="0.5,2.0")
    ap.add_argument("--keep", type=int, default=20)
    ap.add_argument("--cpu-budget", type=float, default=10.0)
    args = ap.parse_args()
    import torch

    import oracle
    from paper_2310_17864_b200 import CUCTCDecoder

    cfg = synth.CONFIGS[int(args.workload[3:])]
    toks = synth.simple_tokens(cfg.vocab)
    lens_all = synth.lengths(cfg)
    T = int(lens_all.max())
    host = np.zeros((cfg.batch, T, cfg.vocab), np.float32)
    _, lens = synth.batch(cfg, out=host, t_pad=T, threads=os.cpu_count() or 8)
    lp = torch.from_numpy(host).cuda()
    ld = torch.from_numpy(lens).cuda()
    frames = int(lens.sum())
    tmp = tempfile.mkdtemp()
    for order in [int(x) for x in args.orders.split(",")]:
        lm = synthetic_lm(os.path.join(tmp, f"o{order}.arpa"), toks[1:], order, args.keep)
        n_ngrams = sum(len(lm.tables[n]) for n in range(1, order + 1))
        flat = glm.flatten(lm)
        tabs = None
        for w in [float(x) for x in args.weights.split(",")]:
            dec = CUCTCDecoder(toks, beam_size=cfg.beam, nbest=cfg.nbest, blank_skip_threshold=cfg.threshold)
            t0 = time.perf_counter()
            dec.set_lm(lm, w)
            torch.cuda.synchronize()
            build_ms = (time.perf_counter() - t0) * 1e3
            for _ in range(args.warmup):
                dec.decode(lp, ld)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(args.steps):
                out = dec.decode(lp, ld)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / args.steps
            assert (out.status.cpu().numpy() == 0).all()
            cnt = dec.debug_counters()
            # CPU: oracle fused search on a bounded sample, all host threads
            if tabs is None:
                tabs = oracle.lm_tables(flat, glm.token_words(lm, toks, 0))
            threads = os.cpu_count() or 1
            done_f, done_u, t0 = 0, 0, time.perf_counter()
            from concurrent.futures import ThreadPoolExecutor

            with ThreadPoolExecutor(threads) as pool:
                while time.perf_counter() - t0 < args.cpu_budget and done_u < cfg.batch:
                    idx = list(range(done_u, min(done_u + 2 * threads, cfg.batch)))
                    list(pool.map(lambda b: oracle.decode(host[b, : lens[b]], beam_size=cfg.beam, n_best=cfg.nbest,
                                                          blank_skip_threshold=cfg.threshold, lm=tabs, lm_weight=w),
                                  idx))
                    done_f += int(lens[idx].sum())
                    done_u = idx[-1] + 1
            cpu_fps = done_f / (time.perf_counter() - t0)
            print(json.dumps({
                "metric": "LM-fused CTC beam-search decode frames/sec", "workload": cfg.name, "order": order,
                "n_ngrams": n_ngrams, "contexts": int(tabs.score.shape[0]), "lm_weight": w, "beam": cfg.beam,
                "value": frames / (ms / 1e3), "unit": "frames/s", "ms_per_step": ms, "table_build_ms": build_ms,
                "fallback_frames": cnt.get("oneshot_fallbacks", 0) // max(args.steps + args.warmup, 1),
                "cpu_oracle": {"value": cpu_fps, "unit": "frames/s", "cores": threads,
                               "sample": f"first {done_u} utterances ({done_f} frames)"},
            }), flush=True)
            del dec


if __name__ == "__main__":
    main()
