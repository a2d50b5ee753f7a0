"""Per-utterance cost of a config's decode: each utterance decoded alone
(B = 1, one CTA / warp), its kernel time, kept frames and slow-path counters.

    python tools/block_utt_times.py [cfg] [--beam B] [--top N]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_17864_b200 import CUCTCDecoder, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("cfg", type=int, nargs="?", default=2)
ap.add_argument("--beam", type=int, default=None)
ap.add_argument("--top", type=int, default=12)
a = ap.parse_args()
cfg = synth.CONFIGS[a.cfg]
beam = a.beam or cfg.beam
nbest = min(beam, 10) if a.cfg == 2 else cfg.nbest
lp, lens = synth.batch(cfg)
dlp = torch.from_numpy(lp).cuda()
dec = CUCTCDecoder(synth.simple_tokens(cfg.vocab), beam_size=beam, nbest=nbest, blank_skip_threshold=cfg.threshold)
rows = []
for u in range(lp.shape[0]):
    x = dlp[u:u + 1, : int(lens[u])].contiguous()
    ln = torch.tensor([int(lens[u])], dtype=torch.int32, device="cuda")
    dec.decode(x, ln)  # warm
    dec.kernel_timing(True)
    out = dec.decode(x, ln)
    torch.cuda.synchronize()
    ms, n, name = dec.kernel_time()
    dec.kernel_timing(False)
    c = dec.debug_counters()
    rows.append({"u": u, "T": int(lens[u]), "ms": ms / max(n, 1), "us_per_frame": 1000 * ms / max(n, 1) / int(lens[u]), **c})
rows.sort(key=lambda r: -r["ms"])
print(json.dumps({"cfg": a.cfg, "beam": beam, "kernel": name,
                  "mean_us_per_frame": float(np.mean([r["us_per_frame"] for r in rows])),
                  "max_ms": rows[0]["ms"], "sum_ms": float(sum(r["ms"] for r in rows))}))
for r in rows[: a.top]:
    print(json.dumps(r))
