"""Per-utterance timeline of one decode of a BASELINE config (CTCB_UTT_TRACE):
which SM / warp ran each utterance, when, and its time per frame.

    python tools/utt_timeline.py [cfg] [--out FILE.json]

Prints the kernel span, per-SM busy fraction (first start to last end of the
SM's utterances, over the kernel span), the distribution of microseconds per
frame, and the slowest utterances.
"""
import argparse
import json
import os
import sys
import tempfile

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_17864_b200 import CUCTCDecoder, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("cfg", type=int, nargs="?", default=4)
ap.add_argument("--out", default=None)
a = ap.parse_args()
cfg = synth.CONFIGS[a.cfg]
lp, lens = synth.batch(cfg)
dlp, dlens = torch.from_numpy(lp).cuda(), torch.from_numpy(lens).cuda()
del lp
dec = CUCTCDecoder(synth.simple_tokens(cfg.vocab), beam_size=cfg.beam, nbest=cfg.nbest,
                   blank_skip_threshold=cfg.threshold)
for _ in range(2):
    dec.decode(dlp, dlens)
torch.cuda.synchronize()
path = tempfile.mktemp()
os.environ["CTCB_UTT_TRACE"] = path
dec.decode(dlp, dlens)
torch.cuda.synchronize()
del os.environ["CTCB_UTT_TRACE"]
tr = np.fromfile(path, dtype=np.uint64)[: 2 * len(lens)].reshape(-1, 2)
sm = (tr[:, 0] >> np.uint64(48)).astype(np.int64)
warp = ((tr[:, 0] >> np.uint64(32)) & np.uint64(0xffff)).astype(np.int64)
end = tr[:, 1].astype(np.int64)
start_lo = (tr[:, 0] & np.uint64(0xffffffff)).astype(np.int64)
start = (end & ~0xffffffff) | start_lo
start = np.where(start > end, start - (1 << 32), start)
t0 = start.min()
start, end = (start - t0) / 1e3, (end - t0) / 1e3  # us
span = end.max()
dur = end - start
upf = dur / np.maximum(lens, 1)
per_sm_end = np.array([end[sm == s].max() for s in np.unique(sm)])
per_warp_end = np.array([end[warp == w].max() for w in np.unique(warp)])
rep = {
    "cfg": a.cfg, "span_us": float(span), "utterances": int(len(lens)),
    "sm_end_frac": {"min": float(per_sm_end.min() / span), "mean": float(per_sm_end.mean() / span)},
    "warp_end_frac": {"min": float(per_warp_end.min() / span), "p10": float(np.percentile(per_warp_end, 10) / span),
                      "mean": float(per_warp_end.mean() / span)},
    "us_per_frame": {q: float(np.percentile(upf, p)) for q, p in (("p1", 1), ("p50", 50), ("p99", 99), ("max", 100))},
    "us_per_frame_by_len": [[int(lo), float(np.median(upf[(lens >= lo) & (lens < lo + 125)]))]
                            for lo in range(125, 876, 125)],
    "utts_per_warp": float(len(lens) / len(np.unique(warp))),
}
slow = np.argsort(-upf)[:10]
rep["slowest"] = [{"u": int(u), "T": int(lens[u]), "us": float(dur[u]), "us_per_frame": float(upf[u]),
                   "start_us": float(start[u]), "sm": int(sm[u])} for u in slow]
late = np.argsort(-end)[:10]
rep["last_to_finish"] = [{"u": int(u), "T": int(lens[u]), "start_us": float(start[u]), "end_us": float(end[u]),
                          "sm": int(sm[u]), "warp": int(warp[u])} for u in late]
print(json.dumps(rep, indent=1))
if a.out:
    np.savez_compressed(a.out, sm=sm, warp=warp, start=start, end=end, lens=lens)
