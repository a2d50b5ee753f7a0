"""Fused vs precomputed top-k mode on cfg4 shards (the per-GPU batch of an
N-GPU strong-scaling run): python tools/shard_modes.py [N ...]"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_17864_b200 import CUCTCDecoder, shard, synth  # noqa: E402

cfg = synth.CONFIGS[4]
L = synth.lengths(cfg)
for n in [int(x) for x in sys.argv[1:]] or [8, 4, 2]:
    idx = shard.lpt_shards(L, n)[0]
    lp, lens = synth.batch(cfg, indices=idx)
    x, ln = torch.from_numpy(lp).cuda(), torch.from_numpy(lens).cuda()
    del lp
    res = {"gpus": n, "batch": len(idx), "frames": int(lens.sum())}
    for mode in ("fused", "precomp"):
        os.environ["CTCB_TOPK_MODE"] = mode
        dec = CUCTCDecoder(synth.simple_tokens(cfg.vocab), beam_size=10, nbest=1, blank_skip_threshold=cfg.threshold)
        for _ in range(3):
            dec.decode(x, ln)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            dec.decode(x, ln)
        e1.record()
        torch.cuda.synchronize()
        res[mode + "_ms"] = round(e0.elapsed_time(e1) / 10, 3)
    del os.environ["CTCB_TOPK_MODE"]
    print(json.dumps(res), flush=True)
    del x, ln
    torch.cuda.empty_cache()
