"""Slow-path counters and single-utterance kernel time for chosen utterances of
a config (fused top-k mode):  python tools/utt_counters.py CFG U [U ...]"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_17864_b200 import CUCTCDecoder, synth  # noqa: E402

os.environ.setdefault("CTCB_TOPK_MODE", "fused")
cfg = synth.CONFIGS[int(sys.argv[1])]
dec = CUCTCDecoder(synth.simple_tokens(cfg.vocab), beam_size=cfg.beam, nbest=cfg.nbest,
                   blank_skip_threshold=cfg.threshold)
L = synth.lengths(cfg)
for u in map(int, sys.argv[2:]):
    x = torch.from_numpy(synth.utterance(cfg, u, int(L[u]))[None]).cuda()
    ln = torch.tensor([int(L[u])], dtype=torch.int32, device="cuda")
    dec.decode(x, ln)
    dec.kernel_timing(True)
    dec.decode(x, ln)
    ms, n, name = dec.kernel_time()
    dec.kernel_timing(False)
    print(json.dumps({"u": u, "T": int(L[u]), "us_per_frame": 1000 * ms / int(L[u]), "kernel": name,
                      **dec.debug_counters()}))
