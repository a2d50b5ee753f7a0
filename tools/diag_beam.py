"""Diagnostic: decode a few utterances at a given beam and print slow-path counters."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2310_17864_b200 import synth, cuda_ctc_decoder
cfg = synth.CONFIGS[int(sys.argv[1])]
beam = int(sys.argv[2]); n = int(sys.argv[3])
dec = cuda_ctc_decoder(synth.simple_tokens(cfg.vocab), nbest=min(beam, 10), beam_size=beam, blank_skip_threshold=cfg.threshold)
lp, lens = synth.batch(cfg, indices=range(n))
x = torch.from_numpy(lp).cuda(); l = torch.from_numpy(lens).cuda()
dec.decode(x, l); torch.cuda.synchronize()
t = time.perf_counter(); dec.decode(x, l); torch.cuda.synchronize(); dt = time.perf_counter() - t
print("beam", beam, "utts", n, "frames", int(lens.sum()), "ms", round(dt * 1e3, 2), dec.debug_counters())
