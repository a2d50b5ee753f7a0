"""Diagnostic: decode single utterances and print slow-path counters."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2310_17864_b200 import synth, cuda_ctc_decoder
cfg = synth.CONFIGS[int(sys.argv[1])]
dec = cuda_ctc_decoder(synth.simple_tokens(cfg.vocab), nbest=cfg.nbest, beam_size=cfg.beam, blank_skip_threshold=cfg.threshold)
for b in [int(x) for x in sys.argv[2:]]:
    lp, lens = synth.batch(cfg, indices=[b])
    x = torch.from_numpy(lp).cuda(); l = torch.from_numpy(lens).cuda()
    dec.decode(x, l); torch.cuda.synchronize()
    t = time.perf_counter(); dec.decode(x, l); torch.cuda.synchronize(); dt = time.perf_counter() - t
    print(b, "len", int(lens[0]), "ms", round(dt * 1e3, 2), dec.debug_counters())
