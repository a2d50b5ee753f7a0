import sys, os
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2310_17864_b200 import synth, CUCTCDecoder
cfg = synth.CONFIGS[2]
lp, lens = synth.batch(cfg, indices=[0])
for beam in (16, 17, 32, 50):
    dec = CUCTCDecoder(synth.simple_tokens(500), beam_size=beam, nbest=min(beam,10), blank_skip_threshold=0.95)
    out = dec.decode(torch.from_numpy(lp).cuda(), torch.from_numpy(lens).cuda())
    torch.cuda.synchronize()
    print(beam, "count", out.counts.cpu().tolist(), "status", out.status.cpu().tolist(), "len", out.lengths.cpu().tolist()[0][:3], dec.debug_counters())
