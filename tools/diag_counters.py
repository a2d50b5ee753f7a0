"""Debug counters and kernel time of one decode of a BASELINE config:
python tools/diag_counters.py CFG [beam]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2310_17864_b200 import synth, CUCTCDecoder
cfg = synth.CONFIGS[int(sys.argv[1])]
beam = int(sys.argv[2]) if len(sys.argv) > 2 else cfg.beam
lens_all = synth.lengths(cfg); T = int(lens_all.max())
host = np.zeros((cfg.batch, T, cfg.vocab), np.float32)
_, lens = synth.batch(cfg, out=host, t_pad=T)
x, l = torch.from_numpy(host).cuda(), torch.from_numpy(lens).cuda()
dec = CUCTCDecoder(synth.simple_tokens(cfg.vocab), beam_size=beam, nbest=min(cfg.nbest, beam), blank_skip_threshold=cfg.threshold)
for _ in range(2): dec.decode(x, l)
torch.cuda.synchronize()
dec.kernel_timing(True)
out = dec.decode(x, l)
ms, n, name = dec.kernel_time()
kept = int(out.lengths.shape[0])
print(cfg.name, "beam", beam, name, f"{ms:.3f} ms", dec.debug_counters(), "frames", int(lens.sum()))
