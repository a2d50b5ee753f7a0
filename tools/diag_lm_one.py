"""One fused-kernel decode of cfg1 (64 utterances) for ncu: python tools/diag_lm_one.py [sil|lm]"""
import os, sys, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import numpy as np, torch
from paper_2310_17864_b200 import synth, CUCTCDecoder
from bench_lm import synthetic_lm
cfg = synth.CONFIGS[int(sys.argv[2]) if len(sys.argv) > 2 else 1]
toks = synth.simple_tokens(cfg.vocab)
lens_all = synth.lengths(cfg); T = int(lens_all.max())
host = np.zeros((cfg.batch, T, cfg.vocab), np.float32)
_, lens = synth.batch(cfg, out=host, t_pad=T)
dec = CUCTCDecoder(toks, beam_size=10, nbest=1, blank_skip_threshold=0.95)
if sys.argv[1:2] == ["sil"]:
    dec.set_silence(cfg.vocab - 1, 0.5)
else:
    dec.set_lm(synthetic_lm(tempfile.mktemp(), toks[1:], 2, 20), 2.0)
out = dec.decode(torch.from_numpy(host).cuda(), torch.from_numpy(lens).cuda())
torch.cuda.synchronize()
print(out.status.cpu().numpy().max())
