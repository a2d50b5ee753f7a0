"""One fused-kernel decode of cfg2 at a given beam with a weight-0 unigram LM (for ncu):
python tools/fused_one.py BEAM"""
import os, sys, tempfile
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2310_17864_b200 import synth, CUCTCDecoder
from paper_2310_17864_b200 import lm as glm
cfg = synth.CONFIGS[2]
toks = synth.simple_tokens(cfg.vocab)
lens_all = synth.lengths(cfg); T = int(lens_all.max())
host = np.zeros((cfg.batch, T, cfg.vocab), np.float32)
_, lens = synth.batch(cfg, out=host, t_pad=T)
p = tempfile.mktemp()
open(p, "w").write("\\data\\\nngram 1=3\n\n\\1-grams:\n-1.0\t<s>\n-1.0\t</s>\n-1.0\tt1\n\n\\end\\\n")
dec = CUCTCDecoder(toks, beam_size=int(sys.argv[1]), nbest=10, blank_skip_threshold=0.95)
dec.set_lm(glm.parse_arpa(p), 0.0)
out = dec.decode(torch.from_numpy(host).cuda(), torch.from_numpy(lens).cuda())
torch.cuda.synchronize()
print(out.status.cpu().numpy().max())
