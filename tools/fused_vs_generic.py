import os, sys, tempfile
sys.path.insert(0, "/root/repo")
import numpy as np, torch
from paper_2310_17864_b200 import synth, CUCTCDecoder
from paper_2310_17864_b200 import lm as glm
cfg = synth.CONFIGS[2]
toks = synth.simple_tokens(cfg.vocab)
lens_all = synth.lengths(cfg); T = int(lens_all.max())
host = np.zeros((cfg.batch, T, cfg.vocab), np.float32)
_, lens = synth.batch(cfg, out=host, t_pad=T)
x, l = torch.from_numpy(host).cuda(), torch.from_numpy(lens).cuda()
p = tempfile.mktemp()
open(p, "w").write("\\data\\\nngram 1=3\n\n\\1-grams:\n-1.0\t<s>\n-1.0\t</s>\n-1.0\tt1\n\n\\end\\\n")
lm = glm.parse_arpa(p)
for beam in (16, 32, 50, 64):
    res = {}
    for mode in ("generic", "fused"):
        dec = CUCTCDecoder(toks, beam_size=beam, nbest=10, blank_skip_threshold=0.95)
        if mode == "fused":
            dec.set_lm(lm, 0.0)
        dec.decode(x, l); torch.cuda.synchronize()
        dec.kernel_timing(True)
        out = dec.decode(x, l)
        ms, n, name = dec.kernel_time()
        tok, _, ln, sc, cnt = dec.to_host(out)
        res[mode] = (ms, [tok[b, 0, :ln[b, 0]].tolist() for b in range(8)])
    print(beam, "generic %.1f ms" % res["generic"][0], "fused %.1f ms" % res["fused"][0], "same top-1:", res["generic"][1] == res["fused"][1])
for beam in (16, 50):
    dec = CUCTCDecoder(toks, beam_size=beam, nbest=10, blank_skip_threshold=0.95)
    dec.set_lm(lm, 0.0)
    dec.decode(x, l); torch.cuda.synchronize()
    print(beam, dec.debug_counters(), "frames", int(lens.sum()))
