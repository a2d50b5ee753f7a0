"""Diagnostic: time cfg4 decode per chunk of utterances to locate stragglers."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2310_17864_b200 import synth, cuda_ctc_decoder
cfg = synth.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 4]
chunk = 64
dec = cuda_ctc_decoder(synth.simple_tokens(cfg.vocab), nbest=cfg.nbest, beam_size=cfg.beam, blank_skip_threshold=cfg.threshold)
res = []
for c0 in range(0, cfg.batch, chunk):
    idx = np.arange(c0, min(c0 + chunk, cfg.batch))
    lp, lens = synth.batch(cfg, indices=idx)
    x = torch.from_numpy(lp).cuda(); l = torch.from_numpy(lens).cuda()
    dec.decode(x, l); torch.cuda.synchronize()
    t = time.perf_counter(); dec.decode(x, l); torch.cuda.synchronize(); dt = time.perf_counter() - t
    res.append((dt, c0, int(lens.max())))
res.sort(reverse=True)
print("slowest chunks:", [(round(d * 1e3, 2), c, m) for d, c, m in res[:6]])
print("median chunk ms", round(1e3 * np.median([r[0] for r in res]), 2))
d, c0, _ = res[0]
for b in range(c0, c0 + chunk):
    lp, lens = synth.batch(cfg, indices=[b])
    x = torch.from_numpy(lp).cuda(); l = torch.from_numpy(lens).cuda()
    dec.decode(x, l); torch.cuda.synchronize()
    t = time.perf_counter(); dec.decode(x, l); torch.cuda.synchronize(); dt = time.perf_counter() - t
    if dt > 3 * 0.0065 * lens[0] / 875:
        print("slow utterance", b, "len", lens[0], "ms", round(dt * 1e3, 2))
