import os, sys, time, tempfile
sys.path.insert(0, "/root/repo"); sys.path.insert(0, "/root/repo/tools")
import numpy as np, torch
from paper_2310_17864_b200 import synth, CUCTCDecoder
from bench_lm import synthetic_lm
cfg = synth.CONFIGS[int(sys.argv[1]) if len(sys.argv) > 1 else 1]
toks = synth.simple_tokens(cfg.vocab)
lens_all = synth.lengths(cfg); T = int(lens_all.max())
host = np.zeros((cfg.batch, T, cfg.vocab), np.float32)
_, lens = synth.batch(cfg, out=host, t_pad=T)
lp = torch.from_numpy(host).cuda(); ld = torch.from_numpy(lens).cuda()
lm = synthetic_lm(tempfile.mktemp(), toks[1:], 2, 20)
def run(name, setup):
    dec = CUCTCDecoder(toks, beam_size=10, nbest=1, blank_skip_threshold=0.95)
    setup(dec)
    for _ in range(2): dec.decode(lp, ld)
    torch.cuda.synchronize()
    dec.kernel_timing(True)
    t0 = time.perf_counter()
    for _ in range(3): out = dec.decode(lp, ld)
    torch.cuda.synchronize()
    k_ms, k_n, k_name = dec.kernel_time()
    print(name, k_name, f"{k_ms / k_n:.2f} ms/launch", dec.debug_counters(), flush=True)
run("plain", lambda d: None)
run("sil-only", lambda d: d.set_silence(cfg.vocab - 1, 0.5))
run("lm w=0", lambda d: d.set_lm(lm, 0.0))
run("lm w=0.5", lambda d: d.set_lm(lm, 0.5))
run("lm w=2", lambda d: d.set_lm(lm, 2.0))
