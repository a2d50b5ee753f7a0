"""Diagnostic: where the e2e time of the host-buffer path goes (cfg4)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2310_17864_b200 import synth, cuda_ctc_decoder
cfg = synth.CONFIGS[4]
lens_all = synth.lengths(cfg)
host = torch.empty((cfg.batch, int(lens_all.max()), cfg.vocab), dtype=torch.float32, pin_memory=True)
_, lens = synth.batch(cfg, out=host.numpy(), t_pad=int(lens_all.max()), threads=os.cpu_count() or 8)
lt = torch.from_numpy(lens)
dec = cuda_ctc_decoder(synth.simple_tokens(cfg.vocab), nbest=1, beam_size=10, blank_skip_threshold=cfg.threshold)
dec.decode_host(host, lt)
for name, fn in (("decode_host", lambda: dec.decode_host(host, lt)), ("__call__", lambda: dec(host, lt)),
                 ("H2D full padded", lambda: host.to("cuda", non_blocking=True))):
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(3): fn()
    torch.cuda.synchronize(); print(name, round((time.perf_counter() - t) / 3 * 1e3, 2), "ms")
out = dec.decode_host(host, lt)
t = time.perf_counter()
for _ in range(3): dec._hypotheses(out[0], out[2], out[3], out[4])
print("_hypotheses", round((time.perf_counter() - t) / 3 * 1e3, 2), "ms", out[0].shape, out[0].flags['C_CONTIGUOUS'])
