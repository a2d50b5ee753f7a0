"""Diagnostic: timeline of the pipelined host path (cfg4): when each range's results arrive."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_17864_b200 import synth, cuda_ctc_decoder
cfg = synth.CONFIGS[4]
lens_all = synth.lengths(cfg)
host = torch.empty((cfg.batch, int(lens_all.max()), cfg.vocab), dtype=torch.float32, pin_memory=True)
_, lens = synth.batch(cfg, out=host.numpy(), t_pad=int(lens_all.max()), threads=os.cpu_count() or 8)
lt = torch.from_numpy(lens)
dec = cuda_ctc_decoder(synth.simple_tokens(cfg.vocab), nbest=1, beam_size=10, blank_skip_threshold=cfg.threshold)
for chunks in (1, 4, 8, 16):
    for rep in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter(); marks = []
        for lo, hi, tok, ln, sc, cnt in dec._decode_host_chunks(host, lt, chunks):
            t1 = time.perf_counter(); h = dec._hypotheses(tok, ln, sc, cnt); marks.append((round((t1 - t0) * 1e3, 1), round((time.perf_counter() - t0) * 1e3, 1)))
        if rep: print(chunks, "chunks: (arrive, built) ms", marks)
