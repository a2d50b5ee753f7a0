"""Decode one utterance of a config alone (profiling helper):
    python tools/one_utt.py CFG U [--beam B] [--reps N]"""
import argparse, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_17864_b200 import CUCTCDecoder, synth  # noqa: E402
ap = argparse.ArgumentParser()
ap.add_argument("cfg", type=int)
ap.add_argument("u", type=int)
ap.add_argument("--beam", type=int, default=None)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
cfg = synth.CONFIGS[a.cfg]
beam = a.beam or cfg.beam
lp, lens = synth.batch(cfg)
x = torch.from_numpy(lp[a.u:a.u + 1, : int(lens[a.u])]).cuda().contiguous()
ln = torch.tensor([int(lens[a.u])], dtype=torch.int32, device="cuda")
dec = CUCTCDecoder(synth.simple_tokens(cfg.vocab), beam_size=beam, nbest=cfg.nbest, blank_skip_threshold=cfg.threshold)
for _ in range(a.reps):
    dec.decode(x, ln)
torch.cuda.synchronize()
print("ok", int(lens[a.u]))
