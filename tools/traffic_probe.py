"""One cfg decode for DRAM-traffic attribution under ncu:
    python tools/traffic_probe.py CFG --thr X [--no-validate]"""
import argparse, os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_17864_b200 import cuda_ctc_decoder, synth  # noqa: E402
ap = argparse.ArgumentParser()
ap.add_argument("cfg", type=int)
ap.add_argument("--thr", type=float, default=None)
ap.add_argument("--no-validate", action="store_true")
a = ap.parse_args()
cfg = synth.CONFIGS[a.cfg]
lp, lens = synth.batch(cfg)
x = torch.from_numpy(lp).cuda()
ln = torch.from_numpy(lens).cuda()
dec = cuda_ctc_decoder(synth.simple_tokens(cfg.vocab), nbest=cfg.nbest, beam_size=cfg.beam,
                       blank_skip_threshold=a.thr if a.thr else cfg.threshold, validate=not a.no_validate)
for _ in range(2):
    out = dec.decode(x, ln)
torch.cuda.synchronize()
print("ok")
