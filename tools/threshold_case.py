"""Replay a stored fuzz batch and print GPU vs oracle n-best around the first
difference, with scores relative to best - beam_threshold:
python tools/threshold_case.py FILE.npy b beam nb thr bthr"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from paper_2310_17864_b200 import CUCTCDecoder
lp = np.load(sys.argv[1]); b = int(sys.argv[2]); beam, nb = int(sys.argv[3]), int(sys.argv[4])
thr, bthr = float(sys.argv[5]), float(sys.argv[6]); lens = [int(x) for x in sys.argv[7].split(",")]
u = lp[b, : lens[b]]
V = u.shape[1]
dec = CUCTCDecoder(["-"] + [f"t{i}" for i in range(1, V)], beam_size=beam, nbest=nb, blank_skip_threshold=thr, beam_threshold=bthr)
tok, _, ln, sc, cnt = dec.to_host(dec.decode(torch.from_numpy(u[None]).cuda(), torch.tensor([u.shape[0]], dtype=torch.int32).cuda()))
ref = oracle.decode(u, beam_size=beam, n_best=nb, blank_skip_threshold=thr, beam_threshold=bthr)
print("gpu count", cnt[0], "oracle count", len(ref.scores))
for j in range(max(cnt[0], len(ref.scores))):
    g = (repr(float(sc[0, j])), tok[0, j, :ln[0, j]].tolist()) if j < cnt[0] else None
    r = (repr(ref.scores[j]), ref.tokens[j]) if j < len(ref.scores) else None
    if g != r:
        print(j, "gpu", g, "ref", r)
