"""Print the GPU and oracle n-best of one stored utterance side by side:
python tools/compare_case.py FILE.npy beam nbest skip_thr beam_thr [K] [merge]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from paper_2310_17864_b200 import CUCTCDecoder
u = np.load(sys.argv[1]); beam, nb = int(sys.argv[2]), int(sys.argv[3]); thr, bthr = float(sys.argv[4]), float(sys.argv[5])
K = int(sys.argv[6]) if len(sys.argv) > 6 and sys.argv[6] != "None" else None
merge = sys.argv[7] if len(sys.argv) > 7 else "logadd"
V = u.shape[1]
dec = CUCTCDecoder(["-"] + [f"t{i}" for i in range(1, V)], beam_size=beam, nbest=nb, blank_skip_threshold=thr, beam_threshold=bthr)
dec.set_beam_size_token(K); dec.set_merge_mode(merge)
tok, _, ln, sc, cnt = dec.to_host(dec.decode(torch.from_numpy(u[None]).cuda(), torch.tensor([u.shape[0]], dtype=torch.int32).cuda()))
ref = oracle.decode(u, beam_size=beam, n_best=nb, blank_skip_threshold=thr, beam_threshold=bthr, beam_size_token=K, merge_mode=merge)
n = max(cnt[0], len(ref.scores))
for j in range(n):
    g = (round(float(sc[0, j]), 12), tok[0, j, :ln[0, j]].tolist()) if j < cnt[0] else None
    r = (round(ref.scores[j], 12), ref.tokens[j]) if j < len(ref.scores) else None
    print(j, "  " if g == r else "!!", g, r)
