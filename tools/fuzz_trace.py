"""Debug a fuzz mismatch: decode growing prefixes of one utterance on the GPU and
with the oracle; print the first prefix length where the n-best differs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import oracle
from paper_2310_17864_b200 import CUCTCDecoder
u = np.load(sys.argv[1]); beam, K, thr = int(sys.argv[2]), int(sys.argv[3]), float(sys.argv[4])
bthr = float(sys.argv[5]) if len(sys.argv) > 5 else 50.0
K = K if K > 0 else None
V = u.shape[1]
dec = CUCTCDecoder(["-"] + [f"t{i}" for i in range(1, V)], beam_size=beam, nbest=beam, blank_skip_threshold=thr,
                   beam_threshold=bthr)
dec.set_beam_size_token(K)
for T in range(1, u.shape[0] + 1):
    x = torch.from_numpy(np.ascontiguousarray(u[None, :T])).cuda()
    tok, _, ln, sc, cnt = dec.to_host(dec.decode(x, torch.tensor([T], dtype=torch.int32).cuda()))
    digits = int(os.environ.get("TRACE_DIGITS", "9"))  # 0: compare scores bit for bit
    rnd = (lambda v: float(v)) if digits == 0 else (lambda v: round(float(v), digits))
    got = [(tok[0, j, :ln[0, j]].tolist(), rnd(sc[0, j])) for j in range(cnt[0])]
    ref = oracle.decode(u[:T], beam_size=beam, n_best=beam, blank_skip_threshold=thr, beam_size_token=K,
                        beam_threshold=bthr)
    exp = [(t, rnd(s)) for t, s in zip(ref.tokens, ref.scores)]
    print(T, "OK" if got == exp else "DIFF", got if got != exp else "")
    if got != exp:
        print("   ref", exp)
        for j, (a, b) in enumerate(zip(got, exp)):
            if a != b:
                print("   first diff at rank", j, a, b)
                break
        break
