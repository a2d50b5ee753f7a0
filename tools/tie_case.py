import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch, tempfile
import oracle
from paper_2310_17864_b200 import CUCTCDecoder
from paper_2310_17864_b200 import lm as glm
u = np.load("tests/golden/regress_ties_beam39.npy")
V = u.shape[1]
toks = ["-"] + [f"t{i}" for i in range(1, V)]
p = tempfile.mktemp()
open(p, "w").write("\\data\\\nngram 1=3\n\n\\1-grams:\n-1.0\t<s>\n-1.0\t</s>\n-1.0\tt1\n\n\\end\\\n")
lm = glm.parse_arpa(p)
for thr in (1.0, 0.95):
    for nb in (1, 5, 39):
        ref = oracle.decode(u, beam_size=39, n_best=nb, blank_skip_threshold=thr, beam_threshold=5.0)
        out = {}
        for mode in ("generic", "fused"):
            dec = CUCTCDecoder(toks, beam_size=39, nbest=nb, blank_skip_threshold=thr, beam_threshold=5.0)
            if mode == "fused":
                dec.set_lm(lm, 0.0)
            tok, _, ln, sc, cnt = dec.to_host(dec.decode(torch.from_numpy(u[None]).cuda(), torch.tensor([u.shape[0]], dtype=torch.int32).cuda()))
            out[mode] = [tok[0, j, :ln[0, j]].tolist() for j in range(cnt[0])]
        print(thr, nb, "generic==ref", out["generic"] == ref.tokens, "fused==ref", out["fused"] == ref.tokens)
        if out["generic"] != ref.tokens:
            for j in range(len(ref.tokens)):
                if j >= len(out["generic"]) or out["generic"][j] != ref.tokens[j]:
                    print("   first diff rank", j, ref.scores[j], ref.tokens[j], out["generic"][j] if j < len(out["generic"]) else None)
                    break
# scores around the first difference
ref = oracle.decode(u, beam_size=39, n_best=39, blank_skip_threshold=1.0, beam_threshold=5.0)
dec = CUCTCDecoder(toks, beam_size=39, nbest=39, blank_skip_threshold=1.0, beam_threshold=5.0)
tok, _, ln, sc, cnt = dec.to_host(dec.decode(torch.from_numpy(u[None]).cuda(), torch.tensor([u.shape[0]], dtype=torch.int32).cuda()))
for j in range(25, 30):
    print(j, repr(float(sc[0, j])), tok[0, j, :ln[0, j]].tolist(), "| ref", repr(ref.scores[j]), ref.tokens[j])
