"""Run one sub-case of test_fused_and_precomputed_topk_modes_agree:
python tools/dbg_cases.py CASE MODE   (CASE 0..4, MODE precomp|staged|fused)"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2310_17864_b200 import CUCTCDecoder, synth
import oracle
ci, mode = int(sys.argv[1]), sys.argv[2]
cases = []
for cfg_id, idx in ((0, range(4)), (1, range(16)), (3, range(2))):
    cfg = synth.CONFIGS[cfg_id]
    lp, lens = synth.batch(cfg, indices=idx)
    cases.append((lp, lens, cfg.beam, cfg.nbest, cfg.threshold))
rng = np.random.default_rng(52)
for V in (1000, 1001):
    x = rng.normal(size=(3, 60, V)) * 2.0
    x[:, 7, :] = 0.0
    x = x - x.max(2, keepdims=True)
    lp = (x - np.log(np.exp(x).sum(2, keepdims=True))).astype(np.float32)
    cases.append((lp, np.array([60, 41, 9], dtype=np.int32), 10, 3, 0.95))
if mode == "staged":
    os.environ["CTCB_TOPK_STAGED"] = "1"; mode = "precomp"
os.environ["CTCB_TOPK_MODE"] = mode
lp, lens, beam, nb, thr = cases[ci]
dec = CUCTCDecoder(synth.simple_tokens(lp.shape[2]), beam_size=beam, nbest=nb, blank_skip_threshold=thr)
out = dec.decode(torch.from_numpy(lp).cuda(), torch.from_numpy(lens).cuda())
tokens, _, lengths, scores, counts = dec.to_host(out)
ref = oracle.decode_batch(lp, lens, beam_size=beam, n_best=nb, blank_skip_threshold=thr)
ok = all([tokens[b, j, :lengths[b, j]].tolist() for j in range(counts[b])] == r.tokens for b, r in enumerate(ref))
print(ci, sys.argv[2], "ok" if ok else "MISMATCH", dec.debug_counters())
