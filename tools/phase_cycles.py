"""Per-phase cycle breakdown of the fast kernel's frame step (a library built
with -DCTCB_PHASES, selected with CTCB_LIB):

    CTCB_LIB=variants/libctcb_ph.so python tools/phase_cycles.py CFG [U ...]

Decodes the given utterances of a config (default: all) in one launch and
prints lane-0 clock() cycles per frame for each phase: 0 frame top (classify,
row issue, mbarrier wait), 1 staged row -> validation / vmax, 2 merge
structure + blank / repeat groups, 3 shortcut test and selection, 4 top-k
(full path), 5 exclusions / append lists / frame best, 6 one-shot
selection, 7 k-way merge, 8 commit, 9 validation verdict / checkpoints.
"""
import json
import os
import sys
import tempfile

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2310_17864_b200 import CUCTCDecoder, synth  # noqa: E402

cfg = synth.CONFIGS[int(sys.argv[1])]
idx = [int(x) for x in sys.argv[2:]] or None
lp, lens = synth.batch(cfg, indices=idx)
dec = CUCTCDecoder(synth.simple_tokens(cfg.vocab), beam_size=cfg.beam, nbest=cfg.nbest,
                   blank_skip_threshold=cfg.threshold)
x, ln = torch.from_numpy(lp).cuda(), torch.from_numpy(lens).cuda()
dec.decode(x, ln)
torch.cuda.synchronize()
path = tempfile.mktemp()
os.environ["CTCB_UTT_TRACE"] = path
dec.kernel_timing(True)
dec.decode(x, ln)
ms, n, name = dec.kernel_time()
del os.environ["CTCB_UTT_TRACE"]
ph = np.fromfile(path, dtype=np.uint64)[2 * len(lens):].astype(np.float64)
frames = float(lens.sum())
names = ["top/stage", "validate/vmax", "structure+groups", "shortcut", "topk", "lists/best", "oneshot",
         "kway", "commit", "verdict/ckpt"]
out = {"kernel": name, "kernel_ms": ms, "frames": frames, "shortcut_frac": ph[14] / frames,
       "cycles_per_frame": {nm: round(ph[q] / frames, 1) for q, nm in enumerate(names)},
       "total_per_frame": round(ph[:10].sum() / frames, 1)}
full = frames - ph[14]
out["full_path_cycles_per_full_frame"] = {nm: round(ph[q] / max(full, 1), 1) for q, nm in ((4, "topk"), (5, "lists/best"), (6, "oneshot"), (7, "kway"))}
print(json.dumps(out, indent=1))
