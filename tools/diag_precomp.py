"""Diagnostic: device time per decode call in fused and precomputed-top-k modes
(cfg4), for the default library and every variant in variants/ (CTCB_LIB)."""
import glob, os, subprocess, sys
if len(sys.argv) == 1:
    libs = ["paper_2310_17864_b200/libctcb.so"] + sorted(glob.glob("variants/*.so"))
    for lib in libs:
        env = dict(os.environ, CTCB_LIB=os.path.abspath(lib))
        out = subprocess.run([sys.executable, __file__, "run"], env=env, capture_output=True, text=True)
        print(os.path.basename(lib), out.stdout.strip(), out.stderr.strip()[-300:])
    sys.exit(0)
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2310_17864_b200 import synth, cuda_ctc_decoder
cfg = synth.CONFIGS[4]
lp, lens = synth.batch(cfg, threads=os.cpu_count() or 8)
x = torch.from_numpy(lp).cuda(); l = torch.from_numpy(lens).cuda()
res = []
for mode in ("fused", "precomp"):
    os.environ["CTCB_TOPK_MODE"] = mode
    dec = cuda_ctc_decoder(synth.simple_tokens(cfg.vocab), nbest=1, beam_size=10, blank_skip_threshold=cfg.threshold)
    for _ in range(3): dec.decode(x, l)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dec.kernel_timing(True)
    e0.record()
    for _ in range(10): dec.decode(x, l)
    e1.record(); torch.cuda.synchronize()
    kms, kn, kname = dec.kernel_time()
    res.append(f"{mode}: step {e0.elapsed_time(e1) / 10:.3f} ms, beam kernel {kms / kn:.3f} ms")
print(" | ".join(res))
