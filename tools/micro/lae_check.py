"""Run lae_check on random score pairs and report disagreements with numpy's logaddexp."""
import os, subprocess, sys
import numpy as np
here = os.path.dirname(os.path.abspath(__file__))
rng = np.random.default_rng(int(sys.argv[1]) if len(sys.argv) > 1 else 0)
n = 4_000_000
x = -rng.uniform(0, 60, n)
d = np.concatenate([rng.uniform(0, 2, n // 2), rng.exponential(5, n - n // 2)])
y = x - d
# quantized-style values too
q = -np.round(rng.uniform(0, 40, n) * 8) / 8
x[: n // 4] = q[: n // 4]
y[: n // 4] = q[: n // 4] - np.round(rng.uniform(0, 6, n // 4) * 8) / 8
xy = np.stack([x, y], 1).astype(np.float64)
xy.tofile("/tmp/lae_in.bin")
subprocess.run([os.path.join(here, "lae_check"), "/tmp/lae_in.bin", "/tmp/lae_out.bin"], check=True)
out = np.fromfile("/tmp/lae_out.bin", dtype=np.float64).reshape(-1, 2)
ref = np.logaddexp(x, y)
for i, name in enumerate(("polynomial", "exact")):
    bad = out[:, i] != ref
    print(f"{name}: {bad.sum()} of {n} differ from numpy")
    if bad.any():
        j = np.flatnonzero(bad)[:3]
        for k in j:
            print("   ", repr(x[k]), repr(y[k]), repr(out[k, i]), repr(ref[k]))
