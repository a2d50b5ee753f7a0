"""H2D bandwidth probe: one big pinned copy vs per-utterance chunks over several streams."""
import time, torch
n = 4 << 30
h = torch.empty(n // 4, dtype=torch.float32, pin_memory=True)
d = torch.empty_like(h, device="cuda")
for rep in range(2):
    torch.cuda.synchronize(); t = time.perf_counter()
    d.copy_(h, non_blocking=True); torch.cuda.synchronize()
    dt = time.perf_counter() - t
print(f"one 4 GiB copy: {n / dt / 1e9:.1f} GB/s")
for chunk_mb, ns in ((1, 1), (1, 4), (8, 4), (64, 4), (256, 2)):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    c = (chunk_mb << 20) // 4
    torch.cuda.synchronize(); t = time.perf_counter()
    for i, o in enumerate(range(0, h.numel(), c)):
        with torch.cuda.stream(streams[i % ns]):
            d[o:o + c].copy_(h[o:o + c], non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"{chunk_mb} MiB chunks x {ns} streams: {n / dt / 1e9:.1f} GB/s")
x = torch.empty(n // 4, dtype=torch.float32, device="cuda")
torch.cuda.synchronize(); t = time.perf_counter(); hh = x.to("cpu"); torch.cuda.synchronize()
print(f"D2H pageable 4 GiB: {n / (time.perf_counter() - t) / 1e9:.1f} GB/s")
