#!/usr/bin/env python
"""Benchmark: CTC prefix beam-search decode frames/s at V=500, beam=10
(BASELINE.json metric) on the whole-box workload (config 4: B=4096 utterances,
T ~ U[125, 875], peaky synthetic posteriors, thr 0.95, nbest 1).

    python bench.py [--gpus N --steps K --warmup W] [--impl reference]
    torchrun --nproc-per-node N bench.py --gpus N ...   (one rank per GPU)

One step = one decode of the rank's length-balanced (LPT) shard of the batch
(strong scaling: the fixed B = 4096 split over the ranks; --weak gives each
rank its own ~B utterances), inputs resident in HBM.  value = frames of all ranks / max-over-ranks step
time (CUDA events on the decode stream).  Inputs (7.2 GB padded at N=1) are
larger than L2, so no flush is needed between steps.  `e2e` is the same
metric through the public API (`CUCTCDecoder.__call__`) from pinned host
memory, H2D + decode + D2H + hypothesis construction inside the timed region.
`--impl reference` times the CPU reference path (the C oracle port of
ctcforge, oracle/) on the host cores instead.  On rank 0 at N=1 the line also
carries `cpu_baseline` (the port on a 512-utterance sample),
`cpu_baseline_reference` (ctcforge itself, baseline/_ref, decode_batch with a
process pool) and `parity`: the timed decode's own results on those samples
against the port and against ctcforge.
"""

from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2310_17864_b200 import synth  # noqa: E402
from paper_2310_17864_b200.shard import lpt_shards  # noqa: E402

METRIC = "CTC beam-search decode frames/sec @V=500,beam=10"
WORKLOADS = {"cfg4": 4, "cfg1": 1, "cfg0": 0, "cfg2": 2, "cfg3": 3}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def measured_peak_gbs():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def algorithmic_bytes(lp: np.ndarray, lens: np.ndarray, cutoff: float) -> tuple[int, int]:
    """Σ_b [4·len_b (blank probe) + 4·(V−1)·kept_b] + 4·B; also Σ kept."""
    V = lp.shape[2]
    total, kept_total = 4 * len(lens), 0
    for b, n in enumerate(lens):
        blank = lp[b, :n, 0]
        kept = int(np.count_nonzero(~(blank >= cutoff)))
        kept_total += kept
        total += 4 * int(n) + 4 * (V - 1) * kept
    return total, kept_total


class ClockSampler:
    """nvidia-smi clocks and throttle reasons, sampled every 50 ms from before
    the warm-up (so nvidia-smi's own start-up, which can hold driver locks, is
    outside the timed region); summary() keeps the samples taken inside it."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.lines: list = []
        self.proc = None
        self.window = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits", "-i",
                 str(self.device), "-lms", "50"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.monotonic(), line.strip()))

    def wait_ready(self, timeout: float = 10.0):
        t_end = time.monotonic() + timeout
        while self.proc is not None and not self.lines and time.monotonic() < t_end:
            time.sleep(0.02)

    def mark(self, t0: float, t1: float):
        self.window = (t0, t1)

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        return False

    def summary(self):
        lines = self.lines
        if self.window is not None:
            t0, t1 = self.window
            inside = [x for x in lines if t0 <= x[0] <= t1 + 0.05]
            after = [x for x in lines if x[0] > t1]
            lines = inside or after[:1]
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for _, line in lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx.append(float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_baseline(cfg, budget_s: float, threads: int, sample_utts: int):
    """Time the oracle port (C restatement of ctcforge) on a bounded sample of
    the workload with `threads` host threads; returns (frames/s, sample desc,
    oracle results of the decoded utterances 0..n-1 for the parity check).
    n_best is raised to 2 so the top-1/top-2 gap is known; it only truncates
    the final sorted list (decoder.py:799-801), so the timing is unchanged."""
    import oracle

    oracle.build()
    idx = np.arange(min(sample_utts, cfg.batch))
    lp, lens = synth.batch(cfg, indices=idx)
    nb = min(cfg.beam, max(cfg.nbest, 2))
    # warm-up one utterance (page in, thread pool)
    oracle.decode_batch(lp[:1], lens[:1], threads=1, beam_size=cfg.beam, n_best=nb,
                        blank_skip_threshold=cfg.threshold)
    done_frames, done_utts, t0 = 0, 0, time.perf_counter()
    chunk = max(threads, 1) * 2
    results = []
    while done_utts < len(idx):
        sl = slice(done_utts, min(done_utts + chunk, len(idx)))
        results += oracle.decode_batch(lp[sl], lens[sl], threads=threads, beam_size=cfg.beam, n_best=nb,
                                       blank_skip_threshold=cfg.threshold)
        done_frames += int(lens[sl].sum())
        done_utts = sl.stop
        if time.perf_counter() - t0 > budget_s:
            break
    dt = time.perf_counter() - t0
    return (done_frames / dt, f"first {done_utts} utterances of {cfg.name} ({done_frames} frames, {dt:.1f} s)",
            [(r.tokens, r.scores) for r in results])


def ctcforge_baseline(cfg, workers: int, sample_utts: int):
    """Time the reference itself -- ctcforge.decode_batch(workers=cores)
    (decoder.py:138-170), installed unmodified in baseline/_ref -- on the first
    `sample_utts` utterances of the workload.  Returns (frames/s, sample desc,
    results) or None when baseline/_ref is absent."""
    ref = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref, "ctcforge")):
        return None
    if ref not in sys.path:
        sys.path.insert(0, ref)
    from ctcforge import DecoderOptions, EmissionMatrix, TokenDictionary, decode_batch

    idx = np.arange(min(sample_utts, cfg.batch))
    lp, lens = synth.batch(cfg, indices=idx)
    toks = TokenDictionary(tuple(synth.simple_tokens(cfg.vocab)), blank_index=0)
    opts = DecoderOptions(beam_size=cfg.beam, n_best=min(cfg.beam, max(cfg.nbest, 2)),
                          blank_skip_threshold=cfg.threshold)
    ems = [EmissionMatrix(lp[b, : lens[b]]) for b in range(len(idx))]
    t0 = time.perf_counter()
    out = decode_batch(ems, toks, opts, workers=workers)
    dt = time.perf_counter() - t0
    frames = int(lens.sum())
    res = [([h.tokens for h in nb], [h.score for h in nb]) for nb in out]
    return frames / dt, f"first {len(idx)} utterances of {cfg.name} ({frames} frames, {dt:.1f} s incl. process pool)", res


def parity_summary(got, refs, nbest: int, against: str) -> dict:
    """Bench self-check (north-star tolerances): tokens exact unless the
    reference's top-1/top-2 gap is <= 1e-3, scores within 1e-4."""
    mism = near = 0
    err = 0.0
    for (gt, gs), (rt, rs) in zip(got, refs):
        if len(gs) != len(rs[:nbest]):
            mism += 1
            continue
        err = max([err] + [abs(a - b) for a, b in zip(gs, rs)])
        if gt != rt[:nbest]:
            if len(rs) > 1 and rs[0] - rs[1] <= 1e-3:
                near += 1
            else:
                mism += 1
    return {"against": against, "utterances": len(refs), "token_mismatches": mism, "near_tie_excluded": near,
            "max_score_err": err}


def run_reference(args, cfg, rank):
    """--impl reference: the CPU reference path (oracle port) on host cores."""
    if rank != 0:
        return
    import oracle

    oracle.build()
    threads = os.cpu_count() or 1
    lens_all = synth.lengths(cfg)
    per_step = max(threads * 16, 16)
    steps = args.steps + args.warmup
    times, frames = [], []
    for s in range(steps):
        idx = (np.arange(per_step) + s * per_step) % cfg.batch
        lp, lens = synth.batch(cfg, indices=idx)
        t0 = time.perf_counter()
        oracle.decode_batch(lp, lens, threads=threads, beam_size=cfg.beam, n_best=cfg.nbest,
                            blank_skip_threshold=cfg.threshold)
        dt = time.perf_counter() - t0
        if s >= args.warmup:
            times.append(dt)
            frames.append(int(lens_all[idx].sum()))
    value = sum(frames) / sum(times)
    sample = f"{per_step} utterances of {cfg.name} per step ({statistics.mean(frames):.0f} frames)"
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * statistics.mean(times),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": cfg.name, "batch": cfg.batch, "vocab": cfg.vocab, "beam": cfg.beam,
                   "nbest": cfg.nbest, "blank_skip_threshold": cfg.threshold, "sample": sample},
        "cpu_baseline": {"value": value, "unit": "frames/s", "cores": threads, "kind": "port", "sample": sample},
        "e2e": {"value": value, "unit": "frames/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "gpu_launches": 0,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=40)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ctcb", choices=["ctcb", "reference"])
    ap.add_argument("--workload", default="cfg4", choices=sorted(WORKLOADS))
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-validate", action="store_true",
                    help="turn off the input validation fused into the decode (on by default, as in ctcforge)")
    ap.add_argument("--cpu-budget", type=float, default=15.0)
    ap.add_argument("--beam", type=int, default=None, help="override the config's beam (cfg2 sweep: 1/10/50/100)")
    ap.add_argument("--weak", action="store_true",
                    help="weak scaling: N x batch utterances, ~batch per rank; the default is strong scaling, the "
                         "config's fixed batch split over the ranks (BASELINE configs[4])")
    args = ap.parse_args()

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    cfg = synth.CONFIGS[WORKLOADS[args.workload]]
    if args.beam is not None:
        import dataclasses

        cfg = dataclasses.replace(cfg, beam=args.beam, nbest=min(args.beam, 10) if cfg.cfg == 2 else min(cfg.nbest, args.beam))

    if args.impl == "reference":
        run_reference(args, cfg, rank)
        return

    import torch

    from paper_2310_17864_b200 import cuda_ctc_decoder

    # one process per GPU; CTCB_DIST_BACKEND=gloo lets several ranks share a
    # GPU to exercise the multi-rank host path (timing reductions only)
    backend = os.environ.get("CTCB_DIST_BACKEND", "nccl")
    local_dev = local_rank % max(torch.cuda.device_count(), 1)
    torch.cuda.set_device(local_dev)
    dev = torch.device("cuda", local_dev)
    dist = None
    if world > 1:
        import torch.distributed as dist

        if backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(backend)

    # -- this rank's shard (LPT on length), generated straight into pinned memory.
    #    Weak scaling (default): the job is world x batch independent utterances
    #    (global utterance index -> its own seed), LPT-sharded so each rank
    #    holds ~batch; strong: the config's batch is split.
    import dataclasses

    if args.weak and world > 1:
        cfg = dataclasses.replace(cfg, batch=cfg.batch * world)
    lens_all = synth.lengths(cfg)
    shard = lpt_shards(lens_all, world)[rank]
    t_pad = int(lens_all[shard].max())
    host = torch.empty((len(shard), t_pad, cfg.vocab), dtype=torch.float32, pin_memory=True)
    t0 = time.perf_counter()
    _, lens = synth.batch(cfg, indices=shard, out=host.numpy(), t_pad=t_pad, threads=os.cpu_count() or 8)
    log(f"[rank {rank}] generated {len(shard)} utterances ({host.numel() * 4 / 1e9:.2f} GB) in "
        f"{time.perf_counter() - t0:.1f} s")
    lp_dev = host.to(dev, non_blocking=True)
    lens_host = torch.from_numpy(lens)
    lens_dev = lens_host.to(dev)
    torch.cuda.synchronize(dev)

    dec = cuda_ctc_decoder(synth.simple_tokens(cfg.vocab), nbest=cfg.nbest, beam_size=cfg.beam,
                           blank_skip_threshold=cfg.threshold, validate=not args.no_validate)
    frames_rank = int(lens.sum())
    alg_bytes, kept_rank = algorithmic_bytes(host.numpy(), lens, dec.cutoff)

    # -- device-timed decode
    stream = torch.cuda.current_stream(dev)
    clocks = ClockSampler(local_dev).__enter__()
    for _ in range(args.warmup):
        dec.decode(lp_dev, lens_dev)
    torch.cuda.synchronize(dev)
    clocks.wait_ready()
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    dec.kernel_timing(True)  # event pair around the beam kernel of each step (same stream)
    launches0 = dec.launch_count()
    t_mark = time.monotonic()
    # a spin kernel ahead of the start event: the K steps are enqueued while
    # it runs, so host-side stalls (Python, driver locks taken by the clock
    # sampler's nvidia-smi) cannot leave the GPU idle inside the timed region;
    # the region itself still holds exactly the K decode steps.  30 ms was not
    # always enough (one run in ~10 measured 6.2 ms/step around 4.46 ms
    # kernels), so the spin covers 5 ms of host time per step, at least 250 ms
    torch.cuda._sleep(int(max(0.25, 0.005 * args.steps) * 1.9e9))
    ev0.record(stream)
    for _ in range(args.steps):
        out = dec.decode(lp_dev, lens_dev)
    ev1.record(stream)
    torch.cuda.synchronize(dev)
    clocks.mark(t_mark, time.monotonic())
    clocks.__exit__(None, None, None)
    if dist:
        dist.barrier()
    torch.cuda.synchronize(dev)
    ms_rank = ev0.elapsed_time(ev1) / args.steps
    launches = dec.launch_count() - launches0
    k_ms, k_n, k_name = dec.kernel_time()
    dec.kernel_timing(False)
    kernel_ms = k_ms / max(k_n, 1)
    status = out.status.cpu().numpy()
    assert (status == 0).all(), "decode failed"
    # the timed decode's own results, by global utterance index (parity below)
    r_tok, _, r_len, r_sc, r_cnt = dec.to_host(out)
    pos_of = {int(g): j for j, g in enumerate(shard)}

    def got_of(g: int):
        j = pos_of[g]
        n = int(r_cnt[j])
        return ([r_tok[j, q, : r_len[j, q]].tolist() for q in range(n)], [float(r_sc[j, q]) for q in range(n)])

    red_dev = dev if backend == "nccl" else torch.device("cpu")

    def reduce_max(x: float) -> float:
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def reduce_sum(x: float) -> float:
        if not dist:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=red_dev)
        dist.all_reduce(t, op=dist.ReduceOp.SUM)
        return float(t.item())

    ms = reduce_max(ms_rank)
    frames_all = reduce_sum(frames_rank)
    utts_all = reduce_sum(len(shard))
    value = frames_all / (ms / 1e3)

    # roofline of the fused decode kernel on this rank (it is ~all of the step, see profiles/)
    peak, peak_src = measured_peak_gbs()
    achieved = alg_bytes / (kernel_ms / 1e3) / 1e9
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as fh:
            tr = json.load(fh)
        if tr.get("workload") == cfg.name and tr.get("n_gpus", 1) == world and tr.get("kernel") == k_name:
            traffic = tr.get("dram_bytes_per_launch")
    except Exception:
        pass

    # -- end to end through the public API with HOST buffers: CUCTCDecoder(...)
    #    on a pinned CPU tensor -> ctcb_decode_host (valid frames H2D, decode,
    #    results D2H) -> Python hypothesis lists; everything inside the timing
    e2e = None
    if not args.no_e2e:
        e2e_steps = max(1, min(args.steps, 3))
        dec(host, lens_host)  # warm (staging allocation)
        if dist:
            dist.barrier()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        for _ in range(e2e_steps):
            hyps = dec(host, lens_host)
        e2e_rank = (time.perf_counter() - t0) / e2e_steps
        e2e_s = reduce_max(e2e_rank)
        nb = cfg.nbest
        h2d = int(sum(int(n) for n in lens) * cfg.vocab * 4 + lens_host.numel() * 4)
        d2h = int(len(lens) * (nb * (t_pad * 4 + 4 + 8) + 8))
        e2e = {"value": frames_all / e2e_s, "unit": "frames/s", "h2d_bytes_per_step": h2d,
               "d2h_bytes_per_step": d2h, "ms_per_step": 1e3 * e2e_s, "steps": e2e_steps,
               "path": "CUCTCDecoder.__call__(pinned CPU tensor) -> ctcb_decode_host_async (C ABI, host buffers, zero-copy gather + decode + D2H per utterance range, hypotheses built while later ranges run) "
                       "-> CUCTCHypothesis lists"}
        del hyps

    cpu = cpu_ref = None
    parity = []
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        v, sample, refs = cpu_baseline(cfg, args.cpu_budget, threads, sample_utts=512)
        cpu = {"value": v, "unit": "frames/s", "cores": threads, "kind": "port", "sample": sample}
        parity.append(parity_summary([got_of(g) for g in range(len(refs))], refs, cfg.nbest, "oracle port"))
        cf = ctcforge_baseline(cfg, threads, sample_utts=256 if cfg.vocab <= 500 else 32)
        if cf is not None:
            v, sample, refs = cf
            cpu_ref = {"value": v, "unit": "frames/s", "cores": threads, "kind": "reference", "sample": sample,
                       "impl": "ctcforge.decode_batch(workers=cores) from baseline/_ref"}
            parity.append(parity_summary([got_of(g) for g in range(len(refs))], refs, cfg.nbest,
                                         "ctcforge (baseline/_ref)"))

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "frames/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak" if args.weak else "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg.name, "batch": cfg.batch, "batch_per_rank": len(shard), "vocab": cfg.vocab, "beam": cfg.beam,
                       "nbest": cfg.nbest, "blank_skip_threshold": cfg.threshold, "t_range": [cfg.t_min, cfg.t_max],
                       "frames": int(frames_all), "parallelism": f"lpt-shard x{world}",
                       "validate": "off" if args.no_validate else "strict (fused)",
                       "l2": f"inputs larger than L2 ({host.numel() * 4 / 1e9:.1f} GB per rank), no flush"},
            "utterances_per_s": utts_all / (ms / 1e3),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "algorithmic_bytes_per_launch": alg_bytes,
                         "kernel": k_name, "kernel_ms": kernel_ms, "kernel_share_of_step": kernel_ms / ms_rank,
                         "kept_frames": kept_rank},
            "cpu_baseline": cpu,
            "cpu_baseline_reference": cpu_ref,
            "parity": parity,
            "e2e": e2e,
            "clocks": clocks.summary(),
            "gpu_launches": launches,
        }
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
