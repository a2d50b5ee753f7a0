"""World-size-2 gloo test of the sharded host pipeline (CPU).

Each rank takes its LPT shard of a batch, generates only its utterances from
the per-utterance seeds, decodes them (here with the CPU oracle — on GPU boxes
bench.py does the same with the CUDA decoder) and the results are gathered and
reassembled in batch order.  The reassembled output must equal an unsharded
decode, and the shards must be length-balanced and disjoint.
"""

import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2310_17864_b200 import synth
from paper_2310_17864_b200.shard import balanced_ranges, lpt_shards, merge_shards

CFG = synth.CONFIGS[0]
INDICES = np.arange(4)


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, out_path):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lens_all = synth.lengths(CFG)[INDICES]
    shard = lpt_shards(lens_all, world)[rank]
    lp, lens = synth.batch(CFG, indices=INDICES[shard], threads=1)
    res = oracle.decode_batch(lp, lens, threads=1, beam_size=CFG.beam, n_best=2,
                              blank_skip_threshold=CFG.threshold)
    mine = [(r.tokens, r.scores) for r in res]
    gathered = [None] * world
    dist.all_gather_object(gathered, (shard.tolist(), mine))
    if rank == 0:
        shards = [np.array(g[0], dtype=np.int64) for g in gathered]
        merged = merge_shards(shards, [g[1] for g in gathered], len(INDICES))
        np.save(out_path, np.array([repr(m) for m in merged], dtype=object), allow_pickle=True)
    dist.barrier()
    dist.destroy_process_group()


def test_lpt_shards_balanced_and_disjoint():
    lens = synth.lengths(synth.CONFIGS[4])
    for n in (1, 2, 4, 8):
        shards = lpt_shards(lens, n)
        allidx = np.concatenate(shards)
        assert sorted(allidx.tolist()) == list(range(len(lens)))
        loads = [int(lens[s].sum()) for s in shards]
        assert max(loads) - min(loads) <= int(lens.max())
    with pytest.raises(ValueError):
        lpt_shards(lens, 0)


def test_balanced_ranges_cover_and_balance():
    """Consecutive ranges (the single-process multi-device split): they tile
    the batch in order and each range's load is within one utterance of the
    even share."""
    lens = synth.lengths(synth.CONFIGS[4])
    for n in (1, 2, 3, 4, 8):
        ranges = balanced_ranges(lens, n)
        assert len(ranges) == n and ranges[0][0] == 0 and ranges[-1][1] == len(lens)
        assert all(a[1] == b[0] for a, b in zip(ranges, ranges[1:]))
        share = lens.sum() / n
        for b0, b1 in ranges:
            assert abs(int(lens[b0:b1].sum()) - share) <= 2 * int(lens.max())
    # more parts than utterances: empty ranges, still a tiling; zero lengths count as 1
    r = balanced_ranges([5, 0, 7], 5)
    assert r[0][0] == 0 and r[-1][1] == 3 and all(b0 <= b1 for b0, b1 in r)
    assert sum(b1 - b0 for b0, b1 in r) == 3
    assert balanced_ranges([], 3) == [(0, 0)] * 3
    with pytest.raises(ValueError):
        balanced_ranges([1, 2], 0)


def test_sharded_decode_equals_unsharded(tmp_path):
    out = tmp_path / "merged.npy"
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(out)), nprocs=2, join=True)
    merged = np.load(out, allow_pickle=True).tolist()
    lp, lens = synth.batch(CFG, indices=INDICES, threads=1)
    ref = oracle.decode_batch(lp, lens, threads=1, beam_size=CFG.beam, n_best=2,
                              blank_skip_threshold=CFG.threshold)
    assert merged == [repr((r.tokens, r.scores)) for r in ref]
