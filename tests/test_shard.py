"""Multi-rank host logic on CPU (gloo, world_size 2): slot partitioning, per-rank
seeding, max-over-ranks timing, and result placement (gather + reassembly).

The detector itself needs a GPU; here each rank runs the fp64 oracle on its
shard (test infrastructure), and rank 0 checks that the gathered shards equal
the oracle run on the concatenated job -- i.e. the sharding loses or
duplicates nothing and needs no exchange step (no collective on the data path).
"""
import os
import socket
import sys

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2510_07843_b200 import shard, synth

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_slot_partition_properties():
    for n in (1, 7, 10, 40, 273):
        for w in (1, 2, 3, 4, 8):
            parts = shard.slot_partition(n, w)
            assert len(parts) == w
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(parts[i][1] == parts[i + 1][0] for i in range(w - 1))
            sizes = [b - a for a, b in parts]
            assert max(sizes) - min(sizes) <= 1
    assert shard.weak_slots(10, 3) == (30, 40)
    assert len({shard.shard_seed(1002, r) for r in range(8)}) == 8


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q):
    sys.path.insert(0, ROOT)
    import torch.distributed as dist
    import oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # strong-scaling view: a 6-slot C2-shaped job split by slot over the ranks
        n_slots, n_sc = 6, 24
        w = synth.generate(2, n_sc=n_sc, n_slots=n_slots)
        s0, s1 = shard.slot_partition(n_slots, world)[rank]
        Hu = w.H_units().reshape(n_slots, n_sc, 4, 4)[s0:s1].reshape(-1, 4, 4)
        y = w.y[s0 * 14:s1 * 14]
        Yu = synth.unit_gather(y, s1 - s0, n_sc, 1)
        r = oracle.detect(Hu, Yu, w.sigma2, w.qm)
        local = synth.unit_scatter(r["llr"], s1 - s0, n_sc, 1)   # [sym][sc][nl][qm]
        t = shard.max_over_ranks(0.5 + rank)                    # max over ranks
        n = shard.sum_over_ranks(float(local.shape[0]))
        full = shard.gather_slot_blocks(local, world)
        if rank == 0:
            ref = oracle.detect(w.H_units(), w.y_units(), w.sigma2, w.qm)
            ref_grid = synth.unit_scatter(ref["llr"], n_slots, n_sc, 1)
            out_q.put((t, n, bool(np.array_equal(full, ref_grid)), full.shape))
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_shard_and_gather():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    t, n, equal, shape = q.get(timeout=5)
    assert t == 1.5            # max over ranks of 0.5 + rank
    assert n == 6 * 14         # every symbol of the job processed exactly once
    assert equal and shape == (84, 24, 4, 4)
