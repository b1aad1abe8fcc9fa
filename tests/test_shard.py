"""Multi-rank host logic on CPU (gloo, world_size 2): the 2-D slot x PRB block partition,
max-over-ranks timing, and result placement (gather + reassembly).

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
    assert len({shard.shard_seed(1002, r) for r in range(8)}) == 8


@pytest.mark.parametrize("n_slots,n_prb", [(40, 273), (10, 273), (20, 273), (1, 1), (6, 4), (7, 5)])
def test_block_partition_covers_job_once(n_slots, n_prb):
    """a = gcd(n_slots, g) slot groups x g/a PRB groups; every (slot, PRB) owned
    exactly once, balanced to within one slot / PRB."""
    for g in (1, 2, 3, 4, 8):
        if g // np.gcd(n_slots, g) > n_prb:
            with pytest.raises(ValueError):
                shard.block_partition(n_slots, n_prb, g)
            continue
        parts = shard.block_partition(n_slots, n_prb, g)
        own = np.zeros((n_slots, n_prb), int)
        for b in parts:
            (s0, s1), (p0, p1) = b["slots"], b["prbs"]
            own[s0:s1, p0:p1] += 1
        assert (own == 1).all()
        a, bb = parts[0]["grid"]
        assert a * bb == g and a == np.gcd(n_slots, g)
        ns = [b["slots"][1] - b["slots"][0] for b in parts]
        npr = [b["prbs"][1] - b["prbs"][0] for b in parts]
        assert max(ns) - min(ns) <= 1 and max(npr) - min(npr) <= 1


def test_block_partition_survey_examples():
    # C5 over 8 GPUs: 5 slots each, whole band (north_star "sharded by slot across 8 GPUs")
    p = shard.block_partition(40, 273, 8)
    assert all(b["slots"][1] - b["slots"][0] == 5 and b["prbs"] == (0, 273) for b in p)
    # C2 over 4 GPUs: 2 slot groups x 2 PRB groups; C2 over 8: 2 x 4 with 69/68/68/68 PRBs
    assert shard.block_partition(10, 273, 4)[0]["grid"] == (2, 2)
    p8 = shard.block_partition(10, 273, 8)
    assert p8[0]["grid"] == (2, 4)
    assert sorted({b["prbs"][1] - b["prbs"][0] for b in p8}) == [68, 69]


@pytest.mark.parametrize("k,sc_per_h", [(2, 1), (3, 12)])
def test_shard_arrays_and_place_block_roundtrip(k, sc_per_h):
    w = synth.generate(k, n_sc=60, n_slots=4)
    for g in (2, 4, 8):
        full = np.zeros_like(w.y)
        for b in shard.block_partition(4, 5, g):
            Hb, yb, nsc, nsl = shard.shard_arrays(w.H, w.y, 4, sc_per_h, b)
            assert Hb.flags.c_contiguous and yb.flags.c_contiguous
            assert yb.shape == (nsl * 14, nsc, w.n_rx) and Hb.shape == (nsl, nsc // sc_per_h, w.n_rx, w.n_layers)
            shard.place_block(full, yb, b)
        assert np.array_equal(full, w.y)


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
        # strong scaling: one seeded 3-slot x 2-PRB C2-shaped job, 2-D block partition over the
        # ranks (3 slots, world 2 -> 1 slot group x 2 PRB groups), each rank detects its block
        n_slots, n_sc = 3, 24
        w = synth.generate(2, n_sc=n_sc, n_slots=n_slots)
        blk = shard.block_partition(n_slots, n_sc // 12, world)[rank]
        Hb, yb, nsc, nsl = shard.shard_arrays(w.H, w.y, n_slots, 1, blk)
        r = oracle.detect(Hb.reshape(-1, 4, 4), synth.unit_gather(yb, nsl, nsc, 1), w.sigma2, w.qm)
        local = synth.unit_scatter(r["llr"], nsl, nsc, 1)        # [sym][sc][nl][qm]
        t = shard.max_over_ranks(0.5 + rank)                    # max over ranks
        n = shard.sum_over_ranks(float(local.shape[0] * local.shape[1]))
        parts = shard.gather_objects((blk, local), world)       # result placement (untimed)
        if rank == 0:
            full = np.zeros((n_slots * 14, n_sc, 4, 4), np.float64)
            for b, part in parts:
                shard.place_block(full, part, b)
            ref = oracle.detect(w.H_units(), w.y_units(), w.sigma2, w.qm)
            ref_grid = synth.unit_scatter(ref["llr"], n_slots, n_sc, 1)
            out_q.put((t, n, bool(np.array_equal(full, ref_grid)), full.shape))
        # the placement bench.py times at N > 1: blocks sent point to point to rank 0 as tensors
        import torch
        blocks = shard.block_partition(n_slots, n_sc // 12, world)
        full_shape = (n_slots * 14, n_sc, 4, 4)
        assert tuple(local.shape) == shard.block_llr_shape(blk, full_shape)
        placed = shard.place_blocks_p2p(torch.from_numpy(np.ascontiguousarray(local)), blocks, full_shape)
        if rank == 0:
            out_q.put(bool(np.array_equal(placed.numpy(), ref_grid)))
        else:
            assert placed is None
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
    assert n == 3 * 14 * 24    # every RE of the job processed exactly once
    assert equal and shape == (42, 24, 4, 4)
    assert q.get(timeout=5)    # point-to-point placement into rank 0's full grid: bit-identical
