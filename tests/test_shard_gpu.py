"""Multi-GPU strong scaling, emulated on one GPU: every rank's
block of the 2-D slot x PRB partition (shard.block_partition) is detected as its own call --
exactly what rank r runs on its own GPU -- and the reassembled LLRs must be BIT-IDENTICAL to the
unsharded call (H-units are independent: no exchange step, so no result may depend on how the
job is split). A plan on a second device is covered when one is present."""
import pytest
import torch

from paper_2510_07843_b200 import mimo, shard, synth

pytestmark = pytest.mark.gpu


def _detect(w, H, y, n_sc, n_slots, device=0):
    p = mimo.Plan(w.n_rx, w.n_layers, w.qm, sc_per_h=w.sc_per_h, llr_dtype=w.llr, device=device)
    with torch.cuda.device(device):
        out = p.detect(torch.as_tensor(H).to(f"cuda:{device}"), torch.as_tensor(y).to(f"cuda:{device}"),
                       float(w.sigma2), n_sc=n_sc, n_sym=n_slots * synth.SYM_PER_SLOT)
        assert p.sync_status() == 0
    p.close()
    return out.cpu()


@pytest.fixture(scope="module", params=[2, 3, 5])
def job(request):
    w = synth.generate(request.param)  # the full BASELINE configuration
    full = _detect(w, w.H, w.y, w.n_sc, w.n_slots)
    return w, full


@pytest.mark.parametrize("n_gpus", [2, 4, 8])
def test_partition_reassembles_bit_identical(job, n_gpus):
    w, full = job
    blocks = shard.block_partition(w.n_slots, w.n_sc // shard.SC_PER_PRB, n_gpus)
    out = torch.empty_like(full)
    for blk in blocks:
        Hb, yb, nsc, nsl = shard.shard_arrays(w.H, w.y, w.n_slots, w.sc_per_h, blk)
        shard.place_block(out, _detect(w, Hb, yb, nsc, nsl), blk)
    assert torch.equal(out, full), f"{w.name} x{n_gpus}: reassembled LLRs differ from the unsharded call"


def test_plan_on_another_device():
    if torch.cuda.device_count() < 2:
        pytest.skip("one GPU: a plan on device 1 cannot be exercised here")
    w = synth.generate(2, n_sc=96, n_slots=2)
    assert torch.equal(_detect(w, w.H, w.y, w.n_sc, w.n_slots, device=1), _detect(w, w.H, w.y, w.n_sc, w.n_slots))
