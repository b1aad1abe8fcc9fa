"""GPU parity of mimo_detect_mmse_sv (per-slot noise variance):
every H time block t is detected with its own sigma2_v[t]; the fp64 oracle runs
each slot's units with that slot's scalar sigma2 (tests/parity.py tolerances)."""
import dataclasses

import numpy as np
import pytest

import parity
from paper_2510_07843_b200 import synth

pytestmark = pytest.mark.gpu

SMALL = {1: dict(n_slots=3), 2: dict(n_sc=300, n_slots=3), 3: dict(n_sc=300, n_slots=3),
         4: dict(n_sc=300, n_slots=3), 5: dict(n_sc=120, n_slots=3)}


def _per_slot_sigma2(w, seed):
    rng = np.random.default_rng(seed)
    n_blk = w.n_sym // w.sym_per_h
    return (w.sigma2 * 10.0 ** rng.uniform(-1.0, 1.0, n_blk)).astype(np.float32)


def _run(w, s2v, **kw):
    import torch
    from paper_2510_07843_b200 import mimo
    plan = mimo.Plan(w.n_rx, w.n_layers, w.qm, sc_per_h=w.sc_per_h, sym_per_h=w.sym_per_h, llr_dtype=w.llr)
    Hd, yd = torch.from_numpy(w.H).cuda(), torch.from_numpy(w.y).cuda()
    sh = plan.shapes(w.n_sc, w.n_sym)
    xd = torch.empty(sh["xhat"], dtype=torch.complex64, device="cuda") if kw.get("xhat", True) else None
    sd = torch.empty(sh["sinr"], dtype=torch.float32, device="cuda")
    out = plan.detect(Hd, yd, torch.from_numpy(s2v).cuda(), xhat=xd, sinr=sd)
    res = dict(llr=out.cpu().numpy(), n_failed=plan.sync_status(), kernel=plan.kernel_name, sinr=sd.cpu().numpy())
    if xd is not None:
        res["xhat"] = xd.cpu().numpy()
    plan.close()
    return res


def _compare_by_slot(w, g, s2v):
    n_fb = w.n_sc // w.sc_per_h
    for t, s2 in enumerate(s2v):
        units = np.arange(t * n_fb, (t + 1) * n_fb)
        parity.compare(dataclasses.replace(w, sigma2=float(s2)), g, units)


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_per_slot_sigma2_matches_oracle(k):
    w = synth.generate(k, **SMALL[k])
    s2v = _per_slot_sigma2(w, 40 + k)
    g = _run(w, s2v, xhat=(k != 5))
    assert g["n_failed"] == 0
    _compare_by_slot(w, g, s2v)


def test_per_block_sigma2_time_varying_generic():
    """sym_per_h = 7: one variance per H time block (two per slot), on the shape's sym_per_h = 7
    kernel (tpu_4x4_q4_f32_s7)."""
    cfg = dict(synth.CONFIGS[2], n_sc=48, n_slots=2, sym_per_h=7)
    w = synth.generate(cfg, seed=5)
    s2v = _per_slot_sigma2(w, 6)
    assert len(s2v) == 4
    g = _run(w, s2v)
    assert g["n_failed"] == 0
    _compare_by_slot(w, g, s2v)


@pytest.mark.parametrize("k", [2, 3, 5])
def test_constant_array_equals_scalar_path(k):
    """An all-equal sigma2_v gives exactly the scalar call's LLRs."""
    w = synth.generate(k, **SMALL[k])
    g_v = _run(w, np.full(w.n_sym // w.sym_per_h, w.sigma2, np.float32), xhat=False)
    g_s = parity.run_gpu(w, xhat=False)
    assert np.array_equal(g_v["llr"], g_s["llr"])


@pytest.mark.parametrize("k", [2, 3, 4, 5])
def test_bad_entries_flag_their_slot_only(k):
    """0, negative and NaN entries are not allowed on this path: that slot's units are flagged
    (zeroed, counted); the other slots are unaffected."""
    w = synth.generate(k, **dict(SMALL[k], n_slots=4))
    s2v = np.full(4, w.sigma2, np.float32)
    s2v[1], s2v[2], s2v[3] = 0.0, np.nan, -1.0
    g = _run(w, s2v, xhat=False)
    n_fb = w.n_sc // w.sc_per_h
    assert g["n_failed"] == 3 * n_fb
    parity.compare(w, g, np.arange(n_fb))  # slot 0 unaffected
    llr = g["llr"].reshape(w.n_sym, w.n_sc, -1)
    assert not np.any(llr[14:].astype(np.float64))
    assert not np.any(g["sinr"].reshape(4, n_fb, -1)[1:])
