"""GPU parity of the non-default kernel variants (selected by name through the plan
descriptor's `kernel` field): every variant compiled into libmimo.so must produce
oracle-exact results too.
Same tolerances as test_parity_gpu.py (tests/parity.py)."""
import numpy as np
import pytest

import parity
from paper_2510_07843_b200 import synth

pytestmark = pytest.mark.gpu

C5_VARIANTS = ["c5_fused_64x16_q6_i8", "c5_fusedbi_64x16_q6_i8", "c5_fusedbid_64x16_q6_i8", "c5_fusedbiw_64x16_q6_i8", "c5_fusedbie_64x16_q6_i8", "c5_fused3_64x16_q6_i8", "c5_bf16_tcs_be_64x16_q6_i8", "c5_bf16kc_tcs_be_64x16_q6_i8",
               "c5_bf16_tcs_64x16_q6_i8", "c5_bf16_gj_64x16_q6_i8", "c5_bf16_chol_64x16_q6_i8", "c5_tf32_gj_64x16_q6_i8",
               "big_64x16_q6_i8"]
C4_VARIANTS = ["lg3hl_16x8_q8_f16", "lg3hl2_16x8_q8_f16", "lg3hq_16x8_q8_f16", "lg3hp_16x8_q8_f16", "lg3_16x8_q8_f16", "lg_16x8_q8_f16"]
C3_VARIANTS = ["stream_8x4_q6_i8", "split_8x4_q6_i8", "prb_8x4_q6_i8"]


def _forced(monkeypatch, name, w, **kw):
    g = parity.run_gpu(w, kernel=name, **kw)
    assert g["kernel"] == name, f"forced {name}, plan selected {g['kernel']}"
    assert g["n_failed"] == 0
    return g


@pytest.mark.parametrize("name", C5_VARIANTS)
def test_c5_variant(monkeypatch, name):
    # 4 slots x 273 PRBs = 1092 units: > 7 units per CTA of the 148-CTA persistent grids, so the
    # stage / TMEM / B-operand rings of the persistent c5 kernels wrap several times
    w = synth.generate(5, n_sc=3276, n_slots=4)
    g = _forced(monkeypatch, name, w, xhat=False, sinr=True)
    rng = np.random.default_rng(7)
    edges = [0, 1, 147, 148, 295, 296, 297, 591, 592, 887, 888, 889, 1090, 1091]
    units = np.unique(np.concatenate([edges, rng.choice(w.n_units, 24, replace=False)]))
    print(name, parity.compare(w, g, units))


@pytest.mark.parametrize("name", C4_VARIANTS)
def test_c4_variant(monkeypatch, name):
    w = synth.generate(4, n_sc=300, n_slots=2)
    g = _forced(monkeypatch, name, w)
    print(name, parity.compare(w, g))


@pytest.mark.parametrize("name", C3_VARIANTS)
def test_c3_variant(monkeypatch, name):
    w = synth.generate(3, n_sc=300, n_slots=2)
    g = _forced(monkeypatch, name, w)
    print(name, parity.compare(w, g))


def test_c5_repeated_calls_and_sinr():
    """Back-to-back calls on one plan (PDL overlap of call i+1's setup with call i's stores) give
    identical results, and every unit's SINR is set."""
    import torch
    from paper_2510_07843_b200 import mimo
    w = synth.generate(5, n_sc=3276, n_slots=4)
    p = mimo.Plan(64, 16, 6, sc_per_h=12, llr_dtype="i8", overlap_calls=True)
    H, y = torch.from_numpy(w.H).cuda(), torch.from_numpy(w.y).cuda()
    sinr = torch.full(p.shapes(w.n_sc, w.n_sym)["sinr"], -1.0, device="cuda")
    a = p.detect(H, y, float(w.sigma2), sinr=sinr).clone()
    for _ in range(3):
        b = p.detect(H, y, float(w.sigma2))
    assert p.sync_status() == 0
    assert torch.equal(a, b)
    assert bool((sinr > 0).all())
    p.close()
