"""Degenerate cases on the C3, C4 and C5 default kernels (test_parity_gpu.py covers them on C2):
zero forcing (sigma2 = 0, readings R11), rank-deficient and NaN units flagged and zeroed
(R17), a zero column at sigma2 > 0 erased without a failure (R19)."""
import numpy as np
import pytest

import parity
from paper_2510_07843_b200 import synth

pytestmark = pytest.mark.gpu

SMALL = {3: dict(n_sc=96, n_slots=1), 4: dict(n_sc=48, n_slots=1), 5: dict(n_sc=48, n_slots=1)}
TYPE_MAX = {"i8": 127, "f16": 65504.0, "f32": np.finfo(np.float32).max}
# (config, kernel): the default kernel of C3 / C4 / C5, plus every C5 setup route
CASES = [(3, None), (4, None), (5, None), (5, "c5_fused3_64x16_q6_i8"), (5, "c5_bf16_tcs_be_64x16_q6_i8"), (5, "c5_bf16_gj_64x16_q6_i8"),
         (5, "c5_bf16_chol_64x16_q6_i8"), (5, "c5_tf32_gj_64x16_q6_i8")]


def _unit_llr(w, g, u):
    return g["llr"][synth.unit_re_index(u, w.n_sc, w.sc_per_h, w.sym_per_h)]


@pytest.mark.parametrize("k,kernel", CASES)
def test_zero_forcing(k, kernel):
    w = synth.generate(k, **SMALL[k], sigma2=0.0)
    g = parity.run_gpu(w, kernel=kernel)
    assert g["n_failed"] == 0
    assert np.all(np.isinf(g["sinr"]))
    assert np.all(np.abs(g["llr"].astype(np.float64)) == TYPE_MAX[w.llr])
    parity.compare(w, g)


@pytest.mark.parametrize("k,kernel", CASES)
def test_rank_deficient_and_nan_units_flagged(k, kernel):
    w = synth.generate(k, **SMALL[k], sigma2=0.0)
    H = w.H.copy()
    Hu = H.reshape(w.n_units, w.n_rx, w.n_layers)
    Hu[1, :, 2] = 0                      # zero column -> pivot exactly 0 at sigma2 = 0
    Hu[2, :, 1] = Hu[2, :, 0]            # duplicate column
    Hu[3, 1, 1] = np.nan                 # NaN entry
    g = parity.run_gpu(w, H=H, kernel=kernel)
    assert g["n_failed"] == 3
    for u in (1, 2, 3):
        assert not np.any(_unit_llr(w, g, u).astype(np.float64))
        assert np.all(g["sinr"].reshape(w.n_units, -1)[u] == 0)
    ok = [u for u in range(w.n_units) if u not in (1, 2, 3)]
    parity.compare(w, g, ok, H=H)


@pytest.mark.parametrize("k,kernel", CASES)
def test_zero_column_erasure(k, kernel):
    w = synth.generate(k, **SMALL[k])
    H = w.H.copy()
    H.reshape(w.n_units, w.n_rx, w.n_layers)[1, :, 1] = 0
    g = parity.run_gpu(w, H=H, kernel=kernel)
    assert g["n_failed"] == 0
    assert not np.any(_unit_llr(w, g, 1)[..., 1, :].astype(np.float64))
    parity.compare(w, g, H=H)
