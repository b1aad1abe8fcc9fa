"""Generator pins and layout helpers. CPU only."""
import numpy as np
import pytest

from paper_2510_07843_b200 import synth


@pytest.mark.parametrize("qm", [2, 4, 6, 8])
def test_constellation_unit_power(qm):
    lab = np.arange(1 << qm)
    lb = ((lab[:, None] >> (qm - 1 - np.arange(qm))) & 1).astype(np.uint8)
    pts = synth.qam_modulate(lb, qm)
    assert abs(np.mean(np.abs(pts) ** 2) - 1) <= 1e-12
    assert len(np.unique(np.round(pts, 12))) == 1 << qm


def test_qpsk_00():
    assert np.isclose(synth.qam_modulate(np.array([0, 0], np.uint8), 2), (1 + 1j) / np.sqrt(2))


def test_awgn_variance_and_determinism():
    w = synth.generate(1, n_sc=12 * 600, n_slots=6, noiseless=False, H_override=np.zeros((2, 2)))
    # H = 0 -> y is pure noise CN(0, sigma^2); 1e6 complex samples
    v = np.mean(np.abs(w.y.astype(np.complex128)) ** 2)
    assert abs(v / np.float64(w.sigma2) - 1) < 0.01
    assert abs(np.var(w.y.real) / (w.sigma2 / 2) - 1) < 0.01
    w2 = synth.generate(1, n_sc=12 * 600, n_slots=6, H_override=np.zeros((2, 2)))
    assert np.array_equal(w.y, w2.y) and w.sha256() == w2.sha256()


def test_kronecker_correlation():
    w = synth.generate(3, n_sc=12 * 273, n_slots=4)
    H = w.H_units().astype(np.complex128)             # [u][8][4]
    Rr = np.einsum("uik,ujk->ij", H, H.conj()) / (H.shape[0] * 4)   # E[H H^H]/nl = R_r
    ref = 0.5 ** np.abs(np.subtract.outer(np.arange(8), np.arange(8)))
    assert np.abs(Rr - ref).max() < 0.05
    Rt = np.einsum("uki,ukj->ij", H, H.conj()) / (H.shape[0] * 8)
    ref_t = 0.5 ** np.abs(np.subtract.outer(np.arange(4), np.arange(4)))
    assert np.abs(Rt.T - ref_t).max() < 0.05


def test_sigma2_readings():
    assert synth.sigma2_of(10.0) == np.float32(0.1)                   # C1 "sigma^2 = 0.1"
    assert np.isclose(synth.sigma2_of(28.0), 10 ** -2.8, rtol=1e-7)


@pytest.mark.parametrize("scph", [1, 12])
def test_unit_gather_roundtrip(scph):
    nsl, nsc = 2, 36
    g = np.arange(nsl * 14 * nsc * 3).reshape(nsl * 14, nsc, 3)
    u = synth.unit_gather(g, nsl, nsc, scph)
    assert u.shape == (nsl * nsc // scph, 14 * scph, 3)
    assert np.array_equal(synth.unit_scatter(u, nsl, nsc, scph), g)
    for unit in [0, 5, u.shape[0] - 1]:
        s, f = synth.unit_re_index(unit, nsc, scph)
        assert np.array_equal(u[unit], g[s, f])


def test_noiseless_y_is_Hx():
    w = synth.generate(2, n_sc=8, n_slots=1, noiseless=True)
    x = synth.qam_modulate(w.bits, w.qm)                # [14][8][4]
    H = w.H.reshape(8, 4, 4).astype(np.complex128)
    ref = np.einsum("frl,sfl->sfr", H, x)
    assert np.abs(w.y - ref).max() < 1e-6


def test_algorithmic_bytes_c2():
    b = synth.config_algorithmic_bytes(2)
    assert b["n_re"] == 458640 and b["n_units"] == 32760
    assert b["total"] == 32760 * 128 + 458640 * 32 + 458640 * 64
