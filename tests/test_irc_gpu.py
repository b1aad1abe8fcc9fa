"""GPU parity of the coloured-noise / interference-rejection detector
(mimo_detect_irc, reading R24) against the oracle's
definition-form route (W = H^H (H H^H + R_nn)^-1, oracle.detect_irc), with the
north_star tolerances; R_nn = sigma2 I reproduces mimo_detect_mmse."""
import numpy as np
import pytest
import torch

import parity
import oracle
from paper_2510_07843_b200 import mimo, synth

pytestmark = pytest.mark.gpu


def run_irc(w, R=None):
    p = mimo.Plan(w.n_rx, w.n_layers, w.qm, sc_per_h=w.sc_per_h, llr_dtype=w.llr)
    sh = p.shapes(w.n_sc, w.n_sym)
    x = torch.empty(sh["xhat"], dtype=torch.complex64, device="cuda")
    s = torch.empty(sh["sinr"], dtype=torch.float32, device="cuda")
    R = w.Rnn if R is None else R
    out = p.detect_irc(torch.from_numpy(w.H).cuda(), torch.from_numpy(w.y).cuda(), torch.from_numpy(R).cuda(),
                       xhat=x, sinr=s)
    nf = p.sync_status()
    p.close()
    return dict(llr=out.cpu().numpy(), xhat=x.cpu().numpy(), sinr=s.cpu().numpy(), n_failed=nf)


def compare_irc(w, g):
    units = np.arange(w.n_units)
    ref = oracle.detect_irc(w.H_units(), w.y_units(), w.Rnn, w.qm, threads=oracle.max_threads())
    gx = parity.gather_units(w, g["xhat"], units)
    err = np.abs(gx - ref["xhat"]) / np.maximum(np.abs(ref["xhat"]), 1.0)
    assert err.max() <= parity.TOL_X, err.max()
    rel = np.abs(g["sinr"].astype(np.float64) - ref["sinr"]) / np.maximum(ref["sinr"], 1e-3)
    assert rel.max() <= parity.TOL_SINR, rel.max()
    rep = parity.compare_llr(parity.gather_units(w, g["llr"], units), ref["llr"], w.llr)
    return dict(xhat_max_err=float(err.max()), sinr_max_rel=float(rel.max()), **rep)


@pytest.mark.parametrize("k,kw", [(1, dict()), (2, dict(n_sc=120, n_slots=2)), (3, dict(n_sc=120, n_slots=2)),
                                  (4, dict(n_sc=48, n_slots=1))])
def test_irc_matches_oracle(k, kw):
    w = synth.generate_irc(k, n_interf=2, inr_db=15.0, **kw)
    g = run_irc(w)
    assert g["n_failed"] == 0
    print(k, compare_irc(w, g))


def test_white_covariance_equals_mmse():
    w = synth.generate(2, n_sc=120, n_slots=1)
    R = np.broadcast_to(np.float32(w.sigma2) * np.eye(4, dtype=np.complex64), (w.n_units, 4, 4)).copy()
    a = run_irc(w, R)
    b = parity.run_gpu(w)
    err = np.abs(a["xhat"] - b["xhat"]) / np.maximum(np.abs(b["xhat"]), 1.0)
    assert err.max() <= 1e-5
    assert np.abs(a["llr"] - b["llr"]).max() <= 1e-3 * max(1.0, np.abs(b["llr"]).max())


def test_non_pd_covariance_flagged():
    w = synth.generate_irc(2, n_sc=24, n_slots=1)
    R = w.Rnn.copy()
    R[3] = 0  # unit 3: R_nn = 0 is not positive definite
    g = run_irc(w, R)
    assert g["n_failed"] == 1
    assert np.all(g["sinr"][3] == 0)


def test_unsupported_nr():
    p = mimo.Plan(64, 16, 6, sc_per_h=12, llr_dtype="i8")
    w = synth.generate(5, n_sc=12, n_slots=1)
    R = np.zeros((w.n_units, 64, 64), np.complex64)
    with pytest.raises(mimo.MimoError) as e:
        p.detect_irc(torch.from_numpy(w.H).cuda(), torch.from_numpy(w.y).cuda(), torch.from_numpy(R).cuda())
    assert e.value.status == mimo.MIMO_ERR_UNSUPPORTED
