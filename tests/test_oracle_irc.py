"""Pins of the oracle's coloured-noise (interference-rejection) route, SURVEY.md
§8(f) NEXT-3 (reading R24): W = H^H (H H^H + R_nn)^-1, written in the oracle as
its definition (covariance + LU inversion). Pinned against (1) the white
Gram/Cholesky route when R_nn = sigma2 I, (2) whitening -- R_nn = L L^H,
H~ = L^-1 H, y~ = L^-1 y, white route with sigma2 = 1 -- an independent
algorithm, on random positive-definite R_nn, and (3) the method's purpose:
with strong interference it detects better than the white detector."""
import numpy as np

import oracle
from paper_2510_07843_b200 import synth


def test_white_covariance_equals_gram_route():
    w = synth.generate(2, n_sc=48, n_slots=1)
    R = np.broadcast_to(np.float32(w.sigma2) * np.eye(4, dtype=np.complex64), (w.n_units, 4, 4)).copy()
    a = oracle.detect_irc(w.H_units(), w.y_units(), R, w.qm)
    b = oracle.detect(w.H_units(), w.y_units(), w.sigma2, w.qm, route="chol")
    assert np.max(np.abs(a["xhat"] - b["xhat"])) < 1e-9
    assert np.max(np.abs(a["sinr"] - b["sinr"]) / b["sinr"]) < 1e-9
    assert np.max(np.abs(a["llr"] - b["llr"]) / np.maximum(np.abs(b["llr"]), 1.0)) < 1e-8


def test_whitening_equivalence():
    for k, kw in ((2, dict(n_sc=36, n_slots=1)), (3, dict(n_sc=48, n_slots=1)), (4, dict(n_sc=24, n_slots=1))):
        w = synth.generate_irc(k, n_interf=3, inr_db=15.0, **kw)
        Hu, Yu, R = w.H_units().astype(np.complex128), w.y_units().astype(np.complex128), w.Rnn.astype(np.complex128)
        L = np.linalg.cholesky(R)                                    # R = L L^H
        Ht = np.linalg.solve(L, Hu)                                  # L^-1 H
        Yt = np.linalg.solve(L, np.swapaxes(Yu, 1, 2))               # L^-1 y per RE
        Yt = np.swapaxes(Yt, 1, 2)
        a = oracle.detect_irc(w.H_units(), w.y_units(), w.Rnn, w.qm)
        # the white detector on the whitened (complex64-rounded) system with sigma2 = 1
        b = oracle.detect(Ht.astype(np.complex64), Yt.astype(np.complex64), 1.0, w.qm, route="chol")
        scale = np.maximum(np.abs(b["xhat"]), 1.0)
        assert np.max(np.abs(a["xhat"] - b["xhat"]) / scale) < 2e-5, k
        assert np.max(np.abs(a["sinr"] - b["sinr"]) / b["sinr"]) < 2e-5, k


def test_interference_rejection_beats_white_detector():
    # 8 rx, 4 layers, 2 strong interferers: enough spatial dimensions to reject them
    w = synth.generate_irc(3, n_sc=120, n_slots=2, n_interf=2, inr_db=20.0)
    irc = oracle.detect_irc(w.H_units(), w.y_units(), w.Rnn, w.qm, threads=oracle.max_threads())
    white = oracle.detect(w.H_units(), w.y_units(), w.sigma2, w.qm, threads=oracle.max_threads())
    bits = np.stack([w.bits[synth.unit_re_index(u, w.n_sc, w.sc_per_h)] for u in range(w.n_units)])
    ber_irc = np.mean((irc["llr"] < 0) != bits)
    ber_white = np.mean((white["llr"] < 0) != bits)
    assert ber_irc < 0.1 * ber_white, (ber_irc, ber_white)  # scratch: 0.0098 vs 0.334
