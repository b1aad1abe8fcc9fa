"""Pins of the fp64 oracle against things other than itself.

Each pin is a closed form, a textbook special case, a library routine used as an
independent computation (numpy/LAPACK), an identity between two different
algorithms, brute force on tiny inputs, or a hand-worked golden fixture
(tests/golden/). A plausible oracle mistake (dropped sigma^2 term, wrong
conjugation, transposed operand, wrong sign/bit order, missing unbiasing) fails
at least one of them. CPU only.
"""
import itertools
import json
import os

import numpy as np
import pytest

import oracle
from paper_2510_07843_b200 import synth

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")
RNG = np.random.default_rng(7)


def cn(shape, rng=RNG):
    return (rng.standard_normal(shape) + 1j * rng.standard_normal(shape)) / np.sqrt(2)


def c64(a):
    return np.asarray(a).astype(np.complex64)


# ---------------------------------------------------------------- P1 Gram --
def test_p1_gram_special_cases():
    for nr, nl in [(2, 2), (4, 2), (8, 8)]:
        assert np.array_equal(oracle.gram(np.zeros((nr, nl)), 0.25), 0.25 * np.eye(nl))
    assert np.allclose(oracle.gram(np.eye(4), 0.1), 1.1 * np.eye(4), atol=1e-15)


@pytest.mark.parametrize("nr,nl", [(1, 1), (2, 2), (4, 4), (8, 4), (16, 8), (64, 16)])
def test_p1_gram_vs_numpy(nr, nl):
    H = cn((nr, nl))
    G = oracle.gram(H, 0.3)
    ref = H.conj().T @ H + 0.3 * np.eye(nl)
    assert np.abs(G - ref).max() <= 1e-12 * max(1, np.abs(ref).max())
    assert np.allclose(G, G.conj().T, atol=0)


def test_covariance_vs_numpy():
    H = cn((8, 4))
    R = oracle.covariance(H, 0.2)
    assert np.abs(R - (H @ H.conj().T + 0.2 * np.eye(8))).max() < 1e-13


# ------------------------------------------------------------ P2 Cholesky --
@pytest.mark.parametrize("n", [1, 2, 4, 8, 16])
def test_p2_cholesky_vs_lapack(n):
    H = cn((2 * n, n))
    G = H.conj().T @ H + 0.05 * np.eye(n)
    L = oracle.cholesky(G)
    assert L is not None
    assert np.allclose(np.triu(L, 1), 0)
    assert np.all(np.diag(L).real > 0) and np.allclose(np.diag(L).imag, 0)
    assert np.abs(L @ L.conj().T - G).max() <= 1e-13 * np.abs(G).max()
    assert np.abs(L - np.linalg.cholesky(G)).max() <= 1e-12 * np.abs(L).max()


def test_p2_cholesky_guard():
    # zero column at sigma^2 = 0 -> pivot exactly 0 -> flagged (reading R17)
    H = cn((4, 3))
    H[:, 1] = 0
    assert oracle.cholesky(oracle.gram(H, 0.0)) is None
    # duplicate column at sigma^2 = 0 -> rank deficient -> flagged
    H = cn((4, 3))
    H[:, 2] = H[:, 0]
    assert oracle.cholesky(oracle.gram(H, 0.0)) is None
    # NaN -> flagged
    G = np.eye(3, dtype=complex)
    G[1, 1] = np.nan
    assert oracle.cholesky(G) is None
    # tau is 16 fp32 unit roundoffs, relative to max diagonal
    assert oracle.pivot_tau() == 16 * 2.0 ** -24
    s = 1e3
    assert oracle.cholesky(np.diag([s, s * 2e-6])) is not None
    assert oracle.cholesky(np.diag([s, s * 5e-7])) is None


# -------------------------------------------------------------- LU (paper) --
def test_lu_spec_examples():
    LU, perm = oracle.lu_factor(np.eye(4))
    assert np.array_equal(LU, np.eye(4)) and list(perm) == [0, 1, 2, 3]
    LU, perm = oracle.lu_factor(np.diag([2.0, 4.0]))
    assert np.array_equal(LU, np.diag([2.0, 4.0]))
    # forward substitution closed form, L = [[1,0],[c,1]]
    c = 0.3 - 0.2j
    LUc = np.array([[1, 0], [c, 1]], dtype=complex)
    b = np.array([1 + 1j, 2 - 1j])
    z = oracle.lu_forward(LUc, [0, 1], b)
    assert np.allclose(z, [b[0], b[1] - c * b[0]], atol=1e-15)
    # backward closed form, U = diag(2,4), z = [2,4] -> x = [1,1]
    assert np.allclose(oracle.lu_backward(np.diag([2.0, 4.0]), [2, 4]), [1, 1])
    assert np.allclose(oracle.lu_invert(np.diag([2.0, 4.0])), np.diag([0.5, 0.25]))
    assert np.array_equal(oracle.lu_invert(np.eye(3)), np.eye(3))


@pytest.mark.parametrize("n", [2, 4, 8, 16])
def test_lu_reconstruction_and_inverse(n):
    A = cn((n, n)) + 0.1 * np.eye(n)
    LU, perm = oracle.lu_factor(A)
    L = np.tril(LU, -1) + np.eye(n)
    U = np.triu(LU)
    assert sorted(perm) == list(range(n))
    assert np.linalg.norm(A[perm] - L @ U) <= 1e-12 * np.linalg.norm(A)
    X = oracle.lu_invert(A)
    assert np.linalg.norm(A @ X - np.eye(n)) <= 1e-10
    assert np.abs(X - np.linalg.inv(A)).max() <= 1e-10 * np.abs(X).max()


# --------------------------------------------------- P3 push-through, P4 ----
@pytest.mark.parametrize("nr,nl,s2", [(2, 2, 0.1), (4, 4, 0.0316), (8, 4, 0.01), (16, 8, 0.002),
                                      (64, 16, 0.01), (4, 1, 0.5)])
def test_p3_push_through(nr, nl, s2):
    """W = (H^H H + s2 I)^-1 H^H (Gram/Cholesky) == H^H (H H^H + s2 I)^-1 (covariance/LU)."""
    H = cn((nr, nl))
    Wc = oracle.weights_chol(H, s2)
    Wl = oracle.weights_lu(H, s2)
    assert np.abs(Wc - Wl).max() <= 1e-11 * np.abs(Wc).max()
    # and against numpy's solve as a library computation
    ref = np.linalg.solve(H.conj().T @ H + s2 * np.eye(nl), H.conj().T)
    assert np.abs(Wc - ref).max() <= 1e-11 * np.abs(ref).max()


def test_p4_identity_channel():
    assert np.allclose(oracle.weights_chol(np.eye(2), 0.0), np.eye(2), atol=1e-15)
    assert np.allclose(oracle.weights_chol(np.eye(2), 1.0), 0.5 * np.eye(2), atol=1e-15)
    assert np.allclose(oracle.weights_lu(np.eye(2), 1.0), 0.5 * np.eye(2), atol=1e-15)


# --------------------------------------------------------------- P5 ZF ------
def _detect1(H, y, s2, qm, route="chol"):
    """Detect one unit with REs y [n_re][nr]."""
    r = oracle.detect(c64(H)[None], c64(y)[None], s2, qm, route=route)
    return {k: (v[0] if isinstance(v, np.ndarray) else v) for k, v in r.items()}


def test_p5_zero_forcing_square_adjugate():
    H = c64(cn((2, 2)))
    y = c64(cn((5, 2)))
    a, b, c, d = H.astype(np.complex128).ravel()
    Hinv = np.array([[d, -b], [-c, a]]) / (a * d - b * c)
    r = _detect1(H, y, 0.0, 2)
    ref = (Hinv @ y.astype(np.complex128).T).T
    cond = np.linalg.cond(H.astype(np.complex128))
    assert np.abs(r["xhat"] - ref).max() <= 1e-12 * cond * np.abs(ref).max()
    assert np.all(np.isinf(r["sinr"]))


@pytest.mark.parametrize("nr,nl", [(4, 2), (8, 4), (16, 8)])
def test_p5_zero_forcing_tall_lstsq(nr, nl):
    H = c64(cn((nr, nl)))
    y = c64(cn((3, nr)))
    r = _detect1(H, y, 0.0, 4)
    ref = np.linalg.lstsq(H.astype(np.complex128), y.astype(np.complex128).T, rcond=None)[0].T
    cond = np.linalg.cond(H.astype(np.complex128))
    assert np.abs(r["xhat"] - ref).max() <= 1e-12 * cond * max(1, np.abs(ref).max())


# ------------------------------------------------------------- P6 SINR ------
@pytest.mark.parametrize("nr,nl", [(2, 2), (4, 4), (8, 4), (16, 8)])
def test_p6_sinr_textbook(nr, nl):
    H = c64(cn((nr, nl)))
    s2 = 0.05
    r = _detect1(H, c64(cn((1, nr))), s2, 2)
    Hd = H.astype(np.complex128)
    for k in range(nl):
        hk = Hd[:, k]
        Hm = np.delete(Hd, k, axis=1)
        ref = (hk.conj() @ np.linalg.solve(Hm @ Hm.conj().T + np.float32(s2) * np.eye(nr), hk)).real
        assert abs(r["sinr"][k] - ref) <= 1e-11 * ref


def test_p6_sinr_orthogonal_and_mrc():
    s2 = np.float32(0.2)
    Q = np.linalg.qr(cn((4, 4)))[0]
    g = np.array([0.5, 1.0, 2.0, 3.0])
    H = c64(Q * g)
    r = _detect1(H, c64(cn((1, 4))), s2, 2)
    nrm = np.sum(np.abs(H.astype(np.complex128)) ** 2, axis=0)
    # columns are orthogonal only up to complex64 rounding of H
    assert np.allclose(r["sinr"], nrm / np.float64(s2), rtol=1e-6)
    h = c64(cn((8, 1)))
    r = _detect1(h, c64(cn((1, 8))), s2, 2)
    assert abs(r["sinr"][0] - np.sum(np.abs(h.astype(np.complex128)) ** 2) / np.float64(s2)) <= 1e-12 * r["sinr"][0]


# ---------------------------------------------------- P7 unbiasing ----------
def test_p7_mu_is_diag_WH():
    H = cn((8, 4))
    s2 = 0.1
    W = oracle.weights_chol(H, s2)
    mu_ref = np.real(np.diag(W @ H))
    r = _detect1(c64(H), c64(cn((1, 8))), s2, 2)
    mu = r["sinr"] / (1 + r["sinr"])
    H64 = c64(H).astype(np.complex128)
    mu_ref = np.real(np.diag(oracle.weights_chol(H64, np.float32(s2)) @ H64))
    assert np.abs(mu - mu_ref).max() <= 1e-12


@pytest.mark.parametrize("qm", [2, 4, 6, 8])
@pytest.mark.parametrize("kind", ["identity", "unitary", "orthogonal"])
@pytest.mark.parametrize("s2", [0.0, 0.03, 0.5])
def test_p7_noiseless_exact_recovery(qm, kind, s2):
    """Noiseless y = Hx, H = I / unitary / U diag(g): x~ = x and all hard bits exact, any sigma^2."""
    rng = np.random.default_rng(qm * 10 + len(kind))
    n = 4
    if kind == "identity":
        H = np.eye(n)
    elif kind == "unitary":
        H = np.linalg.qr(cn((n, n), rng))[0]
    else:
        H = np.linalg.qr(cn((8, n), rng))[0] * np.array([0.7, 1.0, 1.5, 2.5])
    H = c64(H)
    bits = rng.integers(0, 2, size=(50, n, qm)).astype(np.uint8)
    x = synth.qam_modulate(bits, qm)
    y = c64((H.astype(np.complex128) @ x.T).T)
    r = _detect1(H, y, s2, qm)
    tol = 1e-15 if kind == "identity" else 2e-6
    assert np.abs(r["xhat"] - x).max() <= tol + 1e-7  # complex64 rounding of y
    hard = (r["llr"] < 0).astype(np.uint8)
    assert np.array_equal(hard, bits)


# ------------------------------------------------------ P8 exhaustive ML ----
def _ml_llr(H, y, s2, qm):
    """Exhaustive max-log ML over all M^nl transmit vectors (brute force, numpy)."""
    nl = H.shape[1]
    labels = np.array(list(itertools.product(range(1 << qm), repeat=nl)))   # [V][nl]
    lb = ((labels[..., None] >> (qm - 1 - np.arange(qm))) & 1).astype(np.uint8)  # [V][nl][qm]
    X = synth.qam_modulate(lb, qm)                                           # [V][nl]
    d = np.sum(np.abs(y[None, :] - X @ H.T) ** 2, axis=1)                    # [V]
    out = np.zeros((nl, qm))
    for k in range(nl):
        for j in range(qm):
            out[k, j] = (d[lb[:, k, j] == 1].min() - d[lb[:, k, j] == 0].min()) / s2
    return out


@pytest.mark.parametrize("qm", [2, 4])
def test_p8_ml_equals_mmse_orthogonal(qm):
    rng = np.random.default_rng(11 + qm)
    s2 = np.float32(0.3)
    H = np.linalg.qr(cn((2, 2), rng))[0] * np.array([0.8, 1.6])
    H = c64(H).astype(np.complex128)
    # re-orthogonalise after complex64 rounding is impossible; use exactly orthogonal
    # real-rotation columns that survive rounding: [[a, -b], [b, a]] * diag(g)
    a, b = np.float32(0.6), np.float32(0.8)
    H = c64(np.array([[a, -b], [b, a]]) * np.array([0.5, 2.0])).astype(np.complex128)
    for _ in range(20):
        y = c64(cn(2, rng) * 1.5)
        r = _detect1(H, y[None], s2, qm)
        ml = _ml_llr(H, y.astype(np.complex128), np.float64(s2), qm)
        assert np.abs(r["llr"][0] - ml).max() <= 1e-9 * max(1, np.abs(ml).max())


@pytest.mark.parametrize("qm", [2, 4, 6])
def test_p8_ml_equals_mmse_single_layer(qm):
    rng = np.random.default_rng(5 + qm)
    s2 = np.float32(0.1)
    h = c64(cn((3, 1), rng)).astype(np.complex128)
    for _ in range(20):
        y = c64(cn(3, rng))
        r = _detect1(h, y[None], s2, qm)
        ml = _ml_llr(h, y.astype(np.complex128), np.float64(s2), qm)
        assert np.abs(r["llr"][0] - ml).max() <= 1e-9 * max(1, np.abs(ml).max())


def test_p8_noiseless_general_zf_bits():
    """General (non-orthogonal) H, sigma^2 = 0, noiseless: hard bits = ML = transmitted."""
    rng = np.random.default_rng(3)
    for qm in (2, 4):
        H = c64(cn((2, 2), rng))
        bits = rng.integers(0, 2, size=(30, 2, qm)).astype(np.uint8)
        x = synth.qam_modulate(bits, qm)
        y = c64((H.astype(np.complex128) @ x.T).T)
        r = _detect1(H, y, 0.0, qm)
        assert np.array_equal((r["llr"] < 0).astype(np.uint8), bits)


def test_p8_ml_ber_not_worse_than_mmse():
    """Statistics only for general H: ML hard-decision BER <= MMSE BER (2x2 QPSK)."""
    rng = np.random.default_rng(9)
    s2 = np.float32(0.3)
    err_ml = err_mmse = 0
    for _ in range(300):
        H = c64(cn((2, 2), rng))
        bits = rng.integers(0, 2, size=(2, 2)).astype(np.uint8)
        x = synth.qam_modulate(bits, 2)
        y = c64(H.astype(np.complex128) @ x + cn(2, rng) * np.sqrt(s2))
        ml = _ml_llr(H.astype(np.complex128), y.astype(np.complex128), np.float64(s2), 2)
        r = _detect1(H, y[None], s2, 2)
        err_ml += np.sum((ml < 0) != bits)
        err_mmse += np.sum((r["llr"][0] < 0) != bits)
    assert err_ml <= err_mmse


# --------------------------------------------------------- P9 demapper ------
def test_p9_qpsk_closed_form():
    x = cn(200)
    s = np.abs(RNG.standard_normal(200)) * 10
    llr = oracle.maxlog(2, x, s)
    assert np.allclose(llr[:, 0], 2 * np.sqrt(2) * s * x.real, rtol=1e-12, atol=1e-12)
    assert np.allclose(llr[:, 1], 2 * np.sqrt(2) * s * x.imag, rtol=1e-12, atol=1e-12)


@pytest.mark.parametrize("qm", [2, 4, 6, 8])
def test_p9_constellation_and_labels(qm):
    pts = oracle.constellation(qm)
    assert abs(np.mean(np.abs(pts) ** 2) - 1) <= 1e-12
    # independent implementation (synth's transmitter) agrees label by label
    lab = np.arange(1 << qm)
    lb = ((lab[:, None] >> (qm - 1 - np.arange(qm))) & 1).astype(np.uint8)
    assert np.allclose(pts, synth.qam_modulate(lb, qm), atol=1e-15)
    # Gray: horizontally/vertically adjacent points differ in exactly one bit
    a = np.sqrt({2: 2, 4: 10, 6: 42, 8: 170}[qm])
    for i in range(len(pts)):
        for j in range(len(pts)):
            if abs(abs(pts[i] - pts[j]) * a - 2) < 1e-9:
                assert bin(i ^ j).count("1") == 1
    # a point decodes to its own label
    llr = oracle.maxlog(qm, pts, 1.0)
    assert np.array_equal((llr < 0).astype(np.uint8), lb)


@pytest.mark.parametrize("qm", [4, 6, 8])
def test_p9_separable_and_symmetric(qm):
    x = cn(300) * 1.3
    llr = oracle.maxlog(qm, x, 3.0)
    # per-axis 1-D brute force
    m = qm // 2
    a = np.sqrt({4: 10, 6: 42, 8: 170}[qm])
    pts = oracle.constellation(qm)
    for off, comp in ((0, x.real), (1, x.imag)):
        levels = (pts.real if off == 0 else pts.imag)
        for i in range(m):
            j = 2 * i + off
            lab = np.arange(1 << qm)
            b = (lab >> (qm - 1 - j)) & 1
            d = (comp[:, None] - levels[None, :]) ** 2
            ref = 3.0 * (np.where(b[None] == 1, d, np.inf).min(1) - np.where(b[None] == 0, d, np.inf).min(1))
            assert np.allclose(llr[:, j], ref, rtol=1e-12, atol=1e-12)
    # negating Re(x) flips only b_0's LLR sign
    llr2 = oracle.maxlog(qm, -x.conj(), 3.0)
    assert np.allclose(llr2[:, 0], -llr[:, 0], atol=1e-12)
    assert np.allclose(llr2[:, 2::2], llr[:, 2::2], atol=1e-12)
    assert np.allclose(llr2[:, 1::2], llr[:, 1::2], atol=1e-12)
    del a


def closed_form_llr(x, slope_nat, qm):
    """The per-axis closed form the CUDA demapper uses, in numpy fp64.

    u = axis / a; s_q = clamp(2 floor(u/2) + 1, +-(2^m - 1)); D = (u - s_q)^2;
    t_0 = u, t_i = 2^(m-i) - |t_{i-1}|; LLR_i = sgn(t_i) * SINR a^2 * ((|t_i| + 1)^2 - D).
    """
    m = qm // 2
    a = 1 / np.sqrt({2: 2, 4: 10, 6: 42, 8: 170}[qm])
    out = np.zeros(x.shape + (qm,))
    for off, comp in ((0, x.real), (1, x.imag)):
        u = comp / a
        lim = (1 << m) - 1
        sq = np.clip(2 * np.floor(u / 2) + 1, -lim, lim)
        D = (u - sq) ** 2
        ts = [u]
        for i in range(1, m):
            ts.append((1 << (m - i)) - np.abs(ts[-1]))
        # the kernel takes D from the last fold: (|t_{m-1}| - 1)^2 == (u - s_q)^2
        assert np.allclose((np.abs(ts[-1]) - 1) ** 2, D, rtol=1e-12, atol=1e-12)
        for i, t in enumerate(ts):
            out[..., 2 * i + off] = np.sign(t) * slope_nat * a * a * ((np.abs(t) + 1) ** 2 - D)
    return out


@pytest.mark.parametrize("qm", [2, 4, 6, 8])
def test_p10_closed_form_equals_bruteforce(qm):
    """The GPU's O(bits) closed form equals brute-force max-log, incl. boundaries and out of range."""
    a = 1 / np.sqrt({2: 2, 4: 10, 6: 42, 8: 170}[qm])
    m = qm // 2
    lim = (1 << m)
    grid = np.arange(-lim - 3, lim + 3.01, 0.25) * a       # boundaries at integers and beyond
    X = (grid[:, None] + 1j * grid[None, :]).ravel()
    X = np.concatenate([X, cn(2000) * 1.5, cn(200) * 10])
    s = 7.5
    bf = oracle.maxlog(qm, X, s)
    cf = closed_form_llr(X, s, qm)
    assert np.abs(bf - cf).max() <= 1e-9 * max(1, np.abs(bf).max())


# ------------------------------------------------ P11 scale invariance ------
def test_p11_scale_invariance():
    w = synth.generate(2, n_sc=24, n_slots=1)
    Hu, Yu = w.H_units(), w.y_units()
    r1 = oracle.detect(Hu, Yu, w.sigma2, w.qm)
    r2 = oracle.detect(2 * Hu, 2 * Yu, 4 * w.sigma2, w.qm)
    assert np.array_equal(r1["llr"], r2["llr"])
    assert np.array_equal(r1["xhat"], r2["xhat"])


# -------------------------------------------- route equivalence (whole) -----
@pytest.mark.parametrize("k", [1, 2, 3, 4])
def test_detector_routes_agree(k):
    """Gram/Cholesky detector == paper-literal covariance/LU detector (push-through + P7)."""
    w = synth.generate(k, n_sc=24 if k != 1 else 12, n_slots=1)
    Hu, Yu = w.H_units(), w.y_units()
    a = oracle.detect(Hu, Yu, w.sigma2, w.qm)
    b = oracle.detect(Hu, Yu, w.sigma2, w.qm, route="lu")
    assert np.abs(a["xhat"] - b["xhat"]).max() <= 1e-9
    assert np.abs(a["sinr"] - b["sinr"]).max() <= 1e-9 * a["sinr"].max()
    assert np.abs(a["llr"] - b["llr"]).max() <= 1e-8 * max(1, np.abs(a["llr"]).max())


def test_zero_column_erasure():
    """A zero column at sigma^2 > 0 gives mu = 0: the layer is erased (x~ 0, SINR 0, LLR 0)."""
    H = c64(cn((4, 3)))
    H[:, 1] = 0
    r = _detect1(H, c64(cn((5, 4))), 0.1, 4)
    assert r["ok"]
    assert np.all(r["xhat"][:, 1] == 0) and r["sinr"][1] == 0 and np.all(r["llr"][:, 1] == 0)
    r = _detect1(H, c64(cn((5, 4))), 0.0, 4)
    assert not r["ok"] and np.all(r["llr"] == 0)


# ------------------------------------------------------- P13 quantisers -----
def test_p13_quantisers():
    v = np.concatenate([RNG.standard_normal(5000) * 300, [0.5, 1.5, 2.5, -0.5, -2.5, 126.5, 127.4,
                                                         -127.6, 1e9, -1e9, 65519.0, 65520.0, 1e40]])
    q8 = oracle.quantize(v, "i8")
    assert np.array_equal(q8, np.clip(np.rint(v), -127, 127).astype(np.int8))
    q16 = oracle.quantize(v, "f16")
    assert np.array_equal(q16, np.clip(v, -65504, 65504).astype(np.float16))
    q32 = oracle.quantize(v, "f32")
    assert np.array_equal(q32, np.clip(v, -np.finfo(np.float32).max, np.finfo(np.float32).max).astype(np.float32))
    assert oracle.quantize(np.array([np.inf, -np.inf]), "f32").tolist() == [np.finfo(np.float32).max,
                                                                             -np.finfo(np.float32).max]
    assert oracle.quantize(np.array([np.inf, -np.inf]), "i8").tolist() == [127, -127]
    assert np.array_equal(oracle.quantize(v, "i8", 0.5), np.clip(np.rint(v * 0.5), -127, 127).astype(np.int8))


# ------------------------------------------------- golden hand-worked -------
def test_golden_handworked():
    with open(os.path.join(GOLDEN, "handworked.json")) as f:
        cases = json.load(f)["cases"]
    assert len(cases) >= 3
    for c in cases:
        H = np.array(c["H_re"]) + 1j * np.array(c["H_im"])
        y = np.array(c["y_re"]) + 1j * np.array(c["y_im"])
        r = _detect1(H, y[None], c["sigma2"], c["qm"])
        xr = np.array(c["xhat_re"]) + 1j * np.array(c["xhat_im"])
        assert np.allclose(r["xhat"][0], xr, atol=1e-12), c["name"]
        assert np.allclose(r["sinr"], c["sinr"], rtol=1e-12), c["name"]
        assert np.allclose(r["llr"][0], np.array(c["llr"]), rtol=1e-12, atol=1e-12), c["name"]


@pytest.mark.parametrize("qm", [2, 4])
def test_p10_linear_forms_equal_bruteforce(qm):
    """QPSK / 16-QAM linear-region forms used by the CUDA demapper (sigma2 > 0 path) = brute force."""
    a = 1 / np.sqrt({2: 2, 4: 10}[qm])
    grid = np.arange(-7, 7.01, 0.125) * a
    X = np.concatenate([(grid[:, None] + 1j * grid[None, :]).ravel(), cn(3000) * 2.0])
    s = 3.25
    bf = oracle.maxlog(qm, X, s)
    out = np.zeros(X.shape + (qm,))
    sa = s * a * a
    for off, comp in ((0, X.real), (1, X.imag)):
        u = comp / a
        if qm == 2:
            out[:, off] = 4 * sa * u
        else:
            out[:, off] = 4 * sa * (u + np.sign(u) * np.maximum(np.abs(u) - 2, 0))
            out[:, 2 + off] = 4 * sa * (2 - np.abs(u))
    assert np.abs(bf - out).max() <= 1e-9 * max(1, np.abs(bf).max())
