"""GPU parity of the paper-literal route (mimo_detect_lmmse_lu, SURVEY.md §8(f)
NEXT-1): covariance R = HH^H + s2 I, pivoted LU, inversion by forward/backward
substitution, W = H^H R^-1, as five stage kernels.

The fp64 ("PD") route is held to the north_star tolerances against the
oracle's own covariance/LU route (oracle route="lu", written from the same
passages). The fp32 ("PS") route is held to the tolerance DESIGN.md reading R22
derives from the LU forward-error bound (it scales with cond(R), which the
Gram form avoids: that is why the production path uses the Gram matrix)."""
import numpy as np
import pytest
import torch

import oracle
import parity
from paper_2510_07843_b200 import mimo, synth

pytestmark = pytest.mark.gpu

U32 = 2.0 ** -24


def run_lu(w, precision, *, timing=False, plan=None):
    own = plan is None
    if own:
        plan = mimo.Plan(w.n_rx, w.n_layers, w.qm, sc_per_h=w.sc_per_h, llr_dtype=w.llr)
    H = torch.from_numpy(w.H).cuda()
    y = torch.from_numpy(w.y).cuda()
    sh = plan.shapes(w.n_sc, w.n_sym)
    x = torch.empty(sh["xhat"], dtype=torch.complex64, device="cuda")
    s = torch.empty(sh["sinr"], dtype=torch.float32, device="cuda")
    r = plan.detect_lu(H, y, float(w.sigma2), precision=precision, xhat=x, sinr=s, timing=timing)
    out, st = (r if timing else (r, None))
    n_failed = plan.sync_status()
    res = dict(llr=out.cpu().numpy(), xhat=x.cpu().numpy(), sinr=s.cpu().numpy(), n_failed=n_failed,
               stages=st)
    if own:
        plan.close()
    return res


LU_CASES = {
    "C1": (1, dict()),
    "C2": (2, dict(n_sc=300, n_slots=2)),
    "C3": (3, dict(n_sc=300, n_slots=2)),
    "C4": (4, dict(n_sc=96, n_slots=1)),
    "P": ("P", dict(n_sc=720, n_slots=1)),
}


@pytest.mark.parametrize("name", list(LU_CASES))
def test_pd_route_matches_oracle_lu_route(name):
    k, kw = LU_CASES[name]
    w = synth.generate(k, **kw)
    g = run_lu(w, 64)
    assert g["n_failed"] == 0
    rep = parity.compare(w, g, route="lu")
    print(name, rep)


def cond_R(w):
    H = w.H.reshape(w.n_units, w.n_rx, w.n_layers).astype(np.complex128)
    R = H @ np.conj(np.swapaxes(H, 1, 2)) + float(w.sigma2) * np.eye(w.n_rx)
    return np.linalg.cond(R)


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "P"])
def test_ps_route_within_lu_error_bound(name):
    """fp32 LU route: per-unit x~ error <= c * n_rx * cond(R) * u32 * max(|x~|, 1) (reading R22)."""
    k, kw = LU_CASES[name]
    w = synth.generate(k, **kw)
    g = run_lu(w, 32)
    assert g["n_failed"] == 0
    ref = parity.oracle_units(w, np.arange(w.n_units), route="lu")
    gx = parity.gather_units(w, g["xhat"], np.arange(w.n_units))
    err = np.abs(gx - ref["xhat"]) / np.maximum(np.abs(ref["xhat"]), 1.0)
    bound = 4.0 * w.n_rx * cond_R(w) * U32
    ratio = err.max(axis=(1, 2)) / bound
    print(name, "max err", err.max(), "max err / bound", ratio.max())
    assert ratio.max() <= 1.0


def test_routes_agree_pd_vs_cholesky():
    """Push-through identity (pin P3) on the GPU: the LU route and the fused Gram/Cholesky kernel."""
    w = synth.generate(2, n_sc=300, n_slots=2)
    a = run_lu(w, 64)
    b = parity.run_gpu(w)
    err = np.abs(a["xhat"] - b["xhat"]) / np.maximum(np.abs(b["xhat"]), 1.0)
    assert err.max() <= 2e-4
    assert np.array_equal(a["llr"] < 0, b["llr"] < 0) or \
        ((a["llr"] < 0) != (b["llr"] < 0)).sum() <= 2  # ties at |LLR| ~ 0 only


def test_stage_timing_reported():
    w = synth.generate("P", n_sc=720, n_slots=1)
    g = run_lu(w, 32, timing=True)
    st = g["stages"]
    assert list(st) == list(mimo.LU_STAGES)
    assert all(v > 0 for v in st.values()), st
    print(st)


def test_singular_covariance_flagged_at_zero_noise():
    """sigma2 = 0 with n_rx > n_layers: R = HH^H has rank n_layers, every unit fails the LU guard."""
    cfg = dict(synth.CONFIGS[3], n_sc=24, n_slots=1)
    w = synth.generate(cfg)
    w.sigma2 = np.float32(0.0)
    g = run_lu(w, 64)
    assert g["n_failed"] == w.n_units
    assert np.all(g["llr"] == 0) and np.all(g["xhat"] == 0) and np.all(g["sinr"] == 0)
    ref = parity.oracle_units(w, np.arange(w.n_units), route="lu")
    assert not ref["ok"].any()


def test_square_zero_noise_is_zero_forcing():
    w = synth.generate(2, n_sc=60, n_slots=1)
    w.sigma2 = np.float32(0.0)
    g = run_lu(w, 64)
    assert g["n_failed"] == 0
    assert np.all(np.isinf(g["sinr"]))
    rep = parity.compare(w, dict(xhat=g["xhat"], llr=g["llr"]), route="lu")
    print(rep)


def test_unsupported_and_invalid():
    p = mimo.Plan(64, 16, 6, sc_per_h=12, llr_dtype="i8")
    w = synth.generate(5, n_sc=12, n_slots=1)
    with pytest.raises(mimo.MimoError) as e:
        p.detect_lu(torch.from_numpy(w.H).cuda(), torch.from_numpy(w.y).cuda(), float(w.sigma2))
    assert e.value.status == mimo.MIMO_ERR_UNSUPPORTED
    p2 = mimo.Plan(4, 4, 4)
    w2 = synth.generate(2, n_sc=12, n_slots=1)
    with pytest.raises(mimo.MimoError) as e:
        p2.detect_lu(torch.from_numpy(w2.H).cuda(), torch.from_numpy(w2.y).cuda(), float(w2.sigma2), precision=16)
    assert e.value.status == mimo.MIMO_ERR_INVALID_ARG
