"""Parity harness: run the CUDA path and the fp64 oracle on the same seeded
inputs and compare with the north_star tolerances (SURVEY.md §8(c) "Tolerances"):

  x~   : |d| <= 1e-4 * max(|x~_ref|, 1) per complex element
  SINR : relative <= 1e-4 (absolute 1e-7 where SINR_ref < 1e-3: erased layers)
  LLR  : float types |d| <= 1e-3 * max(|L_ref|, 1) after quantising the oracle's
         fp64 LLR the same way (fp16: RNE + saturation; fp32: saturation);
         int8: equal to sat(rint(L_ref * scale)) except +-1 where L_ref * scale
         lies within 1e-3 * max(|v|, 1) of a half-integer;
  bits : hard decisions (LLR < 0) identical wherever |L_ref| >= 1e-3.
"""
from __future__ import annotations

import numpy as np

import oracle
from paper_2510_07843_b200 import synth

TOL_X = 1e-4
TOL_SINR = 1e-4
TOL_LLR = 1e-3


def np_llr_dtype(llr: str):
    return {"f32": np.float32, "f16": np.float16, "i8": np.int8}[llr]


def run_gpu(w: synth.Workload, *, xhat=True, sinr=True, llr_scale=1.0, plan=None, H=None, y=None, kernel=None):
    """Detect the whole workload on cuda:0 through the C ABI; returns numpy arrays.
    kernel: a named kernel specialisation (mimo_plan_desc_t.kernel), default the shape's default."""
    import torch
    from paper_2510_07843_b200 import mimo
    own = plan is None
    if own:
        plan = mimo.Plan(w.n_rx, w.n_layers, w.qm, sc_per_h=w.sc_per_h, sym_per_h=w.sym_per_h, llr_dtype=w.llr,
                         llr_scale=llr_scale, kernel=kernel)
    Hd = torch.from_numpy(w.H if H is None else H).cuda()
    yd = torch.from_numpy(w.y if y is None else y).cuda()
    sh = plan.shapes(w.n_sc, w.n_sym)
    xd = torch.empty(sh["xhat"], dtype=torch.complex64, device="cuda") if xhat else None
    sd = torch.empty(sh["sinr"], dtype=torch.float32, device="cuda") if sinr else None
    out = plan.detect(Hd, yd, float(w.sigma2), xhat=xd, sinr=sd)
    n_failed = plan.sync_status()
    res = dict(llr=out.cpu().numpy(), n_failed=n_failed, kernel=plan.kernel_name)
    if xhat:
        res["xhat"] = xd.cpu().numpy()
    if sinr:
        res["sinr"] = sd.cpu().numpy()
    if own:
        plan.close()
    return res


def oracle_units(w: synth.Workload, units, threads=None, H=None, y=None, route="chol"):
    units = np.asarray(units, dtype=np.int64)
    Hu = (w.H if H is None else H).reshape(w.n_units, w.n_rx, w.n_layers)[units]
    yy = w.y if y is None else y
    Yu = np.stack([yy[synth.unit_re_index(u, w.n_sc, w.sc_per_h, w.sym_per_h)] for u in units]) if len(units) else \
        np.zeros((0, w.sym_per_h * w.sc_per_h, w.n_rx), np.complex64)
    return oracle.detect(Hu, Yu, w.sigma2, w.qm, threads=threads or oracle.max_threads(), route=route)


def gather_units(w: synth.Workload, grid: np.ndarray, units):
    return np.stack([grid[synth.unit_re_index(u, w.n_sc, w.sc_per_h, w.sym_per_h)] for u in units])


def compare(w: synth.Workload, gpu: dict, units=None, llr_scale=1.0, threads=None, H=None, y=None,
            route="chol", tol_x=TOL_X, tol_sinr=TOL_SINR, tol_llr=TOL_LLR) -> dict:
    """Compare GPU outputs against the oracle on the given units (default: all).
    route="lu" compares with the oracle's paper-literal covariance/LU route."""
    if units is None:
        units = np.arange(w.n_units)
    units = np.asarray(units, dtype=np.int64)
    ref = oracle_units(w, units, threads=threads, H=H, y=y, route=route)
    rep = dict(units=len(units), n_failed_ref=int((~ref["ok"]).sum()))
    # x~
    if "xhat" in gpu:
        gx = gather_units(w, gpu["xhat"], units)
        rx = ref["xhat"]
        err = np.abs(gx - rx) / np.maximum(np.abs(rx), 1.0)
        rep["xhat_max_err"] = float(err.max()) if err.size else 0.0
        assert rep["xhat_max_err"] <= tol_x, rep
    # SINR
    if "sinr" in gpu:
        gs = gpu["sinr"][units].astype(np.float64)
        rs = ref["sinr"]
        fin = np.isfinite(rs)
        assert np.array_equal(np.isinf(gs), ~fin), "SINR infinities differ"
        # relative 1e-4; below SINR 1e-3 (erased / near-erased layers) absolute 1e-7
        rel = np.abs(gs[fin] - rs[fin]) / np.maximum(np.abs(rs[fin]), 1e-3)
        rep["sinr_max_rel"] = float(rel.max()) if rel.size else 0.0
        assert rep["sinr_max_rel"] <= tol_sinr, rep
    # LLRs
    gl = gather_units(w, gpu["llr"], units)
    rl = ref["llr"] * llr_scale
    rep.update(compare_llr(gl, rl, w.llr, tol_llr))
    return rep


def compare_llr(gl: np.ndarray, rl: np.ndarray, llr: str, tol_llr: float = TOL_LLR) -> dict:
    """gl: GPU LLRs (quantised); rl: oracle fp64 LLRs already multiplied by llr_scale."""
    rep = {}
    if llr == "i8":
        q = oracle.quantize(rl, "i8").astype(np.int64)
        g = gl.astype(np.int64)
        d = np.abs(g - q)
        v = np.clip(rl, -127.0, 127.0)
        near_half = np.abs(np.abs(v - np.floor(v)) - 0.5) <= tol_llr * np.maximum(np.abs(v), 1.0)
        bad = (d > 1) | ((d == 1) & ~near_half)
        rep["llr_mismatch"] = int((d > 0).sum())
        rep["llr_bad"] = int(bad.sum())
        assert rep["llr_bad"] == 0, rep
        hard_ok = ((g < 0) == (q < 0)) | (np.abs(rl) < 1.0)
    else:
        qref = oracle.quantize(rl, llr).astype(np.float64)
        g = gl.astype(np.float64)
        assert np.all(np.isfinite(g)), "non-finite GPU LLR"
        err = np.abs(g - qref) / np.maximum(np.abs(qref), 1.0)
        rep["llr_max_err"] = float(err.max()) if err.size else 0.0
        assert rep["llr_max_err"] <= tol_llr, rep
        hard_ok = ((g < 0) == (qref < 0)) | (np.abs(rl) < tol_llr)
    rep["hard_bit_mismatch"] = int((~hard_ok).sum())
    assert rep["hard_bit_mismatch"] == 0, rep
    rep["n_llr"] = int(gl.size)
    return rep
