"""GPU parity of detection from BFP-compressed y (mimo_detect_mmse_bfp, SURVEY.md
§8(f) NEXT-4, reading R25) against the oracle run on the oracle's own decode of
the same bytes, at the north_star tolerances."""
import numpy as np
import pytest
import torch

import oracle
import parity
from paper_2510_07843_b200 import mimo, synth

pytestmark = pytest.mark.gpu
SCALE = 2.0 ** -8


def run_bfp(w, W, *, xhat=True):
    p = mimo.Plan(w.n_rx, w.n_layers, w.qm, sc_per_h=w.sc_per_h, llr_dtype=w.llr)
    yb = torch.from_numpy(synth.bfp_compress(w.y, W, SCALE)).cuda()
    sh = p.shapes(w.n_sc, w.n_sym)
    x = torch.empty(sh["xhat"], dtype=torch.complex64, device="cuda") if xhat else None
    s = torch.empty(sh["sinr"], dtype=torch.float32, device="cuda")
    out = p.detect_bfp(torch.from_numpy(w.H).cuda(), yb, float(w.sigma2), n_sym=w.n_sym, n_sc=w.n_sc,
                       iq_width=W, bfp_scale=SCALE, xhat=x, sinr=s)
    nf = p.sync_status()
    p.close()
    r = dict(llr=out.cpu().numpy(), sinr=s.cpu().numpy(), n_failed=nf)
    if xhat:
        r["xhat"] = x.cpu().numpy()
    return r


def decoded_y(w, W):
    d = oracle.bfp_decode(synth.bfp_compress(w.y, W, SCALE), W, SCALE)  # [sym][prb][r][f]
    return np.ascontiguousarray(d.transpose(0, 1, 3, 2).reshape(w.y.shape))


@pytest.mark.parametrize("W", [8, 9, 12, 16])
def test_bfp_matches_oracle_on_decoded_y(W):
    w = synth.generate(3, n_sc=300, n_slots=2)
    g = run_bfp(w, W)
    assert g["n_failed"] == 0
    print(W, parity.compare(w, g, y=decoded_y(w, W)))


def test_bfp_full_size_sampled():
    w = synth.generate(3)
    g = run_bfp(w, 9, xhat=False)
    rng = np.random.default_rng(7)
    units = np.unique(np.concatenate([[0, w.n_units - 1], rng.choice(w.n_units, 200, replace=False)]))
    print(parity.compare(w, g, units, y=decoded_y(w, 9)))


@pytest.mark.parametrize("k,kw", [(2, dict(n_sc=96, n_slots=2)), (4, dict(n_sc=48, n_slots=1)),
                                  (5, dict(n_sc=48, n_slots=1)), (1, {})])
def test_bfp_other_shapes_equal_detect_on_decoded_y(k, kw):
    """Shapes without the fused decode: k_bfp_decode expands the blocks, then the shape's detector
    runs. The LLRs are BIT-identical to the detector on the oracle's decode of the same bytes (which
    pins the decode kernel bit-exactly), and within the north_star tolerances of the oracle."""
    w = synth.generate(k, **kw)
    if w.n_sc % 12:
        pytest.skip("BFP blocks are per PRB")
    g = run_bfp(w, 9)
    yd = decoded_y(w, 9)
    ref = parity.run_gpu(w, y=yd)
    assert g["n_failed"] == 0
    assert np.array_equal(g["llr"], ref["llr"])
    assert np.array_equal(g["xhat"], ref["xhat"])
    parity.compare(w, g, y=yd)


def test_bfp_ragged_n_sc_rejected():
    p = mimo.Plan(4, 4, 4)
    w = synth.generate(2, n_sc=24, n_slots=1)
    yb = torch.zeros((w.n_sym, 1, 4, 28), dtype=torch.uint8, device="cuda")
    with pytest.raises(mimo.MimoError) as e:
        p.detect_bfp(torch.from_numpy(np.ascontiguousarray(w.H[:, :20])).cuda(), yb, float(w.sigma2), n_sym=w.n_sym,
                     n_sc=20)
    assert e.value.status == mimo.MIMO_ERR_INVALID_ARG


def test_bfp_host_path_other_shape_bit_identical():
    """The host path with per-chunk expansion (C5 shape) equals the device BFP call bit for bit."""
    w = synth.generate(5, n_sc=48, n_slots=3)
    ref = run_bfp(w, 9, xhat=False)["llr"]
    p = mimo.Plan(w.n_rx, w.n_layers, w.qm, sc_per_h=w.sc_per_h, llr_dtype=w.llr, host_chunk_bytes=200_000)
    yb = torch.from_numpy(synth.bfp_compress(w.y, 9, SCALE)).pin_memory()
    out = torch.empty(ref.shape, dtype=torch.int8).pin_memory()
    p.detect_bfp_host(torch.from_numpy(w.H).pin_memory(), yb, float(w.sigma2), n_sym=w.n_sym, n_sc=w.n_sc,
                      iq_width=9, bfp_scale=SCALE, out=out, wait=True)
    assert p.sync_status() == 0
    assert np.array_equal(out.numpy(), ref)


@pytest.mark.parametrize("wait", [True, False])
def test_bfp_host_path_bit_identical_to_device_path(wait):
    """mimo_detect_mmse_bfp_host[_async]: the compressed y crosses the host link; results are
    bit-identical to the device-buffer BFP call (same kernels, slot chunks are independent)."""
    w = synth.generate(3, n_sc=300, n_slots=6)
    ref = run_bfp(w, 9, xhat=False)["llr"]
    p = mimo.Plan(w.n_rx, w.n_layers, w.qm, sc_per_h=w.sc_per_h, llr_dtype=w.llr, host_chunk_bytes=100_000)
    yb = torch.from_numpy(synth.bfp_compress(w.y, 9, SCALE)).pin_memory()
    out = torch.empty(ref.shape, dtype=torch.int8).pin_memory()
    p.detect_bfp_host(torch.from_numpy(w.H).pin_memory(), yb, float(w.sigma2), n_sym=w.n_sym, n_sc=w.n_sc,
                      iq_width=9, bfp_scale=SCALE, out=out, wait=wait)
    assert p.sync_status() == 0
    assert np.array_equal(out.numpy(), ref)
