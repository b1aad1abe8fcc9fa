"""C-ABI error behaviour with a device present (include/mimo.h ERRORS)."""
import ctypes

import numpy as np
import pytest

from paper_2510_07843_b200 import mimo, synth

pytestmark = pytest.mark.gpu


@pytest.fixture()
def setup():
    import torch
    w = synth.generate(2, n_sc=32, n_slots=1)
    plan = mimo.Plan(4, 4, 4)
    H = torch.from_numpy(w.H).cuda()
    y = torch.from_numpy(w.y).cuda()
    out = torch.empty((14, 32, 4, 4), dtype=torch.float32, device="cuda")
    yield plan, H, y, out, w
    plan.close()


def _call(plan, H, y, out, sigma2=0.1, nr=4, nl=4, nsc=32, nsym=14, qm=4):
    p = lambda t: ctypes.c_void_p(t if isinstance(t, int) else t.data_ptr()) if t is not None else None
    return plan._lib.mimo_detect_mmse(plan._h, p(H), p(y), ctypes.c_float(sigma2), nr, nl, nsc, nsym, qm, p(out))


def test_ok(setup):
    plan, H, y, out, _ = setup
    assert _call(plan, H, y, out) == mimo.MIMO_OK
    assert plan.sync_status() == 0


@pytest.mark.parametrize("kw", [dict(nr=2), dict(nl=2), dict(qm=6), dict(nsc=-1), dict(nsym=13),
                                dict(sigma2=-0.1), dict(sigma2=float("nan")), dict(sigma2=float("inf"))])
def test_invalid_dims(setup, kw):
    plan, H, y, out, _ = setup
    assert _call(plan, H, y, out, **kw) == mimo.MIMO_ERR_INVALID_ARG
    assert plan._lib.mimo_plan_last_error(plan._h)


def test_null_and_misaligned(setup):
    plan, H, y, out, _ = setup
    assert _call(plan, None, y, out) == mimo.MIMO_ERR_INVALID_ARG
    assert _call(plan, H, y, None) == mimo.MIMO_ERR_INVALID_ARG
    assert _call(plan, H, y.data_ptr() + 8, out) == mimo.MIMO_ERR_INVALID_ARG


def test_host_pointer_rejected(setup):
    plan, H, y, out, w = setup
    host = np.zeros(w.y.size, np.complex64)
    assert _call(plan, H, host.ctypes.data, out) == mimo.MIMO_ERR_INVALID_ARG


def test_python_shape_checks(setup):
    import torch
    plan, H, y, out, _ = setup
    with pytest.raises(ValueError):
        plan.detect(H.cpu(), y, 0.1)
    with pytest.raises(ValueError):
        plan.detect(H, y.to(torch.complex128), 0.1)
    with pytest.raises(mimo.MimoError):
        plan.detect(H, y, -1.0)


def test_sync_status_counts_and_resets():
    import torch
    w = synth.generate(2, n_sc=32, n_slots=1, sigma2=0.0)
    H = w.H.copy()
    H[0, 1, :, 0] = 0
    plan = mimo.Plan(4, 4, 4)
    Hd, yd = torch.from_numpy(H).cuda(), torch.from_numpy(w.y).cuda()
    plan.detect(Hd, yd, 0.0)
    plan.detect(Hd, yd, 0.0)
    assert plan.sync_status() == 2
    assert plan.sync_status() == 0
    st = plan._lib.mimo_plan_sync_status(plan._h, None)
    assert st == mimo.MIMO_OK


def test_kernel_selection():
    assert mimo.Plan(4, 4, 4).kernel_name.startswith("tpu_4x4")
    assert mimo.Plan(2, 2, 2).kernel_name.startswith("tpu_2x2")
    assert mimo.Plan(7, 3, 4).kernel_name == "generic"
    assert mimo.Plan(4, 4, 4).launches_per_call == 1
    # the descriptor's kernel field: a named variant, "generic", an unknown name -> UNSUPPORTED
    assert mimo.Plan(64, 16, 6, sc_per_h=12, llr_dtype="i8").kernel_name.startswith("c5_fused")
    assert mimo.Plan(64, 16, 6, sc_per_h=12, llr_dtype="i8", kernel="big_64x16_q6_i8").kernel_name == "big_64x16_q6_i8"
    assert mimo.Plan(4, 4, 4, kernel="generic").kernel_name == "generic"
    with pytest.raises(mimo.MimoError) as ei:
        mimo.Plan(4, 4, 4, kernel="no_such_kernel")
    assert ei.value.status == mimo.MIMO_ERR_UNSUPPORTED
    with pytest.raises(mimo.MimoError):  # a name of another shape's kernel does not serve this one
        mimo.Plan(4, 4, 4, kernel="c5_fused_64x16_q6_i8")


def test_host_path_async_then_sync_of_other_layout():
    """a synchronous host-buffer call right after an asynchronous one of the same
    plan uses another chunk layout; both must return the device path's LLRs exactly."""
    import torch
    w = synth.generate(2)  # full C2: the async call's 16 MiB chunks vs the sync call's 4 MiB ones
    plan = mimo.Plan(4, 4, 4)
    H, y = torch.from_numpy(w.H), torch.from_numpy(w.y)
    ref = plan.detect(H.cuda(), y.cuda(), float(w.sigma2)).cpu()
    Hh, yh = H.pin_memory(), y.pin_memory()
    la = torch.empty_like(ref).pin_memory()
    lb = torch.empty_like(ref).pin_memory()
    w2 = synth.generate(2, n_slots=3, seed=77)  # another shape, then the full one again
    ref2 = plan.detect(torch.from_numpy(w2.H).cuda(), torch.from_numpy(w2.y).cuda(), float(w2.sigma2)).cpu()
    lc = torch.empty_like(ref2).pin_memory()
    plan.detect_host(Hh, yh, float(w.sigma2), out=la, wait=False)
    plan.detect_host(torch.from_numpy(w2.H).pin_memory(), torch.from_numpy(w2.y).pin_memory(), float(w2.sigma2),
                     out=lc, wait=True)
    plan.detect_host(Hh, yh, float(w.sigma2), out=lb, wait=True)
    assert plan.sync_status() == 0
    assert torch.equal(la, ref) and torch.equal(lb, ref) and torch.equal(lc, ref2)


def test_host_chunk_bytes_descriptor_field():
    import torch
    w = synth.generate(2, n_sc=96, n_slots=6)
    ref = mimo.Plan(4, 4, 4).detect(torch.from_numpy(w.H).cuda(), torch.from_numpy(w.y).cuda(), float(w.sigma2)).cpu()
    for cb in (1, 200_000, 1 << 30):
        p = mimo.Plan(4, 4, 4, host_chunk_bytes=cb)
        out = torch.empty_like(ref)
        p.detect_host(torch.from_numpy(w.H), torch.from_numpy(w.y), float(w.sigma2), out=out)
        assert torch.equal(out, ref)


def test_stream_ordering():
    """Work goes on torch's current stream: results are ready after that stream syncs."""
    import torch
    w = synth.generate(2, n_sc=64, n_slots=2)
    plan = mimo.Plan(4, 4, 4)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        H = torch.from_numpy(w.H).cuda()
        y = torch.from_numpy(w.y).cuda()
        out = plan.detect(H, y, float(w.sigma2))
    s.synchronize()
    ref = plan.detect(H, y, float(w.sigma2))
    torch.cuda.synchronize()
    assert torch.equal(out, ref)


def test_cuda_graph_capture():
    import torch
    w = synth.generate(2, n_sc=64, n_slots=2)
    plan = mimo.Plan(4, 4, 4)
    H = torch.from_numpy(w.H).cuda()
    y = torch.from_numpy(w.y).cuda()
    out = torch.empty((28, 64, 4, 4), device="cuda")
    ref = plan.detect(H, y, float(w.sigma2)).clone()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            plan.detect(H, y, float(w.sigma2), out=out)
    torch.cuda.current_stream().wait_stream(s)
    out.zero_()
    g.replay()
    torch.cuda.synchronize()
    assert torch.equal(out, ref)


def test_overlap_calls_same_output_buffer():
    """MIMO_PLAN_OVERLAP_CALLS: back-to-back calls (PDL) writing one output buffer stay ordered."""
    import torch
    ws = [synth.generate(2, n_sc=3276, n_slots=2, seed=s) for s in (1, 2, 3)]
    ref_plan = mimo.Plan(4, 4, 4)
    refs = [ref_plan.detect(torch.from_numpy(w.H).cuda(), torch.from_numpy(w.y).cuda(), float(w.sigma2)).clone()
            for w in ws]
    plan = mimo.Plan(4, 4, 4, overlap_calls=True)
    Hs = [torch.from_numpy(w.H).cuda() for w in ws]
    ys = [torch.from_numpy(w.y).cuda() for w in ws]
    out = torch.empty_like(refs[0])
    outs = [torch.empty_like(refs[0]) for _ in ws]
    torch.cuda.synchronize()
    for rep in range(20):
        for i, w in enumerate(ws):
            plan.detect(Hs[i], ys[i], float(w.sigma2), out=out)
            plan.detect(Hs[i], ys[i], float(w.sigma2), out=outs[i])
    torch.cuda.synchronize()
    assert torch.equal(out, refs[-1])
    for o, r in zip(outs, refs):
        assert torch.equal(o, r)


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_overlap_mode_parity(k):
    import parity
    w = synth.generate(k, n_sc=120 if k != 1 else 12, n_slots=2 if k != 1 else 1)
    plan = mimo.Plan(w.n_rx, w.n_layers, w.qm, sc_per_h=w.sc_per_h, llr_dtype=w.llr, overlap_calls=True)
    g = parity.run_gpu(w, plan=plan)
    parity.compare(w, g)


def _call_sv(plan, H, y, s2v, out, nr=4, nl=4, nsc=32, nsym=14, qm=4):
    p = lambda t: ctypes.c_void_p(t if isinstance(t, int) else t.data_ptr()) if t is not None else None
    return plan._lib.mimo_detect_mmse_sv(plan._h, p(H), p(y), p(s2v), nr, nl, nsc, nsym, qm, p(out), None, None)


def test_sigma2_array_errors(setup):
    """mimo_detect_mmse_sv: null / host / misaligned sigma2_v and bad dims are INVALID_ARG."""
    import torch
    plan, H, y, out, _ = setup
    s2v = torch.full((1,), 0.1, device="cuda")
    assert _call_sv(plan, H, y, s2v, out) == mimo.MIMO_OK
    assert plan.sync_status() == 0
    assert _call_sv(plan, H, y, None, out) == mimo.MIMO_ERR_INVALID_ARG
    host = np.full(1, 0.1, np.float32)
    assert _call_sv(plan, H, y, host.ctypes.data, out) == mimo.MIMO_ERR_INVALID_ARG
    assert _call_sv(plan, H, y, s2v.data_ptr() + 2, out) == mimo.MIMO_ERR_INVALID_ARG
    assert _call_sv(plan, H, y, s2v, out, nsym=13) == mimo.MIMO_ERR_INVALID_ARG
    with pytest.raises(ValueError):  # binding: one variance per H time block
        plan.detect(H, y, torch.full((2,), 0.1, device="cuda"))


def test_host_async_errors_and_empty(setup):
    """mimo_detect_mmse_host_async validates like the synchronous call; an empty grid is a no-op."""
    plan, H, y, out, w = setup
    f = plan._lib.mimo_detect_mmse_host_async
    llr = np.empty((14, 32, 4, 4), np.float32)
    args = lambda s2, nsym: (plan._h, w.H.ctypes.data_as(ctypes.c_void_p), w.y.ctypes.data_as(ctypes.c_void_p),
                             ctypes.c_float(s2), 4, 4, 32, nsym, 4, llr.ctypes.data_as(ctypes.c_void_p))
    assert f(*args(-1.0, 14)) == mimo.MIMO_ERR_INVALID_ARG
    assert f(*args(0.1, 13)) == mimo.MIMO_ERR_INVALID_ARG
    assert f(*args(0.1, 0)) == mimo.MIMO_OK
    assert f(*args(float(w.sigma2), 14)) == mimo.MIMO_OK
    assert plan.sync_status() == 0
    ref = plan.detect_host(w.H, w.y, float(w.sigma2))
    assert np.array_equal(llr, ref)
