"""C-ABI library checks that need no GPU: it loads, exports every symbol
include/mimo.h declares, and validates arguments before touching CUDA."""
import ctypes
import subprocess

import pytest

from paper_2510_07843_b200 import build, mimo


@pytest.fixture(scope="module")
def lib():
    build.build()
    return mimo.load_library()


def test_header_declares_the_boundary():
    names = mimo.header_functions()
    for n in ["mimo_plan_create", "mimo_detect_mmse", "mimo_plan_destroy", "mimo_detect_mmse_ex",
              "mimo_detect_mmse_host", "mimo_plan_sync_status", "mimo_status_string"]:
        assert n in names


def test_exports_every_header_symbol(lib):
    out = subprocess.run(["nm", "-D", "--defined-only", mimo.LIB_PATH], capture_output=True, text=True).stdout
    exported = {ln.split()[-1] for ln in out.splitlines() if ln.strip()}
    for n in mimo.header_functions():
        assert n in exported, n
        getattr(lib, n)  # resolvable through ctypes


def test_no_torch_or_oracle_in_library():
    out = subprocess.run(["ldd", mimo.LIB_PATH], capture_output=True, text=True).stdout
    assert "torch" not in out and "oracle" not in out
    strings = subprocess.run(["nm", "-D", mimo.LIB_PATH], capture_output=True, text=True).stdout
    assert "oracle_" not in strings


def test_no_environment_configuration_or_ablations_in_library():
    """The plan descriptor is the library's only configuration: no MIMO_* environment
    knobs and no wrong-on-purpose timing-ablation kernels are compiled into libmimo.so."""
    blob = open(mimo.LIB_PATH, "rb").read()
    for s in (b"MIMO_FORCE_KERNEL", b"MIMO_HOST_CHUNK_BYTES", b"MIMO_BFP_G", b"ablation", b"nosetup", b"NoSetup"):
        assert s not in blob, s
    src = open(__import__("os").path.join(mimo._PKG, "csrc", "mimo_api.cu")).read()
    assert "getenv" not in src


def test_descriptor_layout_matches_header():
    """ctypes mirror of mimo_plan_desc_t: field order and the two ABI-2 fields."""
    names = [f[0] for f in mimo._Desc._fields_]
    assert names[-2:] == ["kernel", "host_chunk_bytes"]
    hdr = open(mimo.HEADER).read()
    assert "const char* kernel;" in hdr and "long long host_chunk_bytes;" in hdr


def test_abi_version_and_status_strings(lib):
    assert lib.mimo_abi_version() == 2
    for s in range(6):
        assert lib.mimo_status_string(s).decode().startswith("MIMO_")
    assert lib.mimo_plan_destroy(None) == mimo.MIMO_OK


def _desc(**kw):
    d = dict(device=0, stream=None, n_rx=4, n_layers=4, qam_order=4, sc_per_h=1, sym_per_h=14,
             llr_type=0, llr_scale=1.0, flags=0)
    d.update(kw)
    return mimo._Desc(d["device"], d["stream"], d["n_rx"], d["n_layers"], d["qam_order"], d["sc_per_h"],
                      d["sym_per_h"], d["llr_type"], d["llr_scale"], d["flags"])


@pytest.mark.parametrize("bad", [dict(n_rx=0), dict(n_rx=65), dict(n_layers=5), dict(n_layers=0),
                                 dict(qam_order=16), dict(qam_order=3), dict(sc_per_h=0), dict(sym_per_h=0),
                                 dict(llr_type=3), dict(llr_scale=0.0), dict(llr_scale=float("nan")),
                                 dict(device=-1), dict(n_rx=32, n_layers=17), dict(flags=2)])
def test_create_rejects_bad_descriptor(lib, bad):
    h = ctypes.c_void_p()
    st = lib.mimo_plan_create(ctypes.byref(_desc(**bad)), ctypes.byref(h))
    assert st == mimo.MIMO_ERR_INVALID_ARG
    assert h.value is None
    assert lib.mimo_last_error().decode()


def test_create_null_args(lib):
    h = ctypes.c_void_p()
    assert lib.mimo_plan_create(None, ctypes.byref(h)) == mimo.MIMO_ERR_INVALID_ARG
    assert lib.mimo_plan_create(ctypes.byref(_desc()), None) == mimo.MIMO_ERR_INVALID_ARG


def test_calls_on_null_plan(lib):
    assert lib.mimo_detect_mmse(None, None, None, 0.1, 4, 4, 12, 14, 4, None) == mimo.MIMO_ERR_INVALID_ARG
    assert lib.mimo_plan_sync_status(None, None) == mimo.MIMO_ERR_INVALID_ARG
    assert lib.mimo_plan_kernel_name(None) == b""


def test_no_device_fails_loudly(lib):
    """Without a GPU a valid descriptor is refused with MIMO_ERR_CUDA (no CPU fallback)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("has a GPU")
    h = ctypes.c_void_p()
    assert lib.mimo_plan_create(ctypes.byref(_desc()), ctypes.byref(h)) == mimo.MIMO_ERR_CUDA
    with pytest.raises(RuntimeError):
        mimo.Plan(4, 4, 4)
