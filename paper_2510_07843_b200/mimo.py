"""Thin ctypes binding of include/mimo.h (argument marshalling only).

Every step of the detector runs in libmimo.so's sm_100a kernels; this module
checks tensors (dtype, device, contiguity, shape), passes data_ptr()s and
torch's current CUDA stream, and turns status codes into MimoError. There is no
CPU fallback: without libmimo.so or a CUDA device it raises.

    plan = Plan(n_rx=4, n_layers=4, qm=4)                 # C2
    llr = plan.detect(H, y, sigma2)                       # H, y: complex64 CUDA tensors
"""
from __future__ import annotations

import ctypes
import os
import re

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "lib", "libmimo.so")
HEADER = os.path.join(os.path.dirname(_PKG), "include", "mimo.h")

MIMO_OK = 0
MIMO_ERR_INVALID_ARG = 1
MIMO_ERR_UNSUPPORTED = 2
MIMO_ERR_CUDA = 3
MIMO_ERR_NOT_PD = 4
MIMO_ERR_OOM = 5

LLR_F32, LLR_F16, LLR_I8 = 0, 1, 2
LU_STAGES = ("cov", "lu", "inv", "weights", "apply")  # mimo_detect_lmmse_lu stages (MIMO_LU_STAGES)
PLAN_OVERLAP_CALLS = 1
SYM_PER_SLOT = 14


class MimoError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{msg} [status {status}]")
        self.status = status


class _Desc(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("stream", ctypes.c_void_p), ("n_rx", ctypes.c_int),
                ("n_layers", ctypes.c_int), ("qam_order", ctypes.c_int), ("sc_per_h", ctypes.c_int),
                ("sym_per_h", ctypes.c_int), ("llr_type", ctypes.c_int), ("llr_scale", ctypes.c_float),
                ("flags", ctypes.c_int), ("kernel", ctypes.c_char_p), ("host_chunk_bytes", ctypes.c_longlong)]


_lib = None


def header_functions() -> list[str]:
    """Names of the functions include/mimo.h declares."""
    with open(HEADER) as f:
        src = f.read()
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\*?\s+\*?(mimo_\w+)\s*\(", src, re.M)))


def load_library(path: str | None = None):
    """Load libmimo.so (raises if it was not built: no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    p = path or LIB_PATH
    if not os.path.exists(p):
        raise RuntimeError(f"{p} not found: build it with `python -m paper_2510_07843_b200.build` "
                           "(there is no CPU fallback)")
    L = ctypes.CDLL(p)
    i, vp, f, ll = ctypes.c_int, ctypes.c_void_p, ctypes.c_float, ctypes.c_longlong
    L.mimo_plan_create.argtypes = [ctypes.POINTER(_Desc), ctypes.POINTER(vp)]
    L.mimo_plan_create.restype = i
    L.mimo_plan_set_stream.argtypes = [vp, vp]
    L.mimo_plan_set_stream.restype = i
    L.mimo_detect_mmse.argtypes = [vp, vp, vp, f, i, i, i, i, i, vp]
    L.mimo_detect_mmse.restype = i
    L.mimo_detect_mmse_ex.argtypes = [vp, vp, vp, f, i, i, i, i, i, vp, vp, vp]
    L.mimo_detect_mmse_ex.restype = i
    L.mimo_detect_mmse_sv.argtypes = [vp, vp, vp, vp, i, i, i, i, i, vp, vp, vp]
    L.mimo_detect_mmse_sv.restype = i
    L.mimo_detect_mmse_host.argtypes = [vp, vp, vp, f, i, i, i, i, i, vp]
    L.mimo_detect_mmse_host_async.argtypes = [vp, vp, vp, f, i, i, i, i, i, vp]
    L.mimo_detect_mmse_host_async.restype = i
    for nm in ("mimo_detect_mmse_bfp_host", "mimo_detect_mmse_bfp_host_async"):
        getattr(L, nm).argtypes = [vp, vp, vp, f, i, i, i, i, i, i, f, vp]
        getattr(L, nm).restype = i
    L.mimo_detect_mmse_host.restype = i
    L.mimo_detect_lmmse_lu.argtypes = [vp, vp, vp, f, i, i, i, i, i, i, vp, vp, vp, ctypes.POINTER(f)]
    L.mimo_detect_lmmse_lu.restype = i
    L.mimo_detect_irc.argtypes = [vp, vp, vp, vp, i, i, i, i, i, vp, vp, vp]
    L.mimo_detect_irc.restype = i
    L.mimo_detect_mmse_bfp.argtypes = [vp, vp, vp, f, i, i, i, i, i, i, f, vp, vp, vp]
    L.mimo_detect_mmse_bfp.restype = i
    L.mimo_plan_reserve.argtypes = [vp, i, i]
    L.mimo_plan_reserve.restype = i
    L.mimo_plan_sync_status.argtypes = [vp, ctypes.POINTER(ll)]
    L.mimo_plan_sync_status.restype = i
    L.mimo_plan_destroy.argtypes = [vp]
    L.mimo_plan_destroy.restype = i
    L.mimo_plan_kernel_name.argtypes = [vp]
    L.mimo_plan_kernel_name.restype = ctypes.c_char_p
    L.mimo_plan_launches_per_call.argtypes = [vp]
    L.mimo_plan_launches_per_call.restype = i
    L.mimo_plan_last_error.argtypes = [vp]
    L.mimo_plan_last_error.restype = ctypes.c_char_p
    L.mimo_last_error.restype = ctypes.c_char_p
    L.mimo_status_string.argtypes = [i]
    L.mimo_status_string.restype = ctypes.c_char_p
    L.mimo_abi_version.restype = i
    _lib = L
    return L


def _llr_code(dtype) -> int:
    import torch
    m = {torch.float32: LLR_F32, torch.float16: LLR_F16, torch.int8: LLR_I8,
         "f32": LLR_F32, "f16": LLR_F16, "i8": LLR_I8}
    if dtype not in m:
        raise ValueError(f"unsupported LLR dtype {dtype}")
    return m[dtype]


def _llr_torch_dtype(code: int):
    import torch
    return {LLR_F32: torch.float32, LLR_F16: torch.float16, LLR_I8: torch.int8}[code]


class Plan:
    """A detector plan bound to one CUDA device (wraps mimo_plan_t)."""

    def __init__(self, n_rx: int, n_layers: int, qm: int, *, sc_per_h: int = 1,
                 sym_per_h: int = SYM_PER_SLOT, llr_dtype="f32", llr_scale: float = 1.0,
                 device=None, stream=None, overlap_calls: bool = False, kernel: str | None = None,
                 host_chunk_bytes: int = 0):
        import torch
        L = load_library()
        if not torch.cuda.is_available():
            raise RuntimeError("no CUDA device: the detector has no CPU fallback")
        if device is None:
            idx = torch.cuda.current_device()
        elif isinstance(device, int):
            idx = device
        else:
            idx = torch.device(device).index or 0
        dev = torch.device("cuda", idx)
        self.device = dev
        self.n_rx, self.n_layers, self.qm = n_rx, n_layers, qm
        self.sc_per_h, self.sym_per_h = sc_per_h, sym_per_h
        self.llr_type = _llr_code(llr_dtype)
        self.llr_dtype = _llr_torch_dtype(self.llr_type)
        self._fixed_stream = stream
        d = _Desc(dev.index, ctypes.c_void_p(self._stream_ptr()), n_rx, n_layers, qm, sc_per_h, sym_per_h,
                  self.llr_type, float(llr_scale), PLAN_OVERLAP_CALLS if overlap_calls else 0,
                  kernel.encode() if kernel else None, int(host_chunk_bytes))
        h = ctypes.c_void_p()
        st = L.mimo_plan_create(ctypes.byref(d), ctypes.byref(h))
        if st != MIMO_OK:
            raise MimoError(st, L.mimo_last_error().decode())
        self._h = h
        self._lib = L

    # -- helpers -----------------------------------------------------------
    def _stream_ptr(self) -> int:
        import torch
        if self._fixed_stream is not None:
            s = self._fixed_stream
            return s.cuda_stream if hasattr(s, "cuda_stream") else int(s)
        return torch.cuda.current_stream(self.device).cuda_stream

    def _check(self, st: int):
        if st != MIMO_OK:
            raise MimoError(st, self._lib.mimo_plan_last_error(self._h).decode()
                            or self._lib.mimo_status_string(st).decode())

    @property
    def kernel_name(self) -> str:
        return self._lib.mimo_plan_kernel_name(self._h).decode()

    @property
    def launches_per_call(self) -> int:
        return self._lib.mimo_plan_launches_per_call(self._h)

    def shapes(self, n_sc: int, n_sym: int) -> dict:
        n_units = (n_sym // self.sym_per_h) * (n_sc // self.sc_per_h)
        return dict(H=(n_sym // self.sym_per_h, n_sc // self.sc_per_h, self.n_rx, self.n_layers),
                    y=(n_sym, n_sc, self.n_rx), llr=(n_sym, n_sc, self.n_layers, self.qm),
                    xhat=(n_sym, n_sc, self.n_layers), sinr=(n_units, self.n_layers))

    def _dev_tensor(self, t, name, dtype, shape):
        import torch
        if not isinstance(t, torch.Tensor) or t.device != self.device:
            raise ValueError(f"{name} must be a torch tensor on {self.device}")
        if t.dtype != dtype:
            raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
        if not t.is_contiguous():
            raise ValueError(f"{name} must be contiguous")
        # exact shape, or a flat view with the right element count (a transposed / reshaped
        # tensor of the same size is rejected rather than silently misread)
        if tuple(t.shape) != tuple(shape) and not (t.dim() == 1 and t.numel() == int(np.prod(shape))):
            raise ValueError(f"{name} has shape {tuple(t.shape)}, expected {tuple(shape)}")
        return t

    # -- API ---------------------------------------------------------------
    def detect(self, H, y, sigma2, out=None, xhat=None, sinr=None, *, n_sc=None, n_sym=None,
               want_llr: bool = True):
        """Detect all REs of y (device tensors). Returns the LLR tensor (or None).
        sigma2: a float, or a device float32 tensor [n_sym / sym_per_h] of per-slot (per H time
        block) noise variances, each finite and > 0 (mimo_detect_mmse_sv)."""
        import torch
        n_sym = y.shape[0] if n_sym is None else n_sym
        n_sc = y.shape[1] if n_sc is None else n_sc
        sh = self.shapes(n_sc, n_sym)
        self._dev_tensor(H, "H", torch.complex64, sh["H"])
        self._dev_tensor(y, "y", torch.complex64, sh["y"])
        if want_llr and out is None:
            out = torch.empty(sh["llr"], dtype=self.llr_dtype, device=self.device)
        if out is not None:
            self._dev_tensor(out, "out", self.llr_dtype, sh["llr"])
        if xhat is not None:
            self._dev_tensor(xhat, "xhat", torch.complex64, sh["xhat"])
        if sinr is not None:
            self._dev_tensor(sinr, "sinr", torch.float32, sh["sinr"])
        if self._fixed_stream is None:
            self._lib.mimo_plan_set_stream(self._h, ctypes.c_void_p(self._stream_ptr()))
        ptr = (lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None)
        if isinstance(sigma2, torch.Tensor):
            self._dev_tensor(sigma2, "sigma2", torch.float32, (n_sym // self.sym_per_h,))
            st = self._lib.mimo_detect_mmse_sv(self._h, ptr(H), ptr(y), ptr(sigma2), self.n_rx, self.n_layers,
                                               n_sc, n_sym, self.qm, ptr(out), ptr(xhat), ptr(sinr))
        elif xhat is None and sinr is None:
            st = self._lib.mimo_detect_mmse(self._h, ptr(H), ptr(y), ctypes.c_float(sigma2), self.n_rx,
                                            self.n_layers, n_sc, n_sym, self.qm, ptr(out))
        else:
            st = self._lib.mimo_detect_mmse_ex(self._h, ptr(H), ptr(y), ctypes.c_float(sigma2), self.n_rx,
                                               self.n_layers, n_sc, n_sym, self.qm, ptr(out), ptr(xhat),
                                               ptr(sinr))
        self._check(st)
        return out

    def detect_lu(self, H, y, sigma2: float, *, precision: int = 32, out=None, xhat=None, sinr=None,
                  timing: bool = False, want_llr: bool = True):
        """Paper-literal route (covariance R, pivoted LU, substitution inversion, W = H^H R^-1)
        as five stage kernels; precision 32 ("PS") or 64 ("PD"). Returns the LLR tensor, or
        (llr, {stage: device microseconds}) when timing=True (the call then synchronises)."""
        import torch
        n_sym, n_sc = y.shape[0], y.shape[1]
        sh = self.shapes(n_sc, n_sym)
        self._dev_tensor(H, "H", torch.complex64, sh["H"])
        self._dev_tensor(y, "y", torch.complex64, sh["y"])
        if want_llr and out is None:
            out = torch.empty(sh["llr"], dtype=self.llr_dtype, device=self.device)
        if out is not None:
            self._dev_tensor(out, "out", self.llr_dtype, sh["llr"])
        if xhat is not None:
            self._dev_tensor(xhat, "xhat", torch.complex64, sh["xhat"])
        if sinr is not None:
            self._dev_tensor(sinr, "sinr", torch.float32, sh["sinr"])
        if self._fixed_stream is None:
            self._lib.mimo_plan_set_stream(self._h, ctypes.c_void_p(self._stream_ptr()))
        ptr = (lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None)
        st_us = (ctypes.c_float * len(LU_STAGES))() if timing else None
        st = self._lib.mimo_detect_lmmse_lu(self._h, ptr(H), ptr(y), ctypes.c_float(sigma2), self.n_rx,
                                            self.n_layers, n_sc, n_sym, self.qm, int(precision), ptr(out),
                                            ptr(xhat), ptr(sinr), st_us)
        self._check(st)
        if timing:
            return out, dict(zip(LU_STAGES, (float(v) for v in st_us)))
        return out

    def detect_irc(self, H, y, Rnn, *, out=None, xhat=None, sinr=None, want_llr: bool = True):
        """Coloured-noise / interference-rejection detection: Rnn complex64 [n_units][n_rx][n_rx] on the device."""
        import torch
        n_sym, n_sc = y.shape[0], y.shape[1]
        sh = self.shapes(n_sc, n_sym)
        self._dev_tensor(H, "H", torch.complex64, sh["H"])
        self._dev_tensor(y, "y", torch.complex64, sh["y"])
        n_units = sh["sinr"][0]
        self._dev_tensor(Rnn, "Rnn", torch.complex64, (n_units, self.n_rx, self.n_rx))
        if want_llr and out is None:
            out = torch.empty(sh["llr"], dtype=self.llr_dtype, device=self.device)
        if out is not None:
            self._dev_tensor(out, "out", self.llr_dtype, sh["llr"])
        if xhat is not None:
            self._dev_tensor(xhat, "xhat", torch.complex64, sh["xhat"])
        if sinr is not None:
            self._dev_tensor(sinr, "sinr", torch.float32, sh["sinr"])
        if self._fixed_stream is None:
            self._lib.mimo_plan_set_stream(self._h, ctypes.c_void_p(self._stream_ptr()))
        ptr = (lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None)
        self._check(self._lib.mimo_detect_irc(self._h, ptr(H), ptr(y), ptr(Rnn), self.n_rx, self.n_layers, n_sc,
                                              n_sym, self.qm, ptr(out), ptr(xhat), ptr(sinr)))
        return out

    def detect_bfp(self, H, y_bfp, sigma2: float, *, n_sym: int, n_sc: int, iq_width: int = 9,
                   bfp_scale: float = 2.0 ** -8, out=None, xhat=None, sinr=None, want_llr: bool = True):
        """Detect from BFP-compressed y (uint8 device tensor [n_sym][n_sc/12][n_rx][block_bytes])."""
        import torch
        sh = self.shapes(n_sc, n_sym)
        self._dev_tensor(H, "H", torch.complex64, sh["H"])
        bb = ((1 + 3 * iq_width) + 3) & ~3
        self._dev_tensor(y_bfp, "y_bfp", torch.uint8, (n_sym, n_sc // 12, self.n_rx, bb))
        if want_llr and out is None:
            out = torch.empty(sh["llr"], dtype=self.llr_dtype, device=self.device)
        if out is not None:
            self._dev_tensor(out, "out", self.llr_dtype, sh["llr"])
        if xhat is not None:
            self._dev_tensor(xhat, "xhat", torch.complex64, sh["xhat"])
        if sinr is not None:
            self._dev_tensor(sinr, "sinr", torch.float32, sh["sinr"])
        if self._fixed_stream is None:
            self._lib.mimo_plan_set_stream(self._h, ctypes.c_void_p(self._stream_ptr()))
        ptr = (lambda t: ctypes.c_void_p(t.data_ptr()) if t is not None else None)
        self._check(self._lib.mimo_detect_mmse_bfp(self._h, ptr(H), ptr(y_bfp), ctypes.c_float(sigma2), self.n_rx,
                                                   self.n_layers, n_sc, n_sym, self.qm, int(iq_width),
                                                   ctypes.c_float(bfp_scale), ptr(out), ptr(xhat), ptr(sinr)))
        return out

    def detect_host(self, H, y, sigma2: float, out=None, wait: bool = True):
        """End-to-end detect with HOST buffers (numpy or CPU tensors; pin them for overlap).
        wait=False: mimo_detect_mmse_host_async -- returns at once; call sync_status() before
        reading `out` or reusing H / y (consecutive calls overlap their transfers)."""
        import torch
        to_np = (lambda t: t.numpy() if isinstance(t, torch.Tensor) else t)
        Hn, yn = to_np(H), to_np(y)
        if Hn.dtype != np.complex64 or yn.dtype != np.complex64:
            raise ValueError("H and y must be complex64")
        if not (Hn.flags.c_contiguous and yn.flags.c_contiguous):
            raise ValueError("H and y must be C-contiguous")
        n_sym, n_sc = yn.shape[0], yn.shape[1]
        sh = self.shapes(n_sc, n_sym)
        if Hn.size != int(np.prod(sh["H"])) or yn.size != int(np.prod(sh["y"])):
            raise ValueError("H / y sizes do not match the plan")
        if out is None:
            out = np.empty(sh["llr"], dtype={LLR_F32: np.float32, LLR_F16: np.float16, LLR_I8: np.int8}[self.llr_type])
        on = to_np(out)
        if on.size != int(np.prod(sh["llr"])) or not on.flags.c_contiguous:
            raise ValueError("out has the wrong size or is not contiguous")
        if self._fixed_stream is None:
            self._lib.mimo_plan_set_stream(self._h, ctypes.c_void_p(self._stream_ptr()))
        fn = self._lib.mimo_detect_mmse_host if wait else self._lib.mimo_detect_mmse_host_async
        st = fn(self._h, Hn.ctypes.data_as(ctypes.c_void_p), yn.ctypes.data_as(ctypes.c_void_p),
                ctypes.c_float(sigma2), self.n_rx, self.n_layers, n_sc, n_sym, self.qm,
                on.ctypes.data_as(ctypes.c_void_p))
        self._check(st)
        return out

    def detect_bfp_host(self, H, y_bfp, sigma2: float, *, n_sym: int, n_sc: int, iq_width: int = 9,
                        bfp_scale: float = 2.0 ** -8, out=None, wait: bool = True):
        """End-to-end detect with HOST buffers and block-floating-point y (mimo_detect_mmse_bfp_host[_async]):
        H complex64, y_bfp uint8 [n_sym][n_sc/12][n_rx][block_bytes] (numpy or CPU tensors; pin them)."""
        import torch
        to_np = (lambda t: t.numpy() if isinstance(t, torch.Tensor) else t)
        Hn, yn = to_np(H), to_np(y_bfp)
        if Hn.dtype != np.complex64 or yn.dtype != np.uint8:
            raise ValueError("H must be complex64 and y_bfp uint8")
        if not (Hn.flags.c_contiguous and yn.flags.c_contiguous):
            raise ValueError("H and y_bfp must be C-contiguous")
        bb = ((1 + 3 * iq_width) + 3) & ~3
        sh = self.shapes(n_sc, n_sym)
        if Hn.size != int(np.prod(sh["H"])) or yn.size != n_sym * (n_sc // 12) * self.n_rx * bb:
            raise ValueError("H / y_bfp sizes do not match the plan")
        if out is None:
            out = np.empty(sh["llr"], dtype={LLR_F32: np.float32, LLR_F16: np.float16, LLR_I8: np.int8}[self.llr_type])
        on = to_np(out)
        if on.size != int(np.prod(sh["llr"])) or not on.flags.c_contiguous:
            raise ValueError("out has the wrong size or is not contiguous")
        if self._fixed_stream is None:
            self._lib.mimo_plan_set_stream(self._h, ctypes.c_void_p(self._stream_ptr()))
        fn = self._lib.mimo_detect_mmse_bfp_host if wait else self._lib.mimo_detect_mmse_bfp_host_async
        st = fn(self._h, Hn.ctypes.data_as(ctypes.c_void_p), yn.ctypes.data_as(ctypes.c_void_p), ctypes.c_float(sigma2),
                self.n_rx, self.n_layers, n_sc, n_sym, self.qm, int(iq_width), ctypes.c_float(bfp_scale),
                on.ctypes.data_as(ctypes.c_void_p))
        self._check(st)
        return out

    def reserve(self, n_sc: int, n_sym: int):
        """Pre-allocate the kernel workspace for calls up to n_sc x n_sym (do this before graph capture)."""
        self._check(self._lib.mimo_plan_reserve(self._h, n_sc, n_sym))

    def sync_status(self) -> int:
        """Synchronise; return the number of units flagged by the Cholesky guard since the last call."""
        n = ctypes.c_longlong(0)
        st = self._lib.mimo_plan_sync_status(self._h, ctypes.byref(n))
        if st not in (MIMO_OK, MIMO_ERR_NOT_PD):
            self._check(st)
        return int(n.value)

    def close(self):
        if getattr(self, "_h", None):
            self._lib.mimo_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
