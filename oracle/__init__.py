"""fp64 CPU oracle of the per-RE MMSE detector + max-log demapper (ctypes wrapper).

TEST INFRASTRUCTURE ONLY: only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this package. It shares no code
with paper_2510_07843_b200/ (the CUDA product path), and the product never
imports it. See oracle/mmse_oracle.c for the per-function paper citations.

Parity status (DESIGN.md §"Oracle pins"): every function is pinned by
tests/test_oracle_pins.py except the output conventions (LLR scale, clamp
values, output layout), which are "parity unpinned" by choice (reading R10/R13).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "mmse_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

LLR_TYPES = {"f32": 0, "f16": 1, "i8": 2}


def build(force: bool = False) -> str:
    """Compile the C oracle with gcc (plain -O2, C99 complex, OpenMP)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=gnu11", "-fPIC", "-shared", "-fopenmp",
                               "-fno-fast-math", "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = ctypes.CDLL(_LIB)
            d, i, l, p = ctypes.c_double, ctypes.c_int, ctypes.c_long, ctypes.c_void_p
            L.oracle_version.restype = i
            L.oracle_pivot_tau.restype = d
            L.oracle_constellation.argtypes = [i, p, p]
            L.oracle_constellation.restype = i
            L.oracle_maxlog.argtypes = [i, i, p, p, p]
            L.oracle_gram.argtypes = [i, i, p, d, p]
            L.oracle_covariance.argtypes = [i, i, p, d, p]
            L.oracle_cholesky.argtypes = [i, p, p]
            L.oracle_cholesky.restype = i
            L.oracle_lu_factor.argtypes = [i, p, p, p]
            L.oracle_lu_factor.restype = i
            L.oracle_lu_forward.argtypes = [i, p, p, p, p]
            L.oracle_lu_backward.argtypes = [i, p, p, p]
            L.oracle_lu_invert.argtypes = [i, p, p]
            L.oracle_lu_invert.restype = i
            L.oracle_weights_chol.argtypes = [i, i, p, d, p]
            L.oracle_weights_chol.restype = i
            L.oracle_weights_lu.argtypes = [i, i, p, d, p]
            L.oracle_weights_lu.restype = i
            L.oracle_detect.argtypes = [i, i, i, i, l, i, p, p, ctypes.c_float, p, p, p, p, i]
            L.oracle_detect.restype = l
            L.oracle_quantize.argtypes = [i, l, p, d, p]
            L.oracle_detect_irc.argtypes = [i, i, i, l, i, p, p, p, p, p, p, p, i]
            L.oracle_detect_irc.restype = l
            L.oracle_bfp_decode.argtypes = [l, i, d, p, p]
            L.oracle_bfp_decode.restype = None
            L.oracle_max_threads.restype = i
            _lib = L
    return _lib


def _c128(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.complex128)


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def pivot_tau() -> float:
    return lib().oracle_pivot_tau()


def max_threads() -> int:
    return lib().oracle_max_threads()


def constellation(qm: int) -> np.ndarray:
    """Complex points indexed by label L (b_0 = MSB of L)."""
    re = np.zeros(1 << qm)
    im = np.zeros(1 << qm)
    if lib().oracle_constellation(qm, _ptr(re), _ptr(im)) != (1 << qm):
        raise ValueError(f"unsupported qm {qm}")
    return re + 1j * im


def maxlog(qm: int, x, sinr) -> np.ndarray:
    x = _c128(np.atleast_1d(x))
    s = np.ascontiguousarray(np.broadcast_to(sinr, x.shape), dtype=np.float64)
    out = np.zeros(x.shape + (qm,))
    lib().oracle_maxlog(qm, x.size, _ptr(x), _ptr(s), _ptr(out))
    return out


def gram(H, sigma2: float) -> np.ndarray:
    H = _c128(H)
    nr, nl = H.shape
    G = np.zeros((nl, nl), np.complex128)
    lib().oracle_gram(nr, nl, _ptr(H), float(sigma2), _ptr(G))
    return G


def covariance(H, sigma2: float) -> np.ndarray:
    H = _c128(H)
    nr, nl = H.shape
    R = np.zeros((nr, nr), np.complex128)
    lib().oracle_covariance(nr, nl, _ptr(H), float(sigma2), _ptr(R))
    return R


def cholesky(G):
    """Returns L, or None if the pivot guard (reading R17) trips."""
    G = _c128(G)
    L = np.zeros_like(G)
    return L if lib().oracle_cholesky(G.shape[0], _ptr(G), _ptr(L)) else None


def lu_factor(A):
    A = _c128(A)
    n = A.shape[0]
    LU = np.zeros_like(A)
    perm = np.zeros(n, np.int32)
    ok = lib().oracle_lu_factor(n, _ptr(A), _ptr(LU), _ptr(perm))
    return (LU, perm) if ok else None


def lu_forward(LU, perm, b) -> np.ndarray:
    LU, b = _c128(LU), _c128(b)
    perm = np.ascontiguousarray(perm, np.int32)
    z = np.zeros_like(b)
    lib().oracle_lu_forward(LU.shape[0], _ptr(LU), _ptr(perm), _ptr(b), _ptr(z))
    return z


def lu_backward(LU, z) -> np.ndarray:
    LU, z = _c128(LU), _c128(z)
    x = np.zeros_like(z)
    lib().oracle_lu_backward(LU.shape[0], _ptr(LU), _ptr(z), _ptr(x))
    return x


def lu_invert(A):
    A = _c128(A)
    X = np.zeros_like(A)
    return X if lib().oracle_lu_invert(A.shape[0], _ptr(A), _ptr(X)) else None


def weights_chol(H, sigma2: float):
    H = _c128(H)
    nr, nl = H.shape
    W = np.zeros((nl, nr), np.complex128)
    return W if lib().oracle_weights_chol(nr, nl, _ptr(H), float(sigma2), _ptr(W)) else None


def weights_lu(H, sigma2: float):
    H = _c128(H)
    nr, nl = H.shape
    W = np.zeros((nl, nr), np.complex128)
    return W if lib().oracle_weights_lu(nr, nl, _ptr(H), float(sigma2), _ptr(W)) else None


def detect(H_units, Y_units, sigma2, qm: int, *, route: str = "chol", threads: int = 1):
    """Detect a batch of H-units.

    H_units complex64 [n_units][nr][nl]; Y_units complex64 [n_units][n_re][nr]
    (REs of each unit in unit order, see synth.unit_gather); sigma2 fp32.
    Returns dict(xhat complex128 [u][e][nl], sinr [u][nl], llr fp64 [u][e][nl][qm],
    ok bool [u], n_failed).
    """
    H = np.ascontiguousarray(H_units, dtype=np.complex64)
    Y = np.ascontiguousarray(Y_units, dtype=np.complex64)
    nu, nr, nl = H.shape
    ne = Y.shape[1]
    assert Y.shape == (nu, ne, nr), (Y.shape, H.shape)
    xt = np.zeros((nu, ne, nl), np.complex128)
    sinr = np.zeros((nu, nl))
    llr = np.zeros((nu, ne, nl, qm))
    ok = np.zeros(nu, np.int8)
    nb = lib().oracle_detect(1 if route == "lu" else 0, nr, nl, qm, nu, ne, _ptr(H), _ptr(Y),
                             ctypes.c_float(np.float32(sigma2)), _ptr(xt), _ptr(sinr), _ptr(llr),
                             _ptr(ok), int(threads))
    if nb < 0:
        raise ValueError("unsupported qm")
    return dict(xhat=xt, sinr=sinr, llr=llr, ok=ok.astype(bool), n_failed=int(nb))


def detect_irc(H_units, Y_units, R_units, qm: int, *, threads: int = 1):
    """Coloured-noise (interference-rejection) detector, W = H^H (H H^H + R_nn)^-1 per unit.

    R_units complex64 [n_units][nr][nr] (Hermitian positive definite noise + interference covariance).
    Same outputs as detect()."""
    H = np.ascontiguousarray(H_units, dtype=np.complex64)
    Y = np.ascontiguousarray(Y_units, dtype=np.complex64)
    R = np.ascontiguousarray(R_units, dtype=np.complex64)
    nu, nr, nl = H.shape
    ne = Y.shape[1]
    assert Y.shape == (nu, ne, nr) and R.shape == (nu, nr, nr), (Y.shape, R.shape)
    xt = np.zeros((nu, ne, nl), np.complex128)
    sinr = np.zeros((nu, nl))
    llr = np.zeros((nu, ne, nl, qm))
    ok = np.zeros(nu, np.int8)
    nb = lib().oracle_detect_irc(nr, nl, qm, nu, ne, _ptr(H), _ptr(Y), _ptr(R), _ptr(xt), _ptr(sinr), _ptr(llr),
                                 _ptr(ok), int(threads))
    if nb < 0:
        raise ValueError("unsupported qm")
    return dict(xhat=xt, sinr=sinr, llr=llr, ok=ok.astype(bool), n_failed=int(nb))


def bfp_decode(blocks, iq_width: int, scale: float) -> np.ndarray:
    """BFP blocks uint8 [..., block_bytes] -> complex64 [..., 12] (reading R25)."""
    b = np.ascontiguousarray(blocks, dtype=np.uint8)
    bb = ((1 + 3 * iq_width) + 3) & ~3
    assert b.shape[-1] == bb, (b.shape, bb)
    n = b.size // bb
    out = np.zeros(n * 24, np.float32)
    lib().oracle_bfp_decode(n, int(iq_width), float(scale), _ptr(b), _ptr(out))
    return out.view(np.complex64).reshape(b.shape[:-1] + (12,))


def quantize(llr, llr_type: str, scale: float = 1.0) -> np.ndarray:
    """fp64 LLRs -> float32 / float16 / int8 (reading R10)."""
    v = np.ascontiguousarray(llr, dtype=np.float64)
    t = LLR_TYPES[llr_type]
    if t == 0:
        out = np.zeros(v.shape, np.float32)
    elif t == 1:
        out = np.zeros(v.shape, np.uint16)
    else:
        out = np.zeros(v.shape, np.int8)
    lib().oracle_quantize(t, v.size, _ptr(v), float(scale), _ptr(out))
    return out.view(np.float16) if t == 1 else out
