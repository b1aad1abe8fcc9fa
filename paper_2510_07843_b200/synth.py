"""Seeded synthetic workloads for the per-RE MMSE detector (shared by tests, bench, smoke).

This module holds NO detection arithmetic. It draws channels, bits and noise,
maps bits to QAM symbols (the transmitter side), forms y = H x + n in fp64 and
casts H and y to complex64, which are then the canonical inputs of both the
CUDA path and the fp64 oracle (SURVEY.md §8(d) "Synthetic inputs").

Workloads stand in for the paper's link-level simulator (§IV:
"MIMO-OFDM transmission using 15 kHz subcarrier spacing and 60 resource blocks
... 3GPP TDL-C"). TDL-C and the MCS tables are not available, so
BASELINE.json's five configs use i.i.d. / Kronecker Rayleigh channels; the
recipe is stated in DESIGN.md §"Input recipe".

Layouts (DESIGN.md §"Data layout in HBM"):
  H    complex64 [n_slots][n_fb][n_rx][n_layers]    n_fb = n_sc / sc_per_h, row = rx
  y    complex64 [n_sym][n_sc][n_rx]                n_sym = 14 * n_slots
  bits uint8     [n_sym][n_sc][n_layers][qm]        bit j of a symbol = b_j (38.211 order)
  llr  (any)     [n_sym][n_sc][n_layers][qm]
An H-unit u = slot * n_fb + fb owns the REs (sym, sc) with sym in the slot's
14 symbols and sc in block fb; inside a unit REs are ordered symbol-major.
"""
from __future__ import annotations

import dataclasses
import hashlib

import numpy as np

SYM_PER_SLOT = 14  # NR slot, normal cyclic prefix

# BASELINE.json "configs", in order (C1..C5). sigma2 = 10^(-SNR/10), reading R8
# (C1 states "SNR 10 dB (sigma^2 = 0.1)" explicitly).
CONFIGS = {
    1: dict(name="C1", n_rx=2, n_layers=2, qm=2, n_sc=12, n_slots=1, sc_per_h=1,
            channel="iid", chan_var=1.0, snr_db=10.0, llr="f32"),
    2: dict(name="C2", n_rx=4, n_layers=4, qm=4, n_sc=3276, n_slots=10, sc_per_h=1,
            channel="iid", chan_var=1.0, snr_db=15.0, llr="f32"),
    3: dict(name="C3", n_rx=8, n_layers=4, qm=6, n_sc=3276, n_slots=20, sc_per_h=12,
            channel="kron", chan_var=1.0, rho=0.5, snr_db=20.0, llr="i8"),
    4: dict(name="C4", n_rx=16, n_layers=8, qm=8, n_sc=3276, n_slots=20, sc_per_h=1,
            channel="iid", chan_var=1.0 / 16, snr_db=28.0, llr="f16"),
    5: dict(name="C5", n_rx=64, n_layers=16, qm=6, n_sc=3276, n_slots=40, sc_per_h=12,
            channel="iid", chan_var=1.0 / 64, snr_db=20.0, llr="i8"),
    # Context-only shape of the paper's own timing: 4x4,
    # 60 RB x 12 = 720 subcarriers, one TTI. Not a BASELINE config.
    "P": dict(name="P", n_rx=4, n_layers=4, qm=4, n_sc=720, n_slots=1, sc_per_h=1,
              channel="iid", chan_var=1.0, snr_db=15.0, llr="f32"),
}

# Per-axis PAM normalisation of the 38.211 constellations (transmitter side).
_QAM_NORM = {2: 2.0, 4: 10.0, 6: 42.0, 8: 170.0}


def sigma2_of(snr_db: float) -> np.float32:
    """Total complex noise variance sigma^2 = 10^(-SNR/10), rounded to fp32 (reading R8)."""
    return np.float32(10.0 ** (-snr_db / 10.0))


def qam_modulate(bits: np.ndarray, qm: int) -> np.ndarray:
    """Map bits [..., qm] (b_0 first) to unit-power complex symbols, 3GPP 38.211 §5.1 form.

    Bits b_0, b_2, ... drive I and b_1, b_3, ... drive Q; per axis with m = qm/2
    bits c_0..c_{m-1}: v = (1-2c_{m-1}); v = (1-2c_i)(2^{m-1-i} - v) for i = m-2..0.
    """
    m = qm // 2
    b = bits.astype(np.int64)
    axes = []
    for off in (0, 1):
        c = [b[..., 2 * i + off] for i in range(m)]
        v = 1 - 2 * c[m - 1]
        for i in range(m - 2, -1, -1):
            v = (1 - 2 * c[i]) * ((1 << (m - 1 - i)) - v)
        axes.append(v.astype(np.float64))
    return (axes[0] + 1j * axes[1]) / np.sqrt(_QAM_NORM[qm])


def exp_corr_chol(n: int, rho: float) -> np.ndarray:
    """Lower Cholesky factor C of the exponential correlation matrix R_ij = rho^|i-j|."""
    idx = np.arange(n)
    r = rho ** np.abs(idx[:, None] - idx[None, :])
    return np.linalg.cholesky(r)


def _cn(rng: np.random.Generator, shape, var: float) -> np.ndarray:
    """Circularly-symmetric complex Gaussian CN(0, var), drawn as (re, im) pairs in fp64."""
    g = rng.standard_normal(tuple(shape) + (2,))
    return (g[..., 0] + 1j * g[..., 1]) * np.sqrt(var / 2.0)


def unit_gather(grid: np.ndarray, n_slots: int, n_sc: int, sc_per_h: int, sym_per_h: int = SYM_PER_SLOT) -> np.ndarray:
    """[n_sym][n_sc][...] -> [n_units][sym_per_h*sc_per_h][...] (symbol-major inside a unit). Indexing only."""
    n_fb = n_sc // sc_per_h
    n_tb = grid.shape[0] // sym_per_h
    tail = grid.shape[2:]
    g = grid.reshape((n_tb, sym_per_h, n_fb, sc_per_h) + tail)
    g = np.moveaxis(g, 2, 1)  # [time block][fb][sym][f]...
    return g.reshape((n_tb * n_fb, sym_per_h * sc_per_h) + tail)


def unit_scatter(units: np.ndarray, n_slots: int, n_sc: int, sc_per_h: int, sym_per_h: int = SYM_PER_SLOT) -> np.ndarray:
    """Inverse of unit_gather. Indexing only."""
    n_fb = n_sc // sc_per_h
    n_tb = units.shape[0] // n_fb
    tail = units.shape[2:]
    g = units.reshape((n_tb, n_fb, sym_per_h, sc_per_h) + tail)
    g = np.moveaxis(g, 1, 2)
    return np.ascontiguousarray(g.reshape((n_tb * sym_per_h, n_sc) + tail))


def unit_re_index(u: int, n_sc: int, sc_per_h: int, sym_per_h: int = SYM_PER_SLOT):
    """(sym, sc) index arrays of the REs of unit u, in unit (symbol-major) order."""
    n_fb = n_sc // sc_per_h
    tb, fb = divmod(int(u), n_fb)
    s = np.repeat(np.arange(sym_per_h), sc_per_h) + tb * sym_per_h
    f = np.tile(np.arange(sc_per_h), sym_per_h) + fb * sc_per_h
    return s, f


@dataclasses.dataclass
class Workload:
    name: str
    n_rx: int
    n_layers: int
    qm: int
    n_sc: int
    n_slots: int
    sc_per_h: int
    llr: str
    sigma2: np.float32
    H: np.ndarray      # complex64 [n_slots][n_fb][nr][nl]
    y: np.ndarray      # complex64 [n_sym][n_sc][nr]
    bits: np.ndarray   # uint8 [n_sym][n_sc][nl][qm]
    seed: int
    sym_per_h: int = SYM_PER_SLOT  # symbols sharing one H (14 = one H per slot; NEXT-3: time-varying H)
    Rnn: np.ndarray | None = None  # complex64 [n_units][nr][nr] noise + interference covariance (IRC workloads)

    @property
    def n_sym(self) -> int:
        return self.n_slots * SYM_PER_SLOT

    @property
    def n_fb(self) -> int:
        return self.n_sc // self.sc_per_h

    @property
    def n_units(self) -> int:
        return (self.n_sym // self.sym_per_h) * self.n_fb

    @property
    def n_re(self) -> int:
        return self.n_sym * self.n_sc

    def H_units(self) -> np.ndarray:
        return self.H.reshape(self.n_units, self.n_rx, self.n_layers)

    def y_units(self) -> np.ndarray:
        return unit_gather(self.y, self.n_slots, self.n_sc, self.sc_per_h, self.sym_per_h)

    def sha256(self) -> str:
        h = hashlib.sha256()
        h.update(np.ascontiguousarray(self.H).tobytes())
        h.update(np.ascontiguousarray(self.y).tobytes())
        h.update(np.float32(self.sigma2).tobytes())
        return h.hexdigest()


def generate(cfg, *, n_sc: int | None = None, n_slots: int | None = None,
             seed: int | None = None, snr_db: float | None = None,
             sigma2: float | None = None, H_override: np.ndarray | None = None,
             noiseless: bool = False) -> Workload:
    """Draw one seeded workload.

    Recipe: Generator(PCG64(seed)), seed = 1000 + k by default;
    draws in fp64 in this order: (1) H_w for all units (slot-major, then
    frequency block), (2) bits for all REs in [n_sym][n_sc][nl][qm] order,
    (3) noise slot by slot (time block by time block when sym_per_h != 14) in
    [n_sym][n_sc][nr] order. Channel: iid CN(0, v),
    or Kronecker H = C_r H_w C_t^T with C = chol(rho^|i-j|). y = H x + n in fp64,
    then H and y are cast to complex64.
    """
    if isinstance(cfg, dict):
        c = dict(cfg)
        key = c.get("name", "custom")
    else:
        c = dict(CONFIGS[cfg])
        key = cfg
    if n_sc is not None:
        c["n_sc"] = n_sc
    if n_slots is not None:
        c["n_slots"] = n_slots
    if seed is None:
        seed = 1000 + (key if isinstance(key, int) else 0)
    nr, nl, qm, scph = c["n_rx"], c["n_layers"], c["qm"], c["sc_per_h"]
    sph = c.get("sym_per_h", SYM_PER_SLOT)  # NEXT-3: H constant over sph symbols (14 = per slot)
    nsc, nslots = c["n_sc"], c["n_slots"]
    if nsc % scph:
        raise ValueError("n_sc must be a multiple of sc_per_h")
    if (nslots * SYM_PER_SLOT) % sph:
        raise ValueError("n_sym must be a multiple of sym_per_h")
    s2 = sigma2_of(snr_db if snr_db is not None else c["snr_db"]) if sigma2 is None else np.float32(sigma2)
    rng = np.random.Generator(np.random.PCG64(seed))
    n_fb = nsc // scph
    n_sym = nslots * SYM_PER_SLOT
    n_tb = n_sym // sph
    n_units = n_tb * n_fb

    # (1) channel per H-unit
    Hw = _cn(rng, (n_units, nr, nl), 1.0)
    if H_override is not None:
        H = np.broadcast_to(np.asarray(H_override, dtype=np.complex128), (n_units, nr, nl)).copy()
    elif c["channel"] == "kron":
        cr = exp_corr_chol(nr, c["rho"])
        ct = exp_corr_chol(nl, c["rho"])
        H = np.sqrt(c["chan_var"]) * (cr @ Hw @ ct.T)
    else:
        H = np.sqrt(c["chan_var"]) * Hw
    H64 = H.astype(np.complex64)

    # (2) bits and symbols
    bits = rng.integers(0, 2, size=(n_sym, nsc, nl, qm), dtype=np.uint8)
    x = qam_modulate(bits, qm)  # [n_sym][n_sc][nl] complex128

    # (3) y = H x + n, fp64, per slot (bounded memory), then complex64.
    # The noiseless product uses the complex64-rounded H so that H is exactly
    # the channel the detector sees (noiseless pins compare against x exactly).
    Hq = H64.astype(np.complex128).reshape(n_tb, n_fb, nr, nl)
    y = np.empty((n_sym, nsc, nr), dtype=np.complex64)
    for t in range(n_tb):  # per time block of sph symbols (= per slot when sph = 14)
        xs = x[t * sph:(t + 1) * sph]                            # [sph][nsc][nl]
        xs = xs.reshape(sph, n_fb, scph, nl)
        ys = np.einsum("frl,sfcl->sfcr", Hq[t], xs, optimize=True)  # [sph][n_fb][scph][nr]
        ys = ys.reshape(sph, nsc, nr)
        if not noiseless:
            ys = ys + _cn(rng, (sph, nsc, nr), float(s2))
        y[t * sph:(t + 1) * sph] = ys.astype(np.complex64)

    return Workload(name=c.get("name", str(key)), n_rx=nr, n_layers=nl, qm=qm, n_sc=nsc,
                    n_slots=nslots, sc_per_h=scph, llr=c["llr"], sigma2=s2,
                    H=H64.reshape(n_tb, n_fb, nr, nl), y=y, bits=bits, seed=seed, sym_per_h=sph)


def generate_irc(cfg, *, n_interf: int = 2, inr_db: float = 10.0, **kw) -> Workload:
    """A workload with coloured interference for the interference-rejection detector (NEXT-3).

    Draws the white workload of generate(cfg, **kw), then with Generator(PCG64(seed + 1)):
    (4) per H-unit an interferer channel G_I ~ CN(0, sigma2 * 10^(INR/10)) of shape
    [nr][n_interf], (5) unit-power QPSK interferer symbols per RE; y += G_I x_I (fp64, then
    complex64). The receiver knows R_nn = G_I G_I^H + sigma2 I per unit (complex64)."""
    w = generate(cfg, **kw)
    rng = np.random.Generator(np.random.PCG64(w.seed + 1))
    nr, scph = w.n_rx, w.sc_per_h
    p_i = float(w.sigma2) * 10.0 ** (inr_db / 10.0)
    GI = _cn(rng, (w.n_units, nr, n_interf), p_i)
    xi = (rng.integers(0, 2, size=(w.n_sym, w.n_sc, n_interf, 2)) * 2 - 1) / np.sqrt(2.0)
    xi = xi[..., 0] + 1j * xi[..., 1]
    GI_grid = GI.reshape(w.n_slots, w.n_fb, nr, n_interf)
    y = w.y.astype(np.complex128)
    for t in range(w.n_slots):
        xs = xi[t * SYM_PER_SLOT:(t + 1) * SYM_PER_SLOT].reshape(SYM_PER_SLOT, w.n_fb, scph, n_interf)
        ys = np.einsum("fri,sfci->sfcr", GI_grid[t], xs, optimize=True).reshape(SYM_PER_SLOT, w.n_sc, nr)
        y[t * SYM_PER_SLOT:(t + 1) * SYM_PER_SLOT] += ys
    w.y = y.astype(np.complex64)
    R = GI @ np.conj(np.swapaxes(GI, 1, 2)) + float(w.sigma2) * np.eye(nr)[None]
    w.Rnn = R.astype(np.complex64)
    return w


def bfp_block_bytes(iq_width: int) -> int:
    """Bytes of one BFP block (reading R25): exponent byte + 24 W-bit mantissas, rounded up to 4."""
    return ((1 + 3 * iq_width) + 3) & ~3


def bfp_compress(y: np.ndarray, iq_width: int = 9, scale: float = 2.0 ** -8) -> np.ndarray:
    """RU-side block-floating-point compression of y (NEXT-4, reading R25).

    y complex64 [n_sym][n_sc][n_rx] (n_sc a multiple of 12) -> uint8
    [n_sym][n_sc/12][n_rx][bfp_block_bytes(W)]: per (symbol, PRB, antenna) the smallest
    exponent e in 0..15 with every |I|, |Q| / (scale 2^e) rounding into the W-bit range,
    mantissas round(v / (scale 2^e)) clipped to [-2^(W-1), 2^(W-1) - 1], packed MSB-first
    after the exponent byte. The detector only ever sees what this encodes."""
    W = int(iq_width)
    n_sym, n_sc, nr = y.shape
    n_prb = n_sc // 12
    v = y.reshape(n_sym, n_prb, 12, nr).transpose(0, 1, 3, 2)            # [sym][prb][r][f]
    iq = np.stack([v.real, v.imag], axis=-1).reshape(n_sym, n_prb, nr, 24).astype(np.float64)
    mmax = 2 ** (W - 1) - 1
    amax = np.max(np.abs(iq), axis=-1) / scale                          # [sym][prb][r]
    e = np.zeros(amax.shape, np.int64)
    for _ in range(16):                                                  # smallest e that fits
        over = np.rint(amax / (2.0 ** e)) > mmax
        e = np.where(over & (e < 15), e + 1, e)
    m = np.clip(np.rint(iq / (scale * (2.0 ** e))[..., None]), -mmax - 1, mmax).astype(np.int64)
    bits = ((m[..., None] & (1 << np.arange(W - 1, -1, -1))) != 0).astype(np.uint8)  # MSB-first
    stream = bits.reshape(n_sym, n_prb, nr, 24 * W)
    pad = 8 * (bfp_block_bytes(W) - 1) - 24 * W
    stream = np.concatenate([stream, np.zeros(stream.shape[:-1] + (pad,), np.uint8)], axis=-1)
    payload = np.packbits(stream, axis=-1, bitorder="big")
    return np.concatenate([e.astype(np.uint8)[..., None], payload], axis=-1)


def config_algorithmic_bytes(cfg_key, llr_bytes: int | None = None, n_sc: int | None = None,
                             n_slots: int | None = None) -> dict:
    """Algorithmic bytes of one full pass (H read once, y read once, LLRs written once), SURVEY.md §8(d).
    n_sc / n_slots override the config's grid (a multi-GPU shard)."""
    c = dict(CONFIGS[cfg_key])
    if n_sc is not None:
        c["n_sc"] = n_sc
    if n_slots is not None:
        c["n_slots"] = n_slots
    nr, nl, qm, scph = c["n_rx"], c["n_layers"], c["qm"], c["sc_per_h"]
    n_sym = c["n_slots"] * SYM_PER_SLOT
    n_re = n_sym * c["n_sc"]
    n_units = c["n_slots"] * (c["n_sc"] // scph)
    lb = llr_bytes if llr_bytes is not None else {"f32": 4, "f16": 2, "i8": 1}[c["llr"]]
    h = n_units * nr * nl * 8
    yb = n_re * nr * 8
    lo = n_re * nl * qm * lb
    return dict(H=h, y=yb, llr=lo, total=h + yb + lo, n_re=n_re, n_units=n_units,
                n_llr=n_re * nl * qm)


def config_algorithmic_flops(cfg_key, n_sc: int | None = None, n_slots: int | None = None) -> dict:
    """Algorithmic flops of one full pass (SURVEY.md §8(d) counting convention).

    Setup per H-unit (rows a2-a5), in complex MACs (8 real flops each):
      Gram nr*nl(nl+1)/2 + Cholesky nl^3/6 + L^-1 nl^3/6 + W nl^2*nr;
    per RE: x~ = W~ y, nl*nr cMAC (row a6), and ~8 flops per LLR bit (row a7).
    """
    c = dict(CONFIGS[cfg_key])
    if n_sc is not None:
        c["n_sc"] = n_sc
    if n_slots is not None:
        c["n_slots"] = n_slots
    nr, nl, qm, scph = c["n_rx"], c["n_layers"], c["qm"], c["sc_per_h"]
    n_sym = c["n_slots"] * SYM_PER_SLOT
    n_re = n_sym * c["n_sc"]
    n_units = c["n_slots"] * (c["n_sc"] // scph)
    unit_cmac = nr * nl * (nl + 1) / 2 + nl ** 3 / 3 + nl * nl * nr
    setup = 8.0 * unit_cmac * n_units
    apply = 8.0 * nl * nr * n_re
    demap = 8.0 * nl * qm * n_re
    return dict(setup=setup, apply=apply, demap=demap, total=setup + apply + demap)
