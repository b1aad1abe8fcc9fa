"""Pins of the block-floating-point fronthaul decoder (SURVEY.md §8(f) NEXT-4,
reading R25) in the oracle: a hand-derived golden block, exponent minimality and
the half-LSB round-trip bound of the RU-side compressor (synth.bfp_compress)."""
import json
import os

import numpy as np
import pytest

import oracle
from paper_2510_07843_b200 import synth

GOLD = os.path.join(os.path.dirname(__file__), "golden", "bfp_block.json")


def test_golden_block():
    g = json.load(open(GOLD))
    blk = np.frombuffer(bytes.fromhex(g["block_hex"]), np.uint8)
    assert blk.size == synth.bfp_block_bytes(g["iq_width"])
    out = oracle.bfp_decode(blk[None], g["iq_width"], g["scale"])[0]
    exp = np.array([complex(a, b) for a, b in g["expected"]], np.complex64)
    assert np.array_equal(out, exp)


@pytest.mark.parametrize("W", [8, 9, 12, 16])
def test_round_trip_half_lsb(W):
    w = synth.generate(3, n_sc=48, n_slots=1)
    scale = 2.0 ** -8
    b = synth.bfp_compress(w.y, W, scale)
    assert b.shape == (w.n_sym, w.n_sc // 12, w.n_rx, synth.bfp_block_bytes(W))
    d = oracle.bfp_decode(b, W, scale)                           # [sym][prb][r][f]
    yd = d.transpose(0, 1, 3, 2).reshape(w.y.shape)
    e = b[..., 0].astype(np.int64)                               # [sym][prb][r]
    lsb = np.repeat((scale * 2.0 ** e).transpose(0, 1, 2)[:, :, None, :], 12, axis=2).reshape(w.y.shape)
    assert np.all(np.abs(yd.real - w.y.real) <= 0.5 * lsb + 1e-12)
    assert np.all(np.abs(yd.imag - w.y.imag) <= 0.5 * lsb + 1e-12)
    # exponent minimality: with e - 1 some value of the block would not fit in W bits
    iq = np.stack([w.y.real, w.y.imag], -1).reshape(w.n_sym, w.n_sc // 12, 12, w.n_rx, 2)
    amax = np.abs(iq).max(axis=(2, 4))                           # [sym][prb][r]
    pos = e > 0
    assert np.all(np.rint(amax[pos] / (scale * 2.0 ** (e[pos] - 1))) > 2 ** (W - 1) - 1)
