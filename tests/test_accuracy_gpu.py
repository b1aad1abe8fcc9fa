"""Reduced Fig. 5a analogue (tests/accuracy_study.py):
fp32 ("PS") detection is as accurate as fp64 ("PD") -- PAPER.md:117, :119 --
measured as uncoded BER / EVM on seeded i.i.d. channels, plus sanity: BER falls
with SNR and the PD LU route reproduces the fp64 oracle's hard decisions."""
import pytest

import accuracy_study

pytestmark = pytest.mark.gpu


def test_ps_matches_pd_accuracy():
    rows = accuracy_study.sweep(n_sc=600, slots=1, sizes=(2, 4, 8), snrs=(5, 15, 25), verbose=False)
    for n in ("2x2", "4x4", "8x8"):
        rs = [r for r in rows if r["mimo"] == n]
        bers = [r["oracle_fp64"]["ber"] for r in rs]
        assert bers[0] > bers[-1], (n, bers)                      # BER falls with SNR
        for r in rs:
            assert r["lu_pd"]["dber_vs_oracle"] <= 1e-4, r         # PD == fp64 reference
            assert r["fused"]["dber_vs_oracle"] <= 1e-4, r         # production kernel
            # PS: "comparable accuracy" -- BER within 2% relative (+ 1e-4 absolute)
            assert abs(r["lu_ps"]["ber"] - r["oracle_fp64"]["ber"]) <= 0.02 * r["oracle_fp64"]["ber"] + 1e-4, r
            assert abs(r["lu_ps"]["evm"] - r["oracle_fp64"]["evm"]) <= 1e-3 * r["oracle_fp64"]["evm"] + 1e-5, r
