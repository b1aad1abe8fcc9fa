#!/usr/bin/env python
"""Fig. 5a analogue: detection accuracy of the GPU
detector in fp32 ("PS") against fp64 ("PD") over SNR, at 2x2, 4x4 and 8x8
(PAPER.md:104-110 Fig. 5a, :117 "single precision ... comparable accuracy",
:119). TDL-C and LDPC are not in the container, so the channel is i.i.d.
CN(0,1) per subcarrier (synth recipe) and the metrics are uncoded:

  BER(hard)  hard decisions of the LLRs (LLR < 0 -> 1) against the sent bits
  EVM        rms |x~ - x| / rms |x| of the unbiased equalised symbols
  dBER       fraction of bits whose hard decision differs from the fp64 oracle's

Routes: the fused Gram/Cholesky production kernel (fp32 apply; per-unit setup in
the kernel's precision), the paper-literal covariance/LU route in PS (fp32) and
PD (fp64), and the fp64 oracle (Gram/Cholesky route) on the same inputs.

    python tests/accuracy_study.py [--n-sc 1200] [--slots 2] [--out profiles/r01/accuracy_sweep]

It lives under tests/ because it runs the fp64 oracle (test infrastructure);
tests/test_accuracy_gpu.py runs a reduced sweep and asserts the paper's claim.
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402  (test infrastructure: the fp64 reference of this study)
from paper_2510_07843_b200 import mimo, synth  # noqa: E402


def metrics(w, llr_grid, xhat_grid):
    bits_hat = (llr_grid < 0).astype(np.uint8)
    ber = float((bits_hat != w.bits).mean())
    x = synth.qam_modulate(w.bits, w.qm)
    evm = float(np.sqrt(np.mean(np.abs(xhat_grid - x) ** 2) / np.mean(np.abs(x) ** 2)))
    return ber, evm, bits_hat


def sweep(n_sc=1200, slots=2, qm=4, sizes=(2, 4, 8), snrs=(0, 5, 10, 15, 20, 25, 30), verbose=True):
    """One row per (MIMO size, SNR): BER / EVM of each GPU route and of the fp64 oracle."""
    args = argparse.Namespace(n_sc=n_sc, slots=slots, qm=qm)
    rows = []
    for n in sizes:
        for snr in snrs:
            cfg = dict(name=f"{n}x{n}", n_rx=n, n_layers=n, qm=args.qm, n_sc=args.n_sc, n_slots=args.slots,
                       sc_per_h=1, channel="iid", chan_var=1.0, snr_db=float(snr), llr="f32")
            w = synth.generate(cfg, seed=7000 + 100 * n + snr)
            H = torch.from_numpy(w.H).cuda()
            y = torch.from_numpy(w.y).cuda()
            p = mimo.Plan(n, n, args.qm)
            sh = p.shapes(w.n_sc, w.n_sym)
            res = {}
            for route in ("fused", "lu_ps", "lu_pd"):
                xh = torch.empty(sh["xhat"], dtype=torch.complex64, device="cuda")
                if route == "fused":
                    out = p.detect(H, y, float(w.sigma2), xhat=xh)
                else:
                    out = p.detect_lu(H, y, float(w.sigma2), precision=32 if route == "lu_ps" else 64, xhat=xh)
                nf = p.sync_status()
                res[route] = (out.cpu().numpy(), xh.cpu().numpy().astype(np.complex128), nf)
            name = p.kernel_name
            p.close()
            ref = oracle.detect(w.H_units(), w.y_units(), w.sigma2, w.qm, threads=oracle.max_threads())
            # oracle outputs are in unit order; scatter back to the [sym][sc] grid
            llr_o = np.zeros((w.n_sym, w.n_sc, n, args.qm))
            x_o = np.zeros((w.n_sym, w.n_sc, n), np.complex128)
            for u in range(w.n_units):
                s_idx, f_idx = synth.unit_re_index(u, w.n_sc, w.sc_per_h)
                llr_o[s_idx, f_idx] = ref["llr"][u]
                x_o[s_idx, f_idx] = ref["xhat"][u]
            ber_o, evm_o, bits_o = metrics(w, llr_o, x_o)
            row = dict(mimo=f"{n}x{n}", snr_db=snr, n_bits=int(w.bits.size), oracle_fp64=dict(ber=ber_o, evm=evm_o),
                       fused_kernel=name)
            for route, (llr, xh, nf) in res.items():
                ber, evm, bh = metrics(w, llr, xh)
                row[route] = dict(ber=ber, evm=evm, dber_vs_oracle=float((bh != bits_o).mean()),
                                  max_dx_vs_oracle=float(np.max(np.abs(xh - x_o))), n_failed=nf)
            rows.append(row)
            if verbose:
                print(json.dumps(row), flush=True)
    return rows


def write_report(rows, out, n_sc, slots, qm):
    args = argparse.Namespace(n_sc=n_sc, slots=slots, qm=qm, out=out)
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out + ".json", "w") as f:
        json.dump(rows, f, indent=1)
    lines = [f"Uncoded {2 ** args.qm}-QAM, i.i.d. CN(0,1), {args.n_sc} sc x {14 * args.slots} sym per point "
             f"({rows[0]['n_bits']} bits per 2x2 point)", "",
             "| MIMO | SNR dB | BER fp64 oracle | BER fused fp32 | BER LU PS | BER LU PD | EVM oracle | EVM LU PS | "
             "EVM LU PD | bit flips PS vs oracle | bit flips PD vs oracle | max abs dx PS | max abs dx PD |",
             "|---|---|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        lines.append(f"| {r['mimo']} | {r['snr_db']} | {r['oracle_fp64']['ber']:.3e} | {r['fused']['ber']:.3e} | "
                     f"{r['lu_ps']['ber']:.3e} | {r['lu_pd']['ber']:.3e} | {r['oracle_fp64']['evm']:.4f} | "
                     f"{r['lu_ps']['evm']:.4f} | {r['lu_pd']['evm']:.4f} | {r['lu_ps']['dber_vs_oracle']:.2e} | "
                     f"{r['lu_pd']['dber_vs_oracle']:.2e} | {r['lu_ps']['max_dx_vs_oracle']:.1e} | "
                     f"{r['lu_pd']['max_dx_vs_oracle']:.1e} |")
    with open(args.out + ".md", "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-sc", type=int, default=1200)
    ap.add_argument("--slots", type=int, default=2)
    ap.add_argument("--qm", type=int, default=4)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01", "accuracy_sweep"))
    a = ap.parse_args()
    rows = sweep(a.n_sc, a.slots, a.qm)
    write_report(rows, a.out, a.n_sc, a.slots, a.qm)


if __name__ == "__main__":
    main()
