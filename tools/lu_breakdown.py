#!/usr/bin/env python
"""Fig. 5b analogue on B200: per-stage device time of the
paper-literal LMMSE pipeline (mimo_detect_lmmse_lu: covariance, LU, substitution
inversion, weights, apply+demap) at 2x2, 4x4
and 8x8, in fp32 ("PS") and fp64 ("PD"), next to the fused Gram/Cholesky
production kernel on the same inputs.

Shapes: the paper's own TTI (60 RB x 12 = 720 subcarriers, 14 symbols, one slot;
PAPER.md:117) detected alone (latency: every stage is a few microseconds of
launch + ramp), the same TTI shape batched 100 TTIs per call (per-TTI cost in
a stream of TTIs -- the figure comparable with the paper's per-TTI average over
10,000 TTIs), and a 100 MHz / 30 kHz batch (3276 subcarriers x 10 slots).
16-QAM (reading: MCS 9 -> Qm 4), i.i.d. CN(0,1) channel per subcarrier, SNR 15
dB, fp32 LLRs. The fused production kernel is timed as the mean of 20
back-to-back calls between two events (so host launch overhead is hidden).

    python tools/lu_breakdown.py [--reps 50] [--out profiles/r01/lu_breakdown]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2510_07843_b200 import mimo, synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=50)
    ap.add_argument("--out", default=os.path.join(ROOT, "profiles", "r01", "lu_breakdown"))
    args = ap.parse_args()
    rows = []
    for n_sc, n_slots, shape in ((720, 1, "1 TTI (720 sc x 14 sym)"), (720, 100, "100 TTIs of 720 sc x 14 sym"),
                                 (3276, 10, "3276 sc x 14 sym x 10 slots")):
        for n in (2, 4, 8):
            cfg = dict(name=f"{n}x{n}", n_rx=n, n_layers=n, qm=4, n_sc=n_sc, n_slots=n_slots, sc_per_h=1,
                       channel="iid", chan_var=1.0, snr_db=15.0, llr="f32")
            w = synth.generate(cfg, seed=500 + n)
            H = torch.from_numpy(w.H).cuda()
            y = torch.from_numpy(w.y).cuda()
            p = mimo.Plan(n, n, 4)
            out = torch.empty(p.shapes(w.n_sc, w.n_sym)["llr"], dtype=torch.float32, device="cuda")
            for prec in (32, 64):
                samples = {s: [] for s in mimo.LU_STAGES}
                for r in range(args.reps + 3):
                    _, st = p.detect_lu(H, y, float(w.sigma2), precision=prec, out=out, timing=True)
                    if r >= 3:
                        for s, v in st.items():
                            samples[s].append(v)
                assert p.sync_status() == 0
                med = {s: statistics.median(v) for s, v in samples.items()}
                tot = sum(med.values())
                rows.append(dict(shape=shape, mimo=f"{n}x{n}", precision="PS fp32" if prec == 32 else "PD fp64",
                                 stages_us=med, total_us=tot, n_re=w.n_re, n_tti=n_slots,
                                 share={s: med[s] / tot for s in med}))
            # fused production kernel on the same inputs (single serialised call, events)
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ts = []
            for r in range(args.reps + 3):
                ev0.record()
                for _ in range(20):
                    p.detect(H, y, float(w.sigma2), out=out)
                ev1.record()
                torch.cuda.synchronize()
                if r >= 3:
                    ts.append(ev0.elapsed_time(ev1) * 1e3 / 20)
            rows.append(dict(shape=shape, mimo=f"{n}x{n}", precision=f"fused {p.kernel_name}",
                             stages_us=None, total_us=statistics.median(ts), n_re=w.n_re, n_tti=n_slots, share=None))
            p.close()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    with open(args.out + ".json", "w") as f:
        json.dump(rows, f, indent=1)
    lines = ["| shape | MIMO | route | cov | LU | inv | weights | apply+demap | total (us) | per TTI (us) | "
             "inversion share (LU+inv) |", "|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in rows:
        if r["stages_us"]:
            s = r["stages_us"]
            lines.append(f"| {r['shape']} | {r['mimo']} | {r['precision']} | " +
                         " | ".join(f"{s[k]:.1f}" for k in mimo.LU_STAGES) +
                         f" | {r['total_us']:.1f} | {r['total_us'] / r['n_tti']:.2f} | "
                         f"{r['share']['lu'] + r['share']['inv']:.0%} |")
        else:
            lines.append(f"| {r['shape']} | {r['mimo']} | {r['precision']} | | | | | | {r['total_us']:.1f} | "
                         f"{r['total_us'] / r['n_tti']:.2f} | |")
    with open(args.out + ".md", "w") as f:
        f.write("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    main()
