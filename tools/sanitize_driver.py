"""One small call of every kernel family (all C-ABI routes), for memory-checker runs.

    compute-sanitizer --tool memcheck python tools/sanitize_driver.py
(compute-sanitizer is closed on this round's GPU pool -- DESIGN.md §4 -- so the
driver is used as a plain all-families smoke run.) Exits non-zero if any call
raises; prints the kernel used per case."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_07843_b200 import mimo, synth  # noqa: E402

CASES = [  # (config, generate kwargs, forced kernel or None)
    (1, {}, None),
    (2, dict(n_sc=100, n_slots=1), None),
    (3, dict(n_sc=48, n_slots=1), None),
    (4, dict(n_sc=40, n_slots=1), None),
    (5, dict(n_sc=24, n_slots=1), None),
    (5, dict(n_sc=24, n_slots=1), "c5_bf16_tcs_be_64x16_q6_i8"),
    (5, dict(n_sc=24, n_slots=1), "big_64x16_q6_i8"),
    (2, dict(n_sc=36, n_slots=1), "generic"),
]


def run(k, kw, force):
    w = synth.generate(k, **kw)
    p = mimo.Plan(w.n_rx, w.n_layers, w.qm, sc_per_h=w.sc_per_h, llr_dtype=w.llr, kernel=force)
    H, y = torch.from_numpy(w.H).cuda(), torch.from_numpy(w.y).cuda()
    sh = p.shapes(w.n_sc, w.n_sym)
    x = torch.empty(sh["xhat"], dtype=torch.complex64, device="cuda")
    s = torch.empty(sh["sinr"], dtype=torch.float32, device="cuda")
    p.detect(H, y, float(w.sigma2), xhat=x, sinr=s)
    assert p.sync_status() == 0
    print(f"C{k} {p.kernel_name}: ok", flush=True)
    return p, w, H, y


def main():
    for k, kw, force in CASES:
        run(k, kw, force)
    p, w, H, y = run(2, dict(n_sc=36, n_slots=1), None)
    for prec in (32, 64):
        p.detect_lu(H, y, float(w.sigma2), precision=prec)
    assert p.sync_status() == 0
    print("LU route: ok", flush=True)
    wi = synth.generate_irc(3, n_sc=24, n_slots=1)
    pi = mimo.Plan(wi.n_rx, wi.n_layers, wi.qm, sc_per_h=wi.sc_per_h, llr_dtype=wi.llr)
    pi.detect_irc(torch.from_numpy(wi.H).cuda(), torch.from_numpy(wi.y).cuda(), torch.from_numpy(wi.Rnn).cuda())
    assert pi.sync_status() == 0
    print("IRC route: ok", flush=True)
    torch.cuda.synchronize()


if __name__ == "__main__":
    main()
