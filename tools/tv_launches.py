"""One C5-grid call per sym_per_h (7, 2, 1) on the 64x16 time-varying kernels, for an ncu launch
list (setup vs apply share): ncu --metrics gpu__time_duration.sum -k regex:k_big python tools/tv_launches.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2510_07843_b200 import mimo, synth  # noqa: E402

for sph in (7, 2, 1):
    w = synth.generate(dict(synth.CONFIGS[5], sym_per_h=sph))
    plan = mimo.Plan(w.n_rx, w.n_layers, w.qm, sc_per_h=w.sc_per_h, sym_per_h=sph, llr_dtype=w.llr)
    H, y = torch.from_numpy(w.H).cuda(), torch.from_numpy(w.y).cuda()
    out = torch.empty(plan.shapes(w.n_sc, w.n_sym)["llr"], dtype=plan.llr_dtype, device="cuda")
    for _ in range(2):
        plan.detect(H, y, float(w.sigma2), out=out)
    torch.cuda.synchronize()
    assert plan.sync_status() == 0
    print(sph, plan.kernel_name, w.n_units)
    plan.close()
