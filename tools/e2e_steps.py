"""e2e async host path (C2): steps per measurement, shared vs per-step output buffers."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_07843_b200 import mimo, synth

w = synth.generate(2)
plan = mimo.Plan(w.n_rx, w.n_layers, w.qm, sc_per_h=w.sc_per_h, llr_dtype=w.llr)
H, y = torch.from_numpy(w.H).pin_memory(), torch.from_numpy(w.y).pin_memory()
shape = plan.shapes(w.n_sc, w.n_sym)["llr"]
outs = [torch.empty(shape, dtype=plan.llr_dtype).pin_memory() for _ in range(4)]
n_re = w.n_sym * w.n_sc
for steps in (10, 20, 60):
    for nb in (1, 4):
        for _ in range(3):
            plan.detect_host(H, y, float(w.sigma2), out=outs[0], wait=False)
        plan.sync_status()
        t0 = time.perf_counter()
        for i in range(steps):
            plan.detect_host(H, y, float(w.sigma2), out=outs[i % nb], wait=False)
        plan.sync_status()
        dt = (time.perf_counter() - t0) / steps
        print(f"steps {steps:3d} out buffers {nb}: {dt * 1e3:.3f} ms/step {n_re / dt:.3e} RE/s", flush=True)
