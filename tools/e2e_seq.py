"""Reproduce bench.py's e2e sequence: sync calls, then a stream of async calls (C2)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_07843_b200 import mimo, synth

w = synth.generate(2)
plan = mimo.Plan(w.n_rx, w.n_layers, w.qm, sc_per_h=w.sc_per_h, llr_dtype=w.llr, overlap_calls=True)
H, y = torch.from_numpy(w.H).pin_memory(), torch.from_numpy(w.y).pin_memory()
lh = torch.empty(plan.shapes(w.n_sc, w.n_sym)["llr"], dtype=plan.llr_dtype).pin_memory()
n_re = w.n_sym * w.n_sc
def run(n, wait):
    t0 = time.perf_counter()
    for _ in range(n):
        plan.detect_host(H, y, float(w.sigma2), out=lh, wait=wait)
    plan.sync_status()
    return (time.perf_counter() - t0) / n * 1e3
print("async first", run(20, False))
print("sync", run(60, True))
print("async after sync", run(60, False))
print("async again", run(60, False))
print("sync again", run(20, True))
print("async again", run(60, False))
