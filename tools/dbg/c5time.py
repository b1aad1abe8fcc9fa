"""Tuning: time the C5 default kernel of a tuning library (PROFLIB), 3 rotating buffer sets, 30 calls."""
import os, sys, torch
sys.path.insert(0, '.')
from paper_2510_07843_b200 import mimo, synth
mimo.load_library(os.environ['PROFLIB'])
w = synth.generate(5)
p = mimo.Plan(64, 16, 6, sc_per_h=12, llr_dtype="i8", kernel=(sys.argv[1] if len(sys.argv) > 1 else None))
sets = [(torch.from_numpy(w.H).cuda(), torch.from_numpy(w.y).cuda(),
         torch.empty(p.shapes(w.n_sc, w.n_sym)["llr"], dtype=torch.int8, device="cuda")) for _ in range(2)]
for H, y, o in sets * 3:
    p.detect(H, y, float(w.sigma2), out=o)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 30
e0.record()
for i in range(n):
    H, y, o = sets[i % 2]
    p.detect(H, y, float(w.sigma2), out=o)
e1.record()
torch.cuda.synchronize()
print(os.environ['PROFLIB'], p.kernel_name, f"{e0.elapsed_time(e1) / n * 1e3:.1f} us/call")
