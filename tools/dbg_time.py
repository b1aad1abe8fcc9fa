"""Time one forced kernel on a BASELINE config: single calls, then back-to-back (PDL overlap) calls."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_07843_b200 import mimo, synth

kern, cfg = sys.argv[1], int(sys.argv[2])
n_slots = int(sys.argv[3]) if len(sys.argv) > 3 else None
overlap = int(sys.argv[4]) if len(sys.argv) > 4 else 1
os.environ["MIMO_FORCE_KERNEL"] = kern
w = synth.generate(cfg, **({"n_slots": n_slots} if n_slots else {}))
H, y = torch.from_numpy(w.H).cuda(), torch.from_numpy(w.y).cuda()
p = mimo.Plan(w.n_rx, w.n_layers, w.qm, sc_per_h=w.sc_per_h, llr_dtype=w.llr, overlap_calls=bool(overlap))
out = p.detect(H, y, float(w.sigma2))
torch.cuda.synchronize()
print(kern, p.kernel_name, "first call ok", flush=True)
for n in (1, 10, 100):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        p.detect(H, y, float(w.sigma2), out=out)
    e1.record()
    torch.cuda.synchronize()
    print(n, "calls", round(e0.elapsed_time(e1) * 1000 / n, 1), "us/call", flush=True)
