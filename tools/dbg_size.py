"""Run one forced C5 kernel at a given size and compare its LLRs with the default SIMT kernel."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2510_07843_b200 import mimo, synth

kern, n_sc, n_slots = sys.argv[1], int(sys.argv[2]), int(sys.argv[3])
REF = sys.argv[4] if len(sys.argv) > 4 else "big_64x16_q6_i8"
w = synth.generate(5, n_sc=n_sc, n_slots=n_slots)
H, y = torch.from_numpy(w.H).cuda(), torch.from_numpy(w.y).cuda()
res = {}
for name in (REF, kern):
    os.environ["MIMO_FORCE_KERNEL"] = name
    p = mimo.Plan(64, 16, 6, sc_per_h=12, llr_dtype="i8")
    out = p.detect(H, y, float(w.sigma2))
    print(name, p.kernel_name, "failed units", p.sync_status(), flush=True)
    res[name] = out.cpu().numpy()
d = np.abs(res[kern].astype(int) - res[REF].astype(int))
print(n_sc, n_slots, "max llr diff", d.max(), "n diff", (d > 0).sum())
