"""Localise tensor-core path errors: x~ of a forced kernel vs the SIMT kernel, per RE row / layer."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2510_07843_b200 import mimo, synth

kern = sys.argv[1]
w = synth.generate(5, n_sc=120, n_slots=1)
H, y = torch.from_numpy(w.H).cuda(), torch.from_numpy(w.y).cuda()
res = {}
for name in ("big_64x16_q6_i8", kern):
    os.environ["MIMO_FORCE_KERNEL"] = name
    p = mimo.Plan(64, 16, 6, sc_per_h=12, llr_dtype="i8")
    x = torch.empty((14, 120, 16), dtype=torch.complex64, device="cuda")
    p.detect(H, y, float(w.sigma2), xhat=x)
    torch.cuda.synchronize()
    res[name] = x.cpu().numpy()
    print(name, p.kernel_name)
d = np.abs(res[kern] - res["big_64x16_q6_i8"])            # [sym][sc][layer]
print("max err", d.max())
ds = d.reshape(14, 10, 12, 16)                            # sym, prb, f, layer
print("by symbol :", np.round(ds.max(axis=(1, 2, 3)), 4))
print("by f      :", np.round(ds.max(axis=(0, 1, 3)), 4))
print("by layer  :", np.round(ds.max(axis=(0, 1, 2)), 4))
print("by prb    :", np.round(ds.max(axis=(0, 2, 3)), 4))
