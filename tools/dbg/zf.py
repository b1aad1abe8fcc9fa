import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import parity
from paper_2510_07843_b200 import synth
for s2 in (0.0, 1e-30, 1e-6, 0.01):
    w = synth.generate(5, n_sc=48, n_slots=1, sigma2=s2)
    for kn in ("c5_bf16_tcs_64x16_q6_i8", "c5_bf16_64x16_q6_i8"):
        g = parity.run_gpu(w, kernel=kn)
        print(s2, kn, g["n_failed"], g["sinr"][:, :3].tolist(), float(np.abs(g["xhat"]).max()))
