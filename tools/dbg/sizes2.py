import sys, time, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import parity
from paper_2510_07843_b200 import synth
kn, n_my = sys.argv[1], int(sys.argv[2])
prb = 37 * n_my  # 148 CTAs: 4 slots x 37 n_my PRBs = 148 n_my units
w = synth.generate(5, n_sc=12 * prb, n_slots=4)
g = parity.run_gpu(w, kernel=kn, xhat=False)
print(n_my, w.n_units, "failed", g["n_failed"], parity.compare(w, g, [0, w.n_units - 1]), flush=True)
