import sys, time, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import parity
from paper_2510_07843_b200 import synth, mimo
kn = sys.argv[1]
for n_slots, n_sc in ((1, 96), (1, 3276), (4, 3276), (8, 3276)):
    w = synth.generate(5, n_sc=n_sc, n_slots=n_slots)
    t = time.time()
    g = parity.run_gpu(w, kernel=kn, xhat=False)
    units = [0, w.n_units // 2, w.n_units - 1]
    print(n_slots, n_sc, w.n_units, "failed", g["n_failed"], parity.compare(w, g, units), f"{time.time() - t:.1f}s", flush=True)
