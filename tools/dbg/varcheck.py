"""Tuning check: parity of one tuning-build library (PROFLIB) on C5 against the oracle, sampled units,
plus timing of the default kernel (tools/dbg only; never used by the product)."""
import os, sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
from paper_2510_07843_b200 import mimo, synth
mimo.load_library(os.environ['PROFLIB'])
import parity
w = synth.generate(5)
g = parity.run_gpu(w, kernel=sys.argv[1] if len(sys.argv) > 1 else None)
rng = np.random.default_rng(3)
units = rng.choice(w.n_units, 48, replace=False)
r = parity.compare(w, g, units=units)
print(os.environ['PROFLIB'], g['kernel'], {k: v for k, v in r.items() if not isinstance(v, np.ndarray)})
