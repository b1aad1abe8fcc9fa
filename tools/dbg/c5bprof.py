import ctypes, os, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2510_07843_b200 import mimo, synth
L = mimo.load_library(os.environ.get('PROFLIB', 'tools/dbg/libmimo_prof.so'))
w = synth.generate(5)
H, y = torch.from_numpy(w.H).cuda(), torch.from_numpy(w.y).cuda()
names = {0: "tma wait", 1: "convert", 2: "gram mma", 3: "gram readout", 4: "GJ + B'", 5: "W mma", 6: "W readout+store", 7: "fence+sync", 8: " GJ: pdl", 9: " GJ: ring_wait", 10: " GJ: C load + pivots", 11: " GJ: A, B', slopes", 12: " GJ: sync"}
p = mimo.Plan(64, 16, 6, sc_per_h=12, llr_dtype="i8", kernel=sys.argv[1])
out = torch.empty(p.shapes(w.n_sc, w.n_sym)["llr"], dtype=torch.int8, device="cuda")
p.detect(H, y, float(w.sigma2), out=out); torch.cuda.synchronize()
b0 = np.zeros(148 * 32, np.uint64); L.mimo_c5_sprof_read(ctypes.c_void_p(b0.ctypes.data))
n = 5
for _ in range(n): p.detect(H, y, float(w.sigma2), out=out)
torch.cuda.synchronize()
b1 = np.zeros(148 * 32, np.uint64); L.mimo_c5_sprof_read(ctypes.c_void_p(b1.ctypes.data))
b = (b1 - b0).reshape(148, 32).astype(np.float64)
nb = (w.n_units + 3) // 4 / 444 * 3 if 'fused' not in sys.argv[1] else w.n_units / 148 / 4  # batches per SM
for s_, nm in names.items(): print(f"  {nm:18s} {b[:, s_].mean() / (n * nb):8.0f} cycles/batch (per CTA)")
