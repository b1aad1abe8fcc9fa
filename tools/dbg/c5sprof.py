"""Per-role cycle accounting of the C5 setup kernel (tuning build)."""
import ctypes, os, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2510_07843_b200 import mimo, synth
L = mimo.load_library(os.environ.get('PROFLIB', 'tools/dbg/libmimo_prof.so'))
w = synth.generate(5)
H, y = torch.from_numpy(w.H).cuda(), torch.from_numpy(w.y).cuda()
names = {0: "quad.wait_wdone", 2: "quad.wait_gdone", 10: "worker.wait_hfull", 8: "worker.wait_cready",
         9: "worker.gj+B'", 16: "mma.wait_xready+tfree", 17: "mma.wait_bready", 20: "prod.wait_wdone", 31: "mma.total"}
for kn in sys.argv[1:]:
    p = mimo.Plan(64, 16, 6, sc_per_h=12, llr_dtype="i8", kernel=kn)
    out = torch.empty(p.shapes(w.n_sc, w.n_sym)["llr"], dtype=torch.int8, device="cuda")
    for _ in range(2):
        p.detect(H, y, float(w.sigma2), out=out)
    torch.cuda.synchronize()
    buf0 = np.zeros(148 * 32, np.uint64)
    L.mimo_c5_sprof_read(ctypes.c_void_p(buf0.ctypes.data))
    n = 5
    for _ in range(n):
        p.detect(H, y, float(w.sigma2), out=out)
    torch.cuda.synchronize()
    buf = np.zeros(148 * 32, np.uint64)
    L.mimo_c5_sprof_read(ctypes.c_void_p(buf.ctypes.data))
    b = (buf - buf0).reshape(148, 32).astype(np.float64)
    upc = w.n_units / 148.0
    print(kn)
    for s, nm in sorted(names.items()):
        div = n * upc / (12 if s in (8, 9, 10) else 1)
        print(f"   {nm:26s} {b[:, s].mean() / div:9.0f} cycles/unit" + (" (per worker unit)" if s in (8, 9, 10) else ""))
