"""Per-role cycle accounting of the C5 apply kernel (tuning build, tools/dbg/build_prof.sh)."""
import ctypes, sys, numpy as np, torch
sys.path.insert(0, '.')
from paper_2510_07843_b200 import mimo, synth
import os
L = mimo.load_library(os.environ.get('PROFLIB', 'tools/dbg/libmimo_prof.so'))
L.mimo_c5_prof_read.argtypes = [ctypes.c_void_p]
w = synth.generate(5)
H, y = torch.from_numpy(w.H).cuda(), torch.from_numpy(w.y).cuda()
names = {0: "prod.wait_yfree", 1: "prod.wait_setup(fused)", 31: "prod.total", 8: "mma.wait_bready", 9: "mma.wait_tfree", 10: "mma.wait_afull",
         16: "conv.wait_accfull(B)", 17: "conv.Bbuild", 18: "conv.wait_yfull", 19: "conv.wait_afree",
         20: "conv.convert", 21: "conv.bar+arrive", 24: "epi.wait_accfull", 25: "epi.work", 26: "epi.bar", 27: "epi.Bbuild", 28: "epi.Bbuild.wfull", 29: "epi.Bbuild.issue_w(spin)", 30: "epi.BI first issue (startup)"}
for kn in sys.argv[1:]:
    p = mimo.Plan(64, 16, 6, sc_per_h=12, llr_dtype="i8", kernel=kn)
    out = torch.empty(p.shapes(w.n_sc, w.n_sym)["llr"], dtype=torch.int8, device="cuda")
    for _ in range(3):
        p.detect(H, y, float(w.sigma2), out=out)
    torch.cuda.synchronize()
    L.mimo_c5_prof_reset()
    n = 10
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(n):
        p.detect(H, y, float(w.sigma2), out=out)
    ev1.record()
    torch.cuda.synchronize()
    buf = np.zeros(148 * 32, np.uint64)
    L.mimo_c5_prof_read(buf.ctypes.data)
    b = buf.reshape(148, 32).astype(np.float64)
    units_per_cta = w.n_units / 148.0
    print(f"{kn}: {ev0.elapsed_time(ev1) / n * 1e3:.1f} us/call (prof build)")
    for s, nm in sorted(names.items()):
        v = b[:, s].mean() / (n * units_per_cta)
        print(f"   {nm:24s} {v:9.0f} cycles/unit")
