"""e2e (host-buffer) timing of one config for several host-path chunk sizes."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_07843_b200 import mimo, synth

k = int(sys.argv[1]) if len(sys.argv) > 1 else 2
w = synth.generate(k)
Hh = torch.from_numpy(w.H).pin_memory()
yh = torch.from_numpy(w.y).pin_memory()
for cb in [int(x) for x in (sys.argv[2].split(",") if len(sys.argv) > 2 else ["2097152"])]:
    os.environ["MIMO_HOST_CHUNK_BYTES"] = str(cb)
    plan = mimo.Plan(w.n_rx, w.n_layers, w.qm, sc_per_h=w.sc_per_h, llr_dtype=w.llr)
    lh = torch.empty(plan.shapes(w.n_sc, w.n_sym)["llr"], dtype=plan.llr_dtype).pin_memory()
    for _ in range(3):
        plan.detect_host(Hh, yh, float(w.sigma2), out=lh)
    t0 = time.perf_counter()
    for _ in range(20):
        plan.detect_host(Hh, yh, float(w.sigma2), out=lh)
    dt = (time.perf_counter() - t0) / 20
    print(f"C{k} chunk {cb / 1e6:6.2f} MB: {dt * 1e3:7.3f} ms/step  {w.n_re / dt:.3e} RE/s", flush=True)
    plan.close()
