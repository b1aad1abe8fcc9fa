"""e2e host-path throughput (C2) vs MIMO_HOST_CHUNK_BYTES, synchronous and asynchronous calls."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_07843_b200 import mimo, synth

w = synth.generate(int(sys.argv[1]) if len(sys.argv) > 1 else 2)
plan = mimo.Plan(w.n_rx, w.n_layers, w.qm, sc_per_h=w.sc_per_h, llr_dtype=w.llr)
H, y = torch.from_numpy(w.H).pin_memory(), torch.from_numpy(w.y).pin_memory()
out = torch.empty(plan.shapes(w.n_sc, w.n_sym)["llr"], dtype=plan.llr_dtype).pin_memory()
n_re = w.n_sym * w.n_sc
for cb in [1 << 20, 2 << 20, 4 << 20, 8 << 20, 16 << 20, 64 << 20]:
    os.environ["MIMO_HOST_CHUNK_BYTES"] = str(cb)
    for wait in (True, False):
        for _ in range(3):
            plan.detect_host(H, y, float(w.sigma2), out=out, wait=wait)
        plan.sync_status()
        t0 = time.perf_counter(); t_enq = 0.0
        for _ in range(20):
            t1 = time.perf_counter()
            plan.detect_host(H, y, float(w.sigma2), out=out, wait=wait)
            t_enq += time.perf_counter() - t1
        plan.sync_status()
        dt = (time.perf_counter() - t0) / 20
        print(f"chunk {cb >> 20:3d} MiB wait={wait!s:5}: {dt * 1e3:.3f} ms/step  {n_re / dt:.3e} RE/s  "
              f"(call returns after {t_enq / 20 * 1e3:.3f} ms)", flush=True)
