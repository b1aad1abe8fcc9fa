"""Diagnostic timings (not the bench): per-call device time of detect variants.

    python tools/diag.py --config 2 [--kernels a,b,...]

For each kernel variant (MIMO_FORCE_KERNEL), times through CUDA graphs over
rotating buffer sets (> 3x L2): full detect (LLRs), LLRs+x~ debug, and
setup-only (only the SINR debug output requested -> no per-RE work or stores).
"""
import argparse
import math
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

from paper_2510_07843_b200 import synth  # noqa: E402


def time_calls(fn, n_sets, steps=400):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        for i in range(3):
            fn(i % n_sets)
    s.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for i in range(steps):
                fn(i % n_sets)
    s.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        for _ in range(3):
            g.replay()
        e0.record(s)
        for _ in range(5):
            g.replay()
        e1.record(s)
    s.synchronize()
    return e0.elapsed_time(e1) * 1e3 / (5 * steps)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="2")
    ap.add_argument("--kernels", default="")
    ap.add_argument("--ref", action="store_true", help="also time torch copies of the same byte count")
    ap.add_argument("--overlap", default="0", help="comma list of overlap modes to time (0,1)")
    args = ap.parse_args()
    k = int(args.config)
    from paper_2510_07843_b200 import mimo
    w = synth.generate(k)
    b = synth.config_algorithmic_bytes(k)
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    n_sets = max(2, math.ceil(3 * l2 / b["total"]))
    H0, y0 = torch.from_numpy(w.H).cuda(), torch.from_numpy(w.y).cuda()
    if args.ref:
        for mb in (8, 24, 48, 96, 400):
            n = int(mb * 1e6 / 2 / 4)
            nst = max(2, math.ceil(3 * l2 / (mb * 1e6)))
            bufs = [(torch.empty(n, device="cuda"), torch.empty(n, device="cuda")) for _ in range(nst)]
            t = time_calls(lambda i: bufs[i][1].copy_(bufs[i][0]), nst)
            print(f"torch copy {mb:5d} MB traffic: {t:8.2f} us  {mb * 1e6 / t / 1e3:7.1f} GB/s", flush=True)
            del bufs
        e = torch.empty(1, device="cuda")
        t = time_calls(lambda i: e.add_(0), 1)
        print(f"tiny kernel: {t:8.2f} us", flush=True)
    kernels = [x for x in args.kernels.split(",") if x] or [""]
    for kn, ov in [(kn, int(ov)) for kn in kernels for ov in args.overlap.split(",")]:
        if kn:
            os.environ["MIMO_FORCE_KERNEL"] = kn
        plan = mimo.Plan(w.n_rx, w.n_layers, w.qm, sc_per_h=w.sc_per_h, llr_dtype=w.llr, overlap_calls=bool(ov))
        sh = plan.shapes(w.n_sc, w.n_sym)
        sets = [(H0.clone(), y0.clone(), torch.empty(sh["llr"], dtype=plan.llr_dtype, device="cuda"),
                 torch.empty(sh["sinr"], device="cuda"), torch.empty(sh["xhat"], dtype=torch.complex64, device="cuda"))
                for _ in range(n_sets)]
        s2 = float(w.sigma2)
        full = time_calls(lambda i: plan.detect(sets[i][0], sets[i][1], s2, out=sets[i][2]), n_sets)
        setup = time_calls(lambda i: plan.detect(sets[i][0], sets[i][1], s2, sinr=sets[i][3], want_llr=False), n_sets)
        dbg = time_calls(lambda i: plan.detect(sets[i][0], sets[i][1], s2, out=sets[i][2], xhat=sets[i][4]), n_sets)
        print(f"{plan.kernel_name:36s} ov={ov} full {full:8.2f} us ({b['total'] / full / 1e3:7.1f} GB/s)  "
              f"setup-only {setup:8.2f} us  llr+xhat {dbg:8.2f} us", flush=True)
        del sets
        plan.close()


if __name__ == "__main__":
    main()
