"""Time the time-varying-channel kernels (NEXT-3: H constant over sym_per_h < 14 symbols) against
the generic kernel on the full C2 - C5 grids, through the C ABI (mimo.Plan.detect), the way
bench.py times a step: rotating buffer sets > 3x L2, CUDA-graph replays, CUDA events on the
launching stream. Writes one JSON line per (config, sym_per_h, kernel).

    python tools/time_varying.py [--configs 2 3 4 5] [--out profiles/r02/time_varying.jsonl]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    from paper_2510_07843_b200 import mimo, synth
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--configs", type=int, nargs="*", default=[2, 3, 4, 5])
    args = ap.parse_args()
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    hbm = float(peaks.get("hbm_gbs", 6547.2))
    lines = []
    for k, sph, kernels in ((2, 7, ["tpu_4x4_q4_f32_s7", "generic"]), (2, 2, ["tpu_4x4_q4_f32_s2", "generic"]),
                            (2, 1, ["tpu_4x4_q4_f32_s1", "generic"]), (2, 14, ["tpu_4x4_q4_f32"]),
                            (3, 7, ["stream_8x4_q6_i8_s7", "generic"]), (3, 2, ["stream_8x4_q6_i8_s2", "generic"]),
                            (3, 1, ["stream_8x4_q6_i8_s1", "generic"]), (3, 14, ["stream_8x4_q6_i8"]),
                            (4, 7, ["lg_16x8_q8_f16_s7", "generic"]), (4, 2, ["lg_16x8_q8_f16_s2"]),
                            (4, 1, ["lg_16x8_q8_f16_s1"]), (4, 14, ["lg_16x8_q8_f16", "lg3hl_16x8_q8_f16"]),
                            (5, 7, ["big_64x16_q6_i8_s7", "generic"]), (5, 2, ["big_64x16_q6_i8_s2"]),
                            (5, 1, ["big_64x16_q6_i8_s1"]), (5, 14, ["big_64x16_q6_i8", None])):
        if k not in args.configs:
            continue
        cfg = dict(synth.CONFIGS[k], sym_per_h=sph)
        w = synth.generate(cfg)
        n_units = w.n_units
        llr_b = {"f32": 4, "f16": 2, "i8": 1}[w.llr]
        bytes_step = n_units * w.n_rx * w.n_layers * 8 + w.n_re * w.n_rx * 8 + w.n_re * w.n_layers * w.qm * llr_b
        nset = max(2, int(3 * 126e6 // bytes_step) + 1)
        for kn in kernels:
            plan = mimo.Plan(w.n_rx, w.n_layers, w.qm, sc_per_h=w.sc_per_h, sym_per_h=sph, llr_dtype=w.llr,
                             kernel=kn)
            sets = []
            for _ in range(nset):
                H = torch.from_numpy(w.H).cuda()
                y = torch.from_numpy(w.y).cuda()
                out = torch.empty(plan.shapes(w.n_sc, w.n_sym)["llr"], dtype=plan.llr_dtype, device="cuda")
                sets.append((H, y, out))
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                for H, y, out in sets:  # warm-up (also sizes the plan's workspace before capture)
                    plan.detect(H, y, float(w.sigma2), out=out)
            stream.synchronize()
            assert plan.sync_status() == 0
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=stream):
                for H, y, out in sets:
                    plan.detect(H, y, float(w.sigma2), out=out)
            for _ in range(20):
                g.replay()
            torch.cuda.synchronize()
            reps = max(1, args.steps // nset)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(stream):
                e0.record(stream)
                for _ in range(reps):
                    g.replay()
                e1.record(stream)
            torch.cuda.synchronize()
            us = e0.elapsed_time(e1) * 1e3 / (reps * nset)
            line = {"config": w.name, "sym_per_h": sph, "kernel": plan.kernel_name, "us_per_step": us,
                    "RE_per_s": w.n_re / (us * 1e-6), "algorithmic_bytes": bytes_step,
                    "hbm_frac": bytes_step / (us * 1e-6) / (hbm * 1e9), "n_units": n_units,
                    "l2": f"{nset} rotating buffer sets"}
            print(json.dumps(line), flush=True)
            lines.append(line)
            plan.close()
    if args.out:
        with open(args.out, "w") as f:
            for l in lines:
                f.write(json.dumps(l) + "\n")


if __name__ == "__main__":
    main()
