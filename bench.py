#!/usr/bin/env python
"""Benchmark of the B200 per-RE MMSE detector + max-log demapper.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config 5] [--impl ours|reference]
                    [--emulate 2 4 8] [--kernel NAME]

Metric (BASELINE.json): MIMO-detected REs/s (and LLR Gbit/s) per B200 vs roofline.
A "step" is one mimo_detect_mmse call over one full batch of the configured
workload -- every hot-path row a1-a7 for every RE. The default workload is the
largest config, configs[4] = C5 (64 rx x 16 layers, 64-QAM, 3276 sc x 14 sym x
40 slots, int8 LLRs; BASELINE.json "sharded by slot across 8 GPUs"); --config k
selects another. Inputs are device-resident and rotated over enough buffer sets
that the working set exceeds 3x L2; the K timed steps are replayed from CUDA
graphs and timed with CUDA events on the launching stream.

Multi-GPU (torchrun, N ranks): STRONG scaling of the same configured job. Every
rank draws the whole seeded job and detects its block of the 2-D slot x PRB
partition (shard.block_partition: C5 over 8 GPUs = 5 slots each); there is no
collective on the data path. Timing: barrier, graph replays, synchronize,
barrier; value = job REs x K / max over ranks of the CUDA-event time (the host
wall clock over the same region is reported beside it). --emulate N runs the N
shards one after another on a single GPU, reports their times and checks that
the reassembled LLRs are bit-identical to the unsharded call.

`e2e` times the same metric through the host-buffer C-ABI call
(mimo_detect_mmse_host_async: pinned H/y -> device -> kernels -> LLRs back), and
`cpu_baseline` / `--impl reference` time the fp64 oracle (test infrastructure,
deliberately slow) on a bounded sample on the host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

from paper_2510_07843_b200 import shard, synth  # noqa: E402

METRIC = "MIMO-detected REs/s per B200 (LLR Gbit/s alongside) vs roofline"
FALLBACK_HBM_GBS = 6650.0   # B200_PROFILING.md fallback, used only if MEASURED_PEAKS.json is absent
FALLBACK_BF16_TFLOPS = 2250.0  # B200_PROFILING.md nominal dense bf16
TF32_PER_BF16 = 1.1 / 2.25   # B200_PROFILING.md nominal dense tf32 / bf16
TC_KERNELS = ("c5",)  # kernels whose row a6 runs on tcgen05 (R21, R28)
# The paper's own CPU figure: a 4x4 LMMSE detection of one 720-subcarrier,
# 14-symbol TTI in <= 0.03 ms on an Intel i9-14900KF with AVX2 -- another CPU and workload.
PAPER_CPU_CONTEXT = {"value": 720 * 14 / 0.03e-3, "unit": "RE/s", "hardware": "Intel Core i9-14900KF, AVX2",
                     "workload": "4x4, 60 RB x 12 = 720 subcarriers x 14 symbols, one TTI, <= 0.03 ms",
                     "source": "PAPER.md:117, :123", "note": "context only: different CPU and workload"}


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=50)
    ap.add_argument("--config", default="5",
                    help="BASELINE config 1..5 (default 5 = configs[4], the largest), P (paper shape) or all")
    ap.add_argument("--kernel", default=None, help="kernel specialisation by name (default: the plan's default)")
    ap.add_argument("--emulate", type=int, nargs="*", default=[],
                    help="one-GPU emulation of N-GPU strong scaling (each N: shards run sequentially)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=60)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="CPU budget of the oracle baseline")
    ap.add_argument("--profile", action="store_true", help="short run for ncu (no graphs, no e2e/cpu legs)")
    ap.add_argument("--bfp", type=int, default=0,
                    help="NEXT-4: feed y as W-bit block-floating-point (mimo_detect_mmse_bfp: decoded in the C3 apply "
                         "loads, expanded by k_bfp_decode for the other shapes)")
    ap.add_argument("--overlap", type=int, default=1,
                    help="1: back-to-back calls overlap via PDL (MIMO_PLAN_OVERLAP_CALLS); 0: serialised")
    return ap.parse_args()


def cfg_key(s):
    return "P" if s == "P" else int(s)


def workload_desc(k) -> dict:
    c = synth.CONFIGS[k]
    return {"workload": f"{c['name']}: {c['n_rx']}x{c['n_layers']} {2 ** c['qm']}-QAM, {c['n_sc']} sc x "
                        f"{synth.SYM_PER_SLOT} sym x {c['n_slots']} slots, H per "
                        f"{'subcarrier' if c['sc_per_h'] == 1 else 'PRB'}, {c['llr']} LLR, SNR {c['snr_db']} dB",
            "n_rx": c["n_rx"], "n_layers": c["n_layers"], "qm": c["qm"], "n_sc": c["n_sc"],
            "n_sym": c["n_slots"] * synth.SYM_PER_SLOT, "sc_per_h": c["sc_per_h"], "llr_type": c["llr"]}


def measured_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return dict(hbm_gbs=float(d["hbm_gbs"]), src="measured", sm_max_mhz=float(d.get("sm_max_mhz", 1965.0)),
                    bf16_tflops=float(d.get("bf16_tflops", FALLBACK_BF16_TFLOPS)))
    return dict(hbm_gbs=FALLBACK_HBM_GBS, src="fallback", sm_max_mhz=1965.0, bf16_tflops=FALLBACK_BF16_TFLOPS)


def kernel_share(args, k) -> dict | None:
    """Share of the step of the dominant kernel, from the committed ncu launch list (profiles/)."""
    p = os.path.join(ROOT, "profiles", "kernel_share.json")
    if not os.path.exists(p) or args.kernel:
        return None
    with open(p) as f:
        d = json.load(f)
    return d.get(synth.CONFIGS[k]["name"])


def ncu_traffic(k) -> float | None:
    """DRAM read + write bytes per STEP from the committed ncu range capture (profiles/traffic.json:
    8 back-to-back calls over rotating buffers, so the LLR write-back is counted), comparable with
    the algorithmic bytes per step that `achieved` uses."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    v = d.get(synth.CONFIGS[k]["name"])
    return float(v["dram_bytes_per_step"]) if v and "dram_bytes_per_step" in v else None


# ----------------------------------------------------------------- clocks --
class ClockSampler:
    """Samples SM clock and clock-event reasons through NVML while running."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, torch_index: int, period: float = 0.05):
        self.samples, self.reasons, self.ok = [], set(), False
        self.power, self.power_limit = [], None
        self.period = period
        self._stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            import torch
            uuid = str(torch.cuda.get_device_properties(torch_index).uuid)
            h = None
            for i in range(pynvml.nvmlDeviceGetCount()):
                hh = pynvml.nvmlDeviceGetHandleByIndex(i)
                u = pynvml.nvmlDeviceGetUUID(hh)
                u = u.decode() if isinstance(u, bytes) else u
                if u.replace("GPU-", "") == uuid.replace("GPU-", ""):
                    h = hh
            if h is None:
                h = pynvml.nvmlDeviceGetHandleByIndex(torch_index)
            self.h, self.nvml = h, pynvml
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            try:
                self.power_limit = pynvml.nvmlDeviceGetEnforcedPowerLimit(h) / 1000.0
            except Exception:
                self.power_limit = None
            self.ok = True
        except Exception as e:  # no NVML: report nothing rather than guess
            self.err = repr(e)
            self.max_mhz = None

    def _run(self):
        nv = self.nvml
        while not self._stop.is_set():
            try:
                self.samples.append(nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM))
                try:
                    self.power.append(nv.nvmlDeviceGetPowerUsage(self.h) / 1000.0)
                except Exception:
                    pass
                r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h) \
                    if hasattr(nv, "nvmlDeviceGetCurrentClocksEventReasons") \
                    else nv.nvmlDeviceGetCurrentClocksThrottleReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(self.period)

    def __enter__(self):
        if self.ok:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def __exit__(self, *exc):
        if self.ok:
            self._stop.set()
            self._t.join()

    def result(self) -> dict:
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": [], "note": "NVML unavailable"}
        r = {"sm_mhz": float(statistics.median(self.samples)), "sm_max_mhz": self.max_mhz,
             "reasons": sorted(self.reasons), "samples": len(self.samples)}
        if self.power:  # board power under load vs the enforced limit (sw_power_cap = at the limit)
            r["power_w"] = round(float(statistics.median(self.power)), 1)
            r["power_limit_w"] = self.power_limit
        return r


# ------------------------------------------------------------ oracle legs --
def oracle_rate(w: synth.Workload, seconds: float, threads: int) -> dict:
    """Time the fp64 oracle (as it stands) on a bounded prefix of units, ~`seconds` of CPU work."""
    import oracle
    Hu = w.H_units()
    Yall = synth.unit_gather(w.y, w.n_slots, w.n_sc, w.sc_per_h)
    n = 1
    while True:  # calibrate on a growing prefix, then size the sample
        t0 = time.perf_counter()
        oracle.detect(Hu[:n], Yall[:n], w.sigma2, w.qm, threads=threads)
        dt = time.perf_counter() - t0
        if dt > 0.2 or n >= w.n_units:
            break
        n = min(w.n_units, n * 8)
    n_s = int(min(w.n_units, max(1, n * seconds / max(dt, 1e-6))))
    reps, t0 = 0, time.perf_counter()
    while True:  # repeat a sample that is the whole workload until >= 2 s for a stable rate
        oracle.detect(Hu[:n_s], Yall[:n_s], w.sigma2, w.qm, threads=threads)
        reps += 1
        dt = time.perf_counter() - t0
        if dt >= min(2.0, seconds):
            break
    n_re = n_s * synth.SYM_PER_SLOT * w.sc_per_h * reps
    return dict(value=n_re / dt, unit="RE/s", cores=threads, kind="oracle",
                sample=f"first {n_s} of {w.n_units} H-units of {w.name} x {reps} repeats ({n_re} REs), fp64 Gram/Cholesky + "
                       f"brute-force max-log, OpenMP over units", seconds=dt)


def run_reference(args, k):
    """--impl reference: the fp64 oracle as the reference arm (rank 0 only)."""
    import oracle
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    w = synth.generate(k)
    threads = oracle.max_threads()
    Hu = w.H_units()
    Yall = synth.unit_gather(w.y, w.n_slots, w.n_sc, w.sc_per_h)
    # per-step sample sized so that (W + K) steps take ~120 s in total
    t0 = time.perf_counter()
    oracle.detect(Hu[:64], Yall[:64], w.sigma2, w.qm, threads=threads)
    per_unit = (time.perf_counter() - t0) / 64
    budget = 120.0 / max(1, args.steps + args.warmup)
    n_s = int(max(1, min(w.n_units, budget / max(per_unit, 1e-9))))
    for i in range(args.warmup):
        oracle.detect(Hu[:n_s], Yall[:n_s], w.sigma2, w.qm, threads=threads)
    t0 = time.perf_counter()
    for i in range(args.steps):
        off = (i * n_s) % max(1, w.n_units - n_s + 1)
        oracle.detect(Hu[off:off + n_s], Yall[off:off + n_s], w.sigma2, w.qm, threads=threads)
    dt = time.perf_counter() - t0
    n_re = n_s * synth.SYM_PER_SLOT * w.sc_per_h * args.steps
    v = n_re / dt
    c = synth.CONFIGS[k]
    line = {"impl": "reference", "metric": METRIC, "value": v,
            "unit": "RE/s", "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": dt * 1e3 / args.steps, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE config shapes)",
            "config": workload_desc(k),
            "llr_gbit_s": v * c["n_layers"] * c["qm"] / 1e9,
            "cpu_baseline": {"value": v, "unit": "RE/s", "cores": threads, "kind": "oracle",
                             "sample": f"{n_s} H-units per step ({n_s * 14 * c['sc_per_h']} REs) of {c['name']}"},
            "e2e": {"value": v, "unit": "RE/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# -------------------------------------------------------------- ours -------
def largest_divisor_le(n: int, cap: int) -> int:
    for d in range(min(n, cap), 0, -1):
        if n % d == 0:
            return d
    return 1


class Shard:
    """One plan + rotating device buffer sets for one block of the configured job."""

    def __init__(self, mimo, w, Hn, yn, n_sc, n_slots, dev, k, args, overlap, ybfp=None):
        import torch
        self.n_sc, self.n_slots, self.n_sym = n_sc, n_slots, n_slots * synth.SYM_PER_SLOT
        self.b = synth.config_algorithmic_bytes(k, n_sc=n_sc, n_slots=n_slots)
        self.bfp = args.bfp
        if ybfp is not None:  # NEXT-4: y crosses HBM as BFP blocks (reading R25)
            self.b = dict(self.b, y=int(ybfp.nbytes), total=self.b["H"] + int(ybfp.nbytes) + self.b["llr"])
        self.plan = mimo.Plan(w.n_rx, w.n_layers, w.qm, sc_per_h=w.sc_per_h, llr_dtype=w.llr, device=dev.index,
                              overlap_calls=overlap, kernel=args.kernel)
        self.plan.reserve(n_sc, self.n_sym)
        l2 = torch.cuda.get_device_properties(dev).L2_cache_size
        n_sets = max(2, math.ceil(3 * l2 / self.b["total"]))  # working set >= 3x L2: every step streams HBM
        free = torch.cuda.mem_get_info(dev)[0]
        self.n_sets = int(min(n_sets, max(2, (free * 0.4) // self.b["total"])))
        H0 = torch.from_numpy(Hn).to(dev)
        y0 = torch.from_numpy(yn if ybfp is None else ybfp).to(dev)
        self.sets = [(H0.clone(), y0.clone(),
                      torch.empty(self.plan.shapes(n_sc, self.n_sym)["llr"], dtype=self.plan.llr_dtype, device=dev))
                     for _ in range(self.n_sets)]
        del H0, y0
        self.s2 = float(w.sigma2)
        self.l2 = l2

    def step(self, i):
        H, y, out = self.sets[i % self.n_sets]
        if not self.bfp:
            self.plan.detect(H, y, self.s2, out=out)
        else:
            self.plan.detect_bfp(H, y, self.s2, n_sym=self.n_sym, n_sc=self.n_sc, iq_width=self.bfp, out=out)

    def graph(self, S, stream):
        import torch
        with torch.cuda.stream(stream):
            for i in range(3):  # eager warm-up (module load, first launches)
                self.step(i)
        stream.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(stream):
            with torch.cuda.graph(g, stream=stream):
                for i in range(S):
                    self.step(i)
        stream.synchronize()
        return g


def timed_replays(g, stream, K, S, W, barrier=None):
    """W warm-up steps (>= 0.3 s), then K steps as K/S graph replays bracketed by barrier +
    synchronize; CUDA events on the launching stream. Returns (elapsed_ms, wall_s, per-replay us)."""
    import torch
    with torch.cuda.stream(stream):
        t_end = time.perf_counter() + 0.3
        done = 0
        while done < W or time.perf_counter() < t_end:
            g.replay()
            done += S
        stream.synchronize()
    if barrier:
        barrier()
    torch.cuda.synchronize()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(K // S + 1)]
    t0 = time.perf_counter()
    with torch.cuda.stream(stream):
        evs[0].record(stream)
        for r in range(K // S):
            g.replay()
            evs[r + 1].record(stream)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    if barrier:
        barrier()
    per = sorted(evs[r].elapsed_time(evs[r + 1]) * 1e3 / S for r in range(K // S))
    return evs[0].elapsed_time(evs[-1]), wall, per


def roofline_of(k, plan_kernel, b, fl, step_s, peaks, dev):
    import torch
    n_sm = torch.cuda.get_device_properties(dev).multi_processor_count
    fp32_tflops = n_sm * 128 * 2 * peaks["sm_max_mhz"] * 1e6 / 1e12  # 148 SMs x 128 lanes x 2 x max clock
    t_hbm = b["total"] / (peaks["hbm_gbs"] * 1e9)
    # row a6 on tcgen05 (3-pass split products, R21/R28): its flops leave the FP32 pipe
    tensor_apply = plan_kernel.startswith(TC_KERNELS)
    simt_flops = fl["setup"] + fl["demap"] if tensor_apply else fl["total"]
    t_alu = simt_flops / (fp32_tflops * 1e12)
    tf32_tflops = peaks["bf16_tflops"] * TF32_PER_BF16
    t_tc = 3 * fl["apply"] / (tf32_tflops * 1e12) if tensor_apply else 0.0
    if t_alu > t_hbm and t_alu >= t_tc:
        roof = {"bound": "alu", "achieved": simt_flops / step_s / 1e12, "peak": fp32_tflops, "unit": "TFLOP/s",
                "frac": (simt_flops / step_s / 1e12) / fp32_tflops, "algorithmic_flops_per_step": simt_flops,
                "peak_src": f"derived: {n_sm} SMs x 128 FP32 lanes x 2 x {peaks['sm_max_mhz']:.0f} MHz"}
    elif t_tc > t_hbm:
        roof = {"bound": "tensor", "achieved": 3 * fl["apply"] / step_s / 1e12, "peak": tf32_tflops,
                "unit": "TFLOP/s", "frac": (3 * fl["apply"] / step_s / 1e12) / tf32_tflops,
                "peak_src": "measured bf16 x nominal TF32/BF16 ratio (B200_PROFILING.md)"}
    else:
        ach = b["total"] / step_s / 1e9
        roof = {"bound": "hbm", "achieved": ach, "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": ach / peaks["hbm_gbs"], "peak_src": peaks["src"] + " (MEASURED_PEAKS.json hbm_gbs)"}
    roof.update({"algorithmic_bytes_per_step": b["total"], "t_roof_us": max(t_hbm, t_alu, t_tc) * 1e6,
                 "step_us": step_s * 1e6, "apply_pipe": "tcgen05 (3-pass split, R21/R28)" if tensor_apply else "FP32 SIMT",
                 "t_hbm_us": t_hbm * 1e6, "t_simt_us": t_alu * 1e6, "t_tensor_us": t_tc * 1e6})
    return roof


def emulate_shards(mimo, w, k, args, dev, n_emul, full_llr):
    """One-GPU emulation of an N-GPU strong-scaling run: run every rank's block of
    the 2-D partition sequentially on this device, time each (CUDA graphs, events), and check that
    the reassembled LLRs are bit-identical to the unsharded call. The emulated N-GPU step time is
    the max over shards (the ranks would run concurrently on their own GPUs)."""
    import torch
    n_prb = w.n_sc // shard.SC_PER_PRB
    try:
        blocks = shard.block_partition(w.n_slots, n_prb, n_emul)
    except ValueError as e:
        return {"n": n_emul, "unavailable": str(e)}
    full = torch.empty_like(full_llr)
    stream = torch.cuda.Stream(device=dev)
    shard_us = []
    K = max(8, min(args.steps, 64))
    S = largest_divisor_le(K, 64)
    for blk in blocks:
        Hb, yb, nsc, nsl = shard.shard_arrays(w.H, w.y, w.n_slots, w.sc_per_h, blk)
        sh = Shard(mimo, w, Hb, yb, nsc, nsl, dev, k, args, overlap=bool(args.overlap))
        g = sh.graph(S, stream)
        el, _, _ = timed_replays(g, stream, K, S, 3)
        shard_us.append(el * 1e3 / K)
        H, y, out = sh.sets[0]
        with torch.cuda.stream(stream):
            sh.plan.detect(H, y, sh.s2, out=out)
        stream.synchronize()
        shard.place_block(full, out, blk)
        del sh, g
        torch.cuda.empty_cache()
    t = max(shard_us)
    return {"n": n_emul, "grid": list(blocks[0]["grid"]), "shard_step_us": shard_us, "step_us": t,
            "value": w.n_re / (t * 1e-6), "unit": "RE/s", "steps_per_shard": K,
            "bit_identical": bool(torch.equal(full, full_llr))}


def result_placement(mimo, w, blk, sh, stream, dev, world, rank):
    """N > 1, after (outside) the timed detection: every rank's LLR block goes point to point to
    rank 0 (NCCL over NVLink) and is written into the full grid there (shard.place_blocks_p2p) --
    the north_star's "result placement", timed on its own (CUDA events, max over ranks) and checked
    bit-identical against rank 0 detecting the whole job on its own GPU."""
    import torch
    import torch.distributed as dist
    n_prb = w.n_sc // shard.SC_PER_PRB
    blocks = shard.block_partition(w.n_slots, n_prb, world)
    local = sh.sets[0][2]
    with torch.cuda.stream(stream):
        sh.plan.detect(sh.sets[0][0], sh.sets[0][1], sh.s2, out=local)
    stream.synchronize()
    full_shape = (w.n_sym, w.n_sc) + tuple(local.shape[2:])
    dist.barrier()
    torch.cuda.synchronize(dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    full = shard.place_blocks_p2p(local, blocks, full_shape)
    e1.record()
    torch.cuda.synchronize(dev)
    ms = shard.max_over_ranks(e0.elapsed_time(e1), device=dev)
    nbytes = local.element_size() * int(torch.Size(full_shape).numel())
    out = {"ms": ms, "bytes": nbytes, "GB_s": nbytes / (ms * 1e-3) / 1e9,
           "how": "each rank's LLR block sent point to point to rank 0 (NCCL send/recv), placed into the full "
                  "[sym][sc][layer][bit] grid in rank 0's HBM; not part of the detection step"}
    if rank == 0:  # verification: the whole job on rank 0's GPU alone
        p = mimo.Plan(w.n_rx, w.n_layers, w.qm, sc_per_h=w.sc_per_h, llr_dtype=w.llr, device=dev.index)
        Hd, yd = torch.from_numpy(w.H).to(dev), torch.from_numpy(w.y).to(dev)
        ref = p.detect(Hd, yd, float(w.sigma2))
        torch.cuda.synchronize(dev)
        out["bit_identical_to_1gpu"] = bool(torch.equal(ref, full))
    return out


def run_ours(args, k):
    import torch
    import torch.distributed as dist
    from paper_2510_07843_b200 import mimo

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if args.gpus != world and world > 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    barrier = (lambda: dist.barrier()) if world > 1 else None

    c = synth.CONFIGS[k]
    w = synth.generate(k)  # the whole configured job, one seed: every rank draws the same job
    n_prb = w.n_sc // shard.SC_PER_PRB
    # strong scaling: rank r detects its block of the 2-D slot x PRB partition of THIS job (no
    # collective on the data path); a job too small to split (C1) runs as replicas
    try:
        blk = shard.block_partition(w.n_slots, n_prb, world)[rank] if world > 1 else None
        scaling = "strong"
    except ValueError:
        blk, scaling = None, "replicas"
    if blk is not None:
        Hn, yn, n_sc_r, n_slots_r = shard.shard_arrays(w.H, w.y, w.n_slots, w.sc_per_h, blk)
    else:
        Hn, yn, n_sc_r, n_slots_r = w.H, w.y, w.n_sc, w.n_slots
    ybfp = synth.bfp_compress(yn, args.bfp) if args.bfp else None
    sh = Shard(mimo, w, Hn, yn, n_sc_r, n_slots_r, dev, k, args, overlap=bool(args.overlap), ybfp=ybfp)
    plan = sh.plan
    stream = torch.cuda.Stream(device=dev)

    if args.profile:
        with torch.cuda.stream(stream):
            for i in range(args.warmup + args.steps):
                sh.step(i)
        torch.cuda.synchronize(dev)
        assert plan.sync_status() == 0
        if rank == 0:
            print(json.dumps({"profile_run": True, "kernel": plan.kernel_name,
                              "launches": args.warmup + args.steps}), flush=True)
        return

    K, W = args.steps, max(3, args.warmup)
    S = largest_divisor_le(K, 256)
    g = sh.graph(S, stream)
    sampler = ClockSampler(local)
    with sampler:
        elapsed_ms, wall_s, per_replay_us = timed_replays(g, stream, K, S, W, barrier)
    pct = lambda q: per_replay_us[min(len(per_replay_us) - 1, int(q * len(per_replay_us)))]
    step_dist = {"p10": pct(0.1), "p50": pct(0.5), "p90": pct(0.9), "replays": len(per_replay_us),
                 "steps_per_replay": S}
    n_failed = plan.sync_status()
    assert n_failed == 0, f"{n_failed} units failed the Cholesky guard"

    # context: the same steps with calls serialised (no PDL overlap) -> single-call device time
    sh1 = Shard.__new__(Shard)
    sh1.__dict__.update(sh.__dict__)
    sh1.plan = mimo.Plan(w.n_rx, w.n_layers, w.qm, sc_per_h=w.sc_per_h, llr_dtype=w.llr, device=local,
                         kernel=args.kernel)
    sh1.plan.reserve(n_sc_r, sh.n_sym)
    g1 = sh1.graph(S, stream)
    el1, _, _ = timed_replays(g1, stream, S, S, 1)
    single_us = el1 * 1e3 / S
    del g1

    t_max_ms = shard.max_over_ranks(elapsed_ms, device=dev)
    placement = result_placement(mimo, w, blk, sh, stream, dev, world, rank) if blk is not None else None
    wall_max = shard.max_over_ranks(wall_s, device=dev)
    n_re_job = synth.config_algorithmic_bytes(k)["n_re"]
    n_re_all = n_re_job * K * (world if scaling == "replicas" else 1)
    value = n_re_all / (t_max_ms / 1e3)
    peaks = measured_peaks()
    step_s = (t_max_ms / 1e3) / K
    b = sh.b
    fl = synth.config_algorithmic_flops(k, n_sc=n_sc_r, n_slots=n_slots_r)
    roof = roofline_of(k, plan.kernel_name, b, fl, step_s, peaks, dev)
    roof.update({"traffic": ncu_traffic(k) if world == 1 and not args.bfp else None,
                 "launches_per_step": plan.launches_per_call, "serialised_call_us": single_us,
                 "serialised_frac": roof["t_roof_us"] / single_us})
    dk = kernel_share(args, k)
    if dk:
        roof["dominant_kernel"] = dk
    clocks = sampler.result()

    # e2e: the public host-buffer C-ABI call (mimo_detect_mmse_host_async), pinned host buffers:
    # every step copies its H and y host->device and its LLRs device->host inside the timed region
    e2e = None
    if not args.no_e2e:
        Hh = torch.from_numpy(Hn).pin_memory()
        yh = torch.from_numpy(yn if ybfp is None else ybfp).pin_memory()
        lh = torch.empty(plan.shapes(n_sc_r, sh.n_sym)["llr"], dtype=plan.llr_dtype).pin_memory()
        if ybfp is None:
            host_call = lambda wait: plan.detect_host(Hh, yh, sh.s2, out=lh, wait=wait)
        else:  # NEXT-4: the BFP fronthaul bytes cross PCIe, decompressed inside the apply kernel
            host_call = lambda wait: plan.detect_bfp_host(Hh, yh, sh.s2, n_sym=sh.n_sym, n_sc=n_sc_r,
                                                          iq_width=args.bfp, out=lh, wait=wait)
        for _ in range(2):
            host_call(True)
        if barrier:
            barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            host_call(True)
        dt_sync = shard.max_over_ranks(time.perf_counter() - t0, device=dev)
        for _ in range(3):
            host_call(False)
        plan.sync_status()
        if barrier:
            barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            host_call(False)
        plan.sync_status()
        dt = shard.max_over_ranks(time.perf_counter() - t0, device=dev)
        e2e = {"value": n_re_job * args.e2e_steps * (world if scaling == "replicas" else 1) / dt, "unit": "RE/s",
               "h2d_bytes_per_step": b["H"] + b["y"], "d2h_bytes_per_step": b["llr"],
               "ms_per_step": dt * 1e3 / args.e2e_steps,
               "path": ("mimo_detect_mmse_host_async" if ybfp is None else f"mimo_detect_mmse_bfp_host_async (BFP{args.bfp} y)")
                       + " per step + one plan sync (pinned host buffers, 3-stream slot-chunk pipeline; consecutive "
                         "steps overlap their transfers)",
               "sync_call_ms_per_step": dt_sync * 1e3 / args.e2e_steps,
               "bytes_note": "per rank" if world > 1 else "whole job"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline and ybfp is None:
        import oracle
        cpu = oracle_rate(w, args.cpu_seconds, oracle.max_threads())
        one = oracle_rate(w, min(3.0, args.cpu_seconds), 1)  # also on one thread
        cpu["single_thread"] = {"value": one["value"], "unit": "RE/s", "cores": 1, "sample": one["sample"]}
        cpu["paper_context"] = PAPER_CPU_CONTEXT

    emul = None
    if world == 1 and args.emulate and ybfp is None:
        H, y, out = sh.sets[0]
        with torch.cuda.stream(stream):
            plan.detect(H, y, sh.s2, out=out)
        stream.synchronize()
        full_llr = out.clone()
        emul = [emulate_shards(mimo, w, k, args, dev, n, full_llr) for n in args.emulate]

    if barrier:
        barrier()
    if rank != 0:
        dist.destroy_process_group()
        return
    cfg = workload_desc(k)
    cfg.update({"l2_flush": f"{sh.n_sets} rotating buffer sets x {b['total'] / 1e6:.1f} MB = "
                            f"{sh.n_sets * b['total'] / 1e6:.0f} MB > 3x L2 ({sh.l2 / 1e6:.0f} MB)",
                "graph_steps": S, "kernel": plan.kernel_name + ((f" + BFP{args.bfp} y (k_apply_bfp)" if k == 3 else f" + BFP{args.bfp} y (k_bfp_decode)")
                                              if ybfp is not None else ""),
                "y_format": f"BFP {args.bfp}-bit mantissas, block per (symbol, PRB, antenna) (reading R25)"
                            if ybfp is not None else "complex64",
                "call_overlap": "PDL (MIMO_PLAN_OVERLAP_CALLS): call i+1 loads/sets up while call i stores"
                                if args.overlap else "none (serialised calls)",
                "input_sha256": w.sha256(),
                "parallelism": (f"2-D slot x PRB block partition {blk['grid'][0]}x{blk['grid'][1]} over {world} GPUs, "
                                f"rank 0 block slots {blk['slots']} PRBs {blk['prbs']}, no collective")
                               if blk is not None else (f"{world} replicas (job too small to split)" if world > 1
                                                        else "single GPU, whole job")})
    line = {
        "metric": METRIC,
        "value": value, "unit": "RE/s", "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": t_max_ms / K, "wall_ms_per_step": wall_max * 1e3 / K,
        "step_us_per_replay": step_dist, "higher_is_better": True,
        "scaling": "strong" if world == 1 else scaling,
        "vs_baseline": None, "dtype": "f32", "setup_dtype": "f64" if plan.kernel_name.startswith("tpu") else "f32",
        "data": "synthetic (seeded numpy PCG64, BASELINE config shapes; DESIGN.md input recipe)",
        "config": cfg,
        "llr_gbit_s": value * w.n_layers * w.qm / 1e9,
        "roofline": roof,
        "cpu_baseline": cpu,
        "e2e": e2e,
        "clocks": clocks,
        "gpu_launches": K * plan.launches_per_call,
    }
    if emul is not None:
        line["emulated_multi_gpu"] = emul
    if placement is not None:
        line["placement"] = placement
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    args = parse()
    keys = [1, 2, 3, 4, 5] if args.config == "all" else [cfg_key(args.config)]
    for k in keys:
        if args.impl == "reference":
            run_reference(args, k)
        else:
            run_ours(args, k)


if __name__ == "__main__":
    main()
