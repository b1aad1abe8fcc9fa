"""K back-to-back detect calls of one config over rotating buffer sets (as bench.py), bracketed by
cudaProfilerStart/Stop, for an ncu capture of the DRAM traffic of whole steps WITHOUT cache flushes
between the kernels -- so the LLR write-back that a single cold kernel capture leaves in L2 is
counted in the next kernel (the last step's L2-resident tail, <= 126 MB, is the only undercount):

    ncu --profile-from-start off --cache-control none \\
        --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \\
        python tools/traffic_range.py --config 5 --steps 8
(ncu's --replay-mode range cannot be used: it rejects cuTensorMapEncodeTiled inside the range.)
"""
import argparse
import math
import os
import sys

import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_07843_b200 import mimo, synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--steps", type=int, default=8)
ap.add_argument("--kernel", default=None)
args = ap.parse_args()
w = synth.generate(args.config)
b = synth.config_algorithmic_bytes(args.config)
p = mimo.Plan(w.n_rx, w.n_layers, w.qm, sc_per_h=w.sc_per_h, llr_dtype=w.llr, kernel=args.kernel)
n_sets = max(2, math.ceil(3 * torch.cuda.get_device_properties(0).L2_cache_size / b["total"]))
H0, y0 = torch.from_numpy(w.H).cuda(), torch.from_numpy(w.y).cuda()
sets = [(H0.clone(), y0.clone(), torch.empty(p.shapes(w.n_sc, w.n_sym)["llr"], dtype=p.llr_dtype, device="cuda"))
        for _ in range(n_sets)]
for i in range(2 * n_sets):  # warm-up (module load, workspace)
    H, y, o = sets[i % n_sets]
    p.detect(H, y, float(w.sigma2), out=o)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStart()
for i in range(args.steps):
    H, y, o = sets[i % n_sets]
    p.detect(H, y, float(w.sigma2), out=o)
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
assert p.sync_status() == 0
print(f"config {args.config}: {args.steps} steps, {n_sets} buffer sets, algorithmic {b['total']} B/step, kernel {p.kernel_name}")
