"""Summarise an ncu capture directory (tools/profile_round.sh) into profiles/<tag>/.

    python tools/ncu_summary.py gpurun_out/prof_r02 profiles/r02

Writes launches_c*.csv (copied), full_*.txt (selected raw metrics + SASS instruction
classes of the dominant kernels), range_c*.csv (copied), summary.md, and updates
profiles/traffic.json (DRAM bytes per STEP from the range captures -- whole steps of
back-to-back calls, LLR write-back included) and profiles/kernel_share.json (the
dominant kernel's share of the step from the launch lists).
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys
from collections import Counter

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2510_07843_b200 import synth  # noqa: E402

RAW = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_bytes.sum",
       "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__issue_active.avg.pct_of_peak_sustained_active",
       "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
       "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
       "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "launch__grid_size",
       "launch__block_size", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
       "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smsp__inst_executed.sum",
       "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio",
       "smsp__average_warps_issue_stalled_no_instruction_per_issue_active.ratio"]
SCALE = {"Mbyte": 1e6, "Kbyte": 1e3, "Gbyte": 1e9, "byte": 1.0, "us": 1.0, "ns": 1e-3, "ms": 1e3, "usecond": 1.0,
         "nsecond": 1e-3, "msecond": 1e3}
FULL = [("c2", 2, "k_tpu"), ("c3", 3, "k_apply_stream"), ("c4", 4, "k_lg3"), ("c5", 5, "k_c5_apply"),
        ("c5_setup", 5, "k_c5_setup")]
# SASS instruction classes that evidence the Blackwell data paths (B200_PROFILING.md)
CLASSES = {"UTCHMMA": "tcgen05.mma (kind::f16/tf32)", "UTCBAR": "tcgen05.commit", "UTMALDG": "TMA tensor load",
           "UBLKCP": "bulk copy (cp.async.bulk)", "LDTM": "tcgen05.ld (TMEM -> regs)", "STTM": "tcgen05.st (regs -> TMEM)",
           "FFMA2": "packed fp32 FMA", "FFMA": "fp32 FMA", "F2FP": "fp32 -> bf16/fp16 pack", "SHFL": "warp shuffle"}


def _csv(path):
    lines = [ln for ln in open(path) if not ln.startswith("==")]
    return list(csv.reader(io.StringIO("".join(lines))))


def read_launches(path):
    rows = _csv(path)
    if not rows:
        return []
    h = rows[0]
    out = {}
    for r in rows[1:]:
        d = dict(zip(h, r))
        key = (int(d["ID"]), d["Kernel Name"])
        out.setdefault(key, {})[d["Metric Name"]] = (float(d["Metric Value"].replace(",", "")), d["Metric Unit"])
    return [(i, n, m) for (i, n), m in sorted(out.items())]


def _val(m, key):
    v, u = m.get(key, (0.0, "byte"))
    return v * SCALE.get(u, 1.0)


def raw_metrics(rep):
    r = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True)
    rows = list(csv.reader(io.StringIO(r.stdout)))
    if len(rows) < 3:
        return {}, ""
    h, u, v = rows[0], rows[1], rows[2]
    d = {a: (c, b) for a, b, c in zip(h, u, v)}
    return d, d.get("Kernel Name", ("", ""))[0]


def sass_classes(rep, n_units):
    r = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                       capture_output=True, text=True)
    rows = list(csv.reader(io.StringIO(r.stdout)))
    if len(rows) < 3:
        return {}, 0
    h = rows[1]
    iS, iE = h.index("Source"), h.index("Instructions Executed")
    c = Counter()
    for row in rows[2:]:
        if len(row) <= iE or not row[iE].strip().isdigit():
            continue
        op = row[iS].split()
        if not op:
            continue
        o = op[1] if op[0].startswith("@") else op[0]
        c[o.split(".")[0]] += int(row[iE])
    tot = sum(c.values())
    return {k: c.get(k, 0) / n_units for k in CLASSES}, tot / n_units


def main():
    src, dst = sys.argv[1], sys.argv[2]
    tag = os.path.basename(dst.rstrip("/"))
    os.makedirs(dst, exist_ok=True)
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    spath = os.path.join(ROOT, "profiles", "kernel_share.json")
    traffic, share = {}, {}
    md = [f"# ncu summary ({tag})", "",
          "Launch lists: `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
          "--clock-control none` over `python bench.py --config k --profile --steps 3 --warmup 2` "
          "(serialised, cold-cache launches: compare shares, not absolutes). Step traffic: "
          "`ncu --cache-control none` over 8 back-to-back calls of `tools/traffic_range.py` (rotating buffer sets "
          "> 3x L2, no cache flush between kernels), so the LLR write-back is counted.", ""]
    for k in (1, 2, 3, 4, 5):
        name = synth.CONFIGS[k]["name"]
        b = synth.config_algorithmic_bytes(k)
        lp = os.path.join(src, f"launches_c{k}.csv")
        if os.path.exists(lp):
            shutil.copy(lp, os.path.join(dst, f"launches_c{k}.csv"))
            L = read_launches(lp)
            md += [f"## {name}: algorithmic bytes per step {b['total'] / 1e6:.2f} MB", "",
                   "| launch | kernel | time (us) | DRAM read (MB) | DRAM write (MB) |", "|---|---|---|---|---|"]
            per = Counter()
            for i, n, m in L:
                t = _val(m, "gpu__time_duration.sum") if m["gpu__time_duration.sum"][1] != "ns" else \
                    m["gpu__time_duration.sum"][0] * 1e-3
                per[n.split("(")[0]] += t
                md.append(f"| {i} | `{n[:64]}` | {t:.2f} | {_val(m, 'dram__bytes_read.sum') / 1e6:.2f} | "
                          f"{_val(m, 'dram__bytes_write.sum') / 1e6:.2f} |")
            md.append("")
            if per:
                top, tt = per.most_common(1)[0]
                share[name] = {"kernel": top, "share_of_step": tt / sum(per.values()),
                               "source": f"profiles/{tag}/launches_c{k}.csv"}
                md += [f"Dominant kernel `{top[:70]}`: {100 * tt / sum(per.values()):.1f}% of the serialised step.", ""]
        rp = os.path.join(src, f"range_c{k}.csv")
        if os.path.exists(rp):
            shutil.copy(rp, os.path.join(dst, f"range_c{k}.csv"))
            L = read_launches(rp)  # every kernel of 8 back-to-back steps, caches not flushed in between
            if L:
                rd = sum(_val(m, "dram__bytes_read.sum") for _, _, m in L) / 8
                wr = sum(_val(m, "dram__bytes_write.sum") for _, _, m in L) / 8
                traffic[name] = {"dram_bytes_per_step": rd + wr, "dram_read_per_step": rd, "dram_write_per_step": wr,
                                 "algorithmic_bytes_per_step": b["total"], "ratio": (rd + wr) / b["total"],
                                 "launches": len(L), "source": f"profiles/{tag}/range_c{k}.csv",
                                 "note": "ncu --cache-control none over 8 back-to-back calls (rotating buffers): L2 "
                                         "write-back of one kernel's LLRs lands in the next; per step, includes the "
                                         "setup kernel's W~ workspace traffic where there is one"}
                md += [f"Step traffic (8 calls, no cache flush between kernels): read {rd / 1e6:.1f} MB + write "
                       f"{wr / 1e6:.1f} MB = {(rd + wr) / 1e6:.1f} MB per step = {(rd + wr) / b['total']:.3f} x "
                       f"the algorithmic {b['total'] / 1e6:.1f} MB.", ""]
    for nm, k, _ in FULL:
        rep = os.path.join(src, f"full_{nm}.ncu-rep")
        if not os.path.exists(rep):
            continue
        d, kname = raw_metrics(rep)
        n_units = synth.config_algorithmic_bytes(k)["n_units"]
        cls, tot = sass_classes(rep, n_units)
        with open(os.path.join(dst, f"full_{nm}.txt"), "w") as f:
            f.write(f"# ncu --set full, {synth.CONFIGS[k]['name']}, kernel {kname}\n")
            for m in RAW:
                if m in d:
                    f.write(f"{m} = {d[m][0]} {d[m][1]}\n")
            f.write(f"# SASS instructions executed per H-unit (warp level; all classes: {tot:.0f})\n")
            for c, v in cls.items():
                f.write(f"sass.{c} = {v:.1f}   # {CLASSES[c]}\n")
        md += [f"Full capture `{nm}`: `{kname[:80]}` -> `full_{nm}.txt` (raw metrics, SASS classes per unit: "
               + ", ".join(f"{c} {v:.0f}" for c, v in cls.items() if v) + ").", ""]
    open(os.path.join(dst, "summary.md"), "w").write("\n".join(md) + "\n")
    if traffic:
        json.dump(traffic, open(tpath, "w"), indent=1)
    if share:
        json.dump(share, open(spath, "w"), indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
