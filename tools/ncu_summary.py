"""Summarise an ncu capture directory (tools/profile_round.sh) into profiles/<tag>/.

    python tools/ncu_summary.py gpurun_out/prof_r01 profiles/r01

Writes launches_c*.csv (copied), full_c*.txt (selected raw metrics of the
dominant kernel), summary.md, and updates profiles/traffic.json (per-launch DRAM
bytes of each config's dominant kernel from its --set full capture).
"""
import csv
import io
import json
import os
import shutil
import subprocess
import sys

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
       "smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio"]
SCALE = {"Mbyte": 1e6, "Kbyte": 1e3, "Gbyte": 1e9, "byte": 1.0, "us": 1.0, "ns": 1e-3, "ms": 1e3}


def read_launches(path):
    lines = [ln for ln in open(path) if not ln.startswith("==")]
    rows = list(csv.reader(io.StringIO("".join(lines))))
    if not rows:
        return []
    h = rows[0]
    out = {}
    for r in rows[1:]:
        d = dict(zip(h, r))
        key = (int(d["ID"]), d["Kernel Name"])
        out.setdefault(key, {})[d["Metric Name"]] = (float(d["Metric Value"].replace(",", "")), d["Metric Unit"])
    return [(i, n, m) for (i, n), m in sorted(out.items())]


def raw_metrics(rep):
    r = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True)
    rows = list(csv.reader(io.StringIO(r.stdout)))
    if len(rows) < 3:
        return {}, ""
    h, u, v = rows[0], rows[1], rows[2]
    d = {a: (c, b) for a, b, c in zip(h, u, v)}
    return d, d.get("Kernel Name", ("", ""))[0]


def main():
    src, dst = sys.argv[1], sys.argv[2]
    os.makedirs(dst, exist_ok=True)
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    traffic = json.load(open(tpath)) if os.path.exists(tpath) else {}
    md = [f"# ncu summary ({os.path.basename(dst)})", "",
          "Launch lists: `ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum "
          "--clock-control none` over `python bench.py --config k --profile --steps 3 --warmup 2` "
          "(serialised, cold-cache launches: compare shares, not absolutes).", ""]
    for k in (1, 2, 3, 4, 5):
        name = synth.CONFIGS[k]["name"]
        b = synth.config_algorithmic_bytes(k)
        lp = os.path.join(src, f"launches_c{k}.csv")
        if os.path.exists(lp):
            shutil.copy(lp, os.path.join(dst, f"launches_c{k}.csv"))
            L = read_launches(lp)
            md += [f"## {name}: algorithmic bytes per step {b['total'] / 1e6:.2f} MB", "",
                   "| launch | kernel | time (us) | DRAM read (MB) | DRAM write (MB) |", "|---|---|---|---|---|"]
            for i, n, m in L:
                t = m["gpu__time_duration.sum"][0] * (1e-3 if m["gpu__time_duration.sum"][1] == "ns" else 1)
                rd = m.get("dram__bytes_read.sum", (0, "byte"))
                wr = m.get("dram__bytes_write.sum", (0, "byte"))
                md.append(f"| {i} | `{n[:60]}` | {t:.2f} | {rd[0] * SCALE.get(rd[1], 1) / 1e6:.2f} | "
                          f"{wr[0] * SCALE.get(wr[1], 1) / 1e6:.2f} |")
            md.append("")
        rep = os.path.join(src, f"full_c{k}.ncu-rep")
        if os.path.exists(rep):
            d, kname = raw_metrics(rep)
            with open(os.path.join(dst, f"full_c{k}.txt"), "w") as f:
                f.write(f"# ncu --set full, {name}, kernel {kname}\n")
                for m in RAW:
                    if m in d:
                        f.write(f"{m} = {d[m][0]} {d[m][1]}\n")
            rd = float(d["dram__bytes_read.sum"][0]) * SCALE.get(d["dram__bytes_read.sum"][1], 1)
            wr = float(d["dram__bytes_write.sum"][0]) * SCALE.get(d["dram__bytes_write.sum"][1], 1)
            traffic[name] = {"kernel": kname, "dram_bytes_per_launch": rd + wr, "dram_read": rd, "dram_write": wr,
                             "source": f"profiles/{os.path.basename(dst)}/full_c{k}.txt",
                             "note": "cold single-launch capture: LLR writes still resident in L2 at kernel end "
                                     "are not counted as DRAM writes"}
            md += [f"Full capture of `{kname[:70]}`: DRAM read {rd / 1e6:.2f} MB, write {wr / 1e6:.2f} MB, "
                   f"see `full_c{k}.txt`.", ""]
    open(os.path.join(dst, "summary.md"), "w").write("\n".join(md) + "\n")
    json.dump(traffic, open(tpath, "w"), indent=1)
    print("\n".join(md))


if __name__ == "__main__":
    main()
