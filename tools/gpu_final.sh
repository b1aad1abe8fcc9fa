#!/bin/bash
# Round-end evidence: GPU tests, smoke, bench lines (default + all configs + reference arm), studies.
mkdir -p gpurun_out/final
export PYTHONUNBUFFERED=1
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/final/pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"; tail -2 gpurun_out/final/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/final/smoke.log
timeout 600 python bench.py > gpurun_out/final/bench_default.json 2> gpurun_out/final/bench_default.err; echo "bench rc=$?"
timeout 1200 python bench.py --config all --no-e2e --no-cpu-baseline > gpurun_out/final/bench_all.jsonl 2> gpurun_out/final/bench_all.err; echo "bench all rc=$?"
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/final/bench_reference.json 2>&1; echo "ref rc=$?"
timeout 600 python tools/lu_breakdown.py --reps 30 --out gpurun_out/final/lu_breakdown > /dev/null 2>&1; echo "lu rc=$?"
timeout 900 python tests/accuracy_study.py --out gpurun_out/final/accuracy_sweep > /dev/null 2>&1; echo "acc rc=$?"
python - <<'PY'
import json
for f in ["gpurun_out/final/bench_default.json", "gpurun_out/final/bench_all.jsonl", "gpurun_out/final/bench_reference.json"]:
    try:
        for ln in open(f):
            if ln.startswith("{"):
                d = json.loads(ln)
                r = d.get("roofline") or {}
                print(f.split("/")[-1], d.get("config", {}).get("workload", "")[:12], d.get("config", {}).get("kernel"), "value", d.get("value"), "ms", d.get("ms_per_step"), "frac", r.get("frac"), r.get("bound"), "e2e", (d.get("e2e") or {}).get("value"), "clk", d.get("clocks"))
    except Exception as e:
        print(f, "ERR", e)
PY
