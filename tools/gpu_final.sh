#!/bin/bash
# Round-end evidence: GPU tests, smoke, bench lines (default + all configs + reference arm + BFP), studies.
mkdir -p gpurun_out/final
export PYTHONUNBUFFERED=1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/final/pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"; tail -2 gpurun_out/final/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/final/smoke.log
timeout 600 python bench.py > gpurun_out/final/bench_default.json 2> gpurun_out/final/bench_default.err; echo "bench rc=$?"
timeout 1200 python bench.py --config all --no-e2e --no-cpu-baseline > gpurun_out/final/bench_all.jsonl 2> gpurun_out/final/bench_all.err; echo "bench all rc=$?"
timeout 300 python bench.py --config 3 --bfp 9 --no-e2e --no-cpu-baseline > gpurun_out/final/bench_c3_bfp9.json 2>&1; echo "bfp rc=$?"
timeout 600 python bench.py --impl reference --steps 20 --warmup 3 > gpurun_out/final/bench_reference.json 2>&1; echo "ref rc=$?"
python - <<'PY'
import json
for f in ["gpurun_out/final/bench_default.json", "gpurun_out/final/bench_all.jsonl", "gpurun_out/final/bench_c3_bfp9.json", "gpurun_out/final/bench_reference.json"]:
    try:
        for ln in open(f):
            if ln.startswith("{"):
                d = json.loads(ln)
                r = d.get("roofline") or {}
                print(f.split("/")[-1], d.get("config", {}).get("workload", "")[:12], d.get("config", {}).get("kernel"), "value %.4g" % d.get("value"), "us/step %.2f" % (1000 * d.get("ms_per_step")), "frac", r.get("frac"), r.get("bound"), "e2e", (d.get("e2e") or {}).get("value"), "clk", (d.get("clocks") or {}).get("sm_mhz"), (d.get("clocks") or {}).get("reasons"))
    except Exception as e:
        print(f, "ERR", e)
PY
bash tools/profile_round.sh r01 > gpurun_out/final/profile_round.log 2>&1; echo "profile rc=$?"
