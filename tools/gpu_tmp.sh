#!/bin/bash
mkdir -p gpurun_out/final2
timeout 600 python bench.py > gpurun_out/final2/bench_default.json 2> gpurun_out/final2/bench_default.err; echo "bench rc=$?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final2/smoke.log 2>&1; echo "smoke rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/final2/bench_default.json').read().strip().splitlines()[-1]); print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['cpu_baseline']['value'], d['cpu_baseline']['single_thread']['value'], d['clocks'])"
