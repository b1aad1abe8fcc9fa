#!/bin/bash
for i in 1 2 3 4; do
BENCH_DEBUG_E2E=1 timeout 400 python bench.py 2>gpurun_out/err.txt | tail -1 > gpurun_out/b.json; grep "e2e async" gpurun_out/err.txt; python -c "import json; d=json.loads(open('gpurun_out/b.json').read()); print(d['ms_per_step']*1e3, d['e2e']['ms_per_step'], d['e2e']['sync_call_ms_per_step'])"
done
