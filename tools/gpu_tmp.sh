#!/bin/bash
timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_api_gpu.py -q -x 2>&1 | tail -2
timeout 400 python bench.py --config 2 2>/dev/null | tail -1 > gpurun_out/bench_c2.json; python -c "import json; d=json.loads(open('gpurun_out/bench_c2.json').read()); print(d['ms_per_step'], d['e2e'], d['cpu_baseline'])"
