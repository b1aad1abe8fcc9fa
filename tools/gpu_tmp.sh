#!/bin/bash
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --config 5 --no-e2e --no-cpu-baseline > gpurun_out/bench_c5.json 2>gpurun_out/bench_c5.err; echo "bench rc=$?"
python -c "import json; d=json.loads(open('gpurun_out/bench_c5.json').read().strip().splitlines()[-1]); print(d['config']['kernel'], d['ms_per_step']*1000, d['roofline']['frac'], d['roofline']['bound'], d['clocks'])"
