#!/bin/bash
timeout 300 python bench.py --config P --no-cpu-baseline 2>/dev/null | tail -1 | cut -c1-400
timeout 300 python bench.py --config 5 --steps 50 --warmup 3 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['ms_per_step'], d['roofline']['frac'], d['gpu_launches'], d['step_us_per_replay'])"
