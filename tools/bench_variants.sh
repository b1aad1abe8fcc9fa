#!/bin/bash
# usage: tools_bench_variants.sh CONFIG kernel1 kernel2 ...
cfg=$1; shift
for k in "$@"; do
  MIMO_FORCE_KERNEL=$k python bench.py --config $cfg --no-e2e --no-cpu-baseline --steps 2000 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['kernel'], round(d['roofline']['step_us'],2), 'us', round(d['roofline']['frac'],3), d['clocks']['sm_mhz'], d['clocks']['reasons'])" || echo "$k failed"
done
