#!/bin/bash
# Round evidence: bench lines of every config (+ BFP e2e, reference arm), step traffic ranges.
set -u
out=gpurun_out/${TAG:-final}; mkdir -p $out
timeout 1500 python bench.py --config all --emulate 2 4 8 > $out/bench_all.jsonl 2> $out/bench_all.err
timeout 300 python bench.py --config 3 --bfp 9 > $out/bench_c3_bfp9.json 2> $out/bench_c3_bfp9.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > $out/bench_reference.json 2> $out/bench_reference.err
for k in 2 3 4 5; do
  timeout 600 ncu --profile-from-start off --cache-control none --clock-control none --csv \
      --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --log-file $out/range_c$k.csv python tools/traffic_range.py --config $k --steps 8 > $out/ncu_range_c$k.log 2>&1
done
ls -la $out
