#!/bin/bash
# C5-only evidence refresh: GPU suite, smoke, bench C5 default, ncu launch list / step range / full capture
set -u
out=gpurun_out/ev_c5; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $out/smoke.log 2>&1
timeout 300 python bench.py > $out/bench_default.json 2> $out/bench_default.err
timeout 300 python bench.py --config 5 --steps 300 --warmup 20 --no-cpu-baseline --no-e2e --kernel c5_fusedbid_64x16_q6_i8 > $out/bench_bid.json 2>/dev/null
timeout 300 python bench.py > $out/bench_default2.json 2> $out/bench_default2.err
cmd="python bench.py --config 5 --profile --steps 3 --warmup 2"
$cmd > $out/plain_c5.log 2>&1 && timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --csv --log-file $out/launches_c5.csv $cmd > $out/ncu_launch_c5.log 2>&1
python tools/traffic_range.py --config 5 --steps 8 > $out/range_plain_c5.log 2>&1 && \
  timeout 600 ncu --profile-from-start off --cache-control none --clock-control none --csv \
      --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --log-file $out/range_c5.csv python tools/traffic_range.py --config 5 --steps 8 > $out/ncu_range_c5.log 2>&1
$cmd > $out/plain_full_c5.log 2>&1 && timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_c5_apply -s 1 -c 1 -o $out/full_c5 $cmd > $out/ncu_full_c5.log 2>&1
ls -la $out
