#!/bin/bash
# Capture the ncu evidence committed under profiles/ (run under gpurun, 1 GPU).
# Usage: tools/profile_round.sh <round tag>
# Each ncu command runs only after the same command exited 0 without ncu.
set -u
tag=${1:-r02}
out=gpurun_out/prof_$tag
mkdir -p $out
for k in 1 2 3 4 5; do
  cmd="python bench.py --config $k --profile --steps 3 --warmup 2"
  $cmd > $out/plain_c$k.log 2>&1 || { echo "plain run failed for C$k"; continue; }
  timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --csv --log-file $out/launches_c$k.csv $cmd > $out/ncu_launch_c$k.log 2>&1
done
# DRAM traffic of whole steps over a range of back-to-back calls (counts the LLR write-back)
for k in 2 3 4 5; do
  python tools/traffic_range.py --config $k --steps 8 > $out/range_plain_c$k.log 2>&1 && \
  timeout 600 ncu --profile-from-start off --cache-control none --clock-control none --csv \
      --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --log-file $out/range_c$k.csv python tools/traffic_range.py --config $k --steps 8 > $out/ncu_range_c$k.log 2>&1
done
# full captures of the dominant kernels
full() {  # config kernel-regex skip name [bench args]
  local k=$1 re=$2 skip=$3 name=$4 extra=${5:-}
  python bench.py --config $k --profile --steps 3 --warmup 2 $extra > $out/plain_full_$name.log 2>&1 && \
    timeout 600 ncu --set full --clock-control none --import-source on -k regex:$re -s $skip -c 1 -o $out/full_$name \
        python bench.py --config $k --profile --steps 3 --warmup 2 $extra > $out/ncu_full_$name.log 2>&1
}
full 2 k_tpu 2 c2
full 3 k_apply_stream 2 c3
full 4 k_lg3 2 c4
full 5 k_c5_apply 1 c5
full 5 k_c5_setup 1 c5_setup "--kernel c5_bf16kc_tcs_be_64x16_q6_i8"  # the two-kernel variant's setup
timeout 600 python tools/time_varying.py --out $out/time_varying.jsonl > $out/time_varying.log 2>&1
ls -la $out
