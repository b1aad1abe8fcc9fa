#!/bin/bash
# Capture the ncu evidence committed under profiles/ (run under gpurun, 1 GPU).
# Usage: tools/profile_round.sh <round tag>
# Each ncu command runs only after the same command exited 0 without ncu.
set -u
tag=${1:-r01}
out=gpurun_out/prof_$tag
mkdir -p $out
for k in 1 2 3 4 5; do
  cmd="python bench.py --config $k --profile --steps 3 --warmup 2"
  $cmd > $out/plain_c$k.log 2>&1 || { echo "plain run failed for C$k"; continue; }
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
      --csv --log-file $out/launches_c$k.csv $cmd > $out/ncu_launch_c$k.log 2>&1
done
# full captures of the dominant kernel of each config
full() {  # config kernel-regex skip
  local k=$1 re=$2 skip=$3
  python bench.py --config $k --profile --steps 3 --warmup 2 > $out/plain_full_c$k.log 2>&1 && \
    ncu --set full --clock-control none --import-source on -k regex:$re -s $skip -c 1 -o $out/full_c$k \
        python bench.py --config $k --profile --steps 3 --warmup 2 > $out/ncu_full_c$k.log 2>&1
}
full 2 k_tpu 2
full 3 k_apply_stream 2
full 4 k_lg3 2
full 5 k_big_apply4 1
python bench.py --config 5 --profile --steps 3 --warmup 2 > /dev/null 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_big_setup -s 1 -c 1 -o $out/full_c5_setup \
      python bench.py --config 5 --profile --steps 3 --warmup 2 > $out/ncu_full_c5_setup.log 2>&1
ls -la $out
