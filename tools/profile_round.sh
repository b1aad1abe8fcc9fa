#!/bin/bash
# Capture the ncu evidence committed under profiles/ (run under gpurun, 1 GPU).
# Usage: tools/profile_round.sh <round tag>
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
# full captures of the dominant kernels
python bench.py --config 2 --profile --steps 3 --warmup 2 > $out/plain_full_c2.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_tpu -s 2 -c 1 -o $out/full_c2 \
      python bench.py --config 2 --profile --steps 3 --warmup 2 > $out/ncu_full_c2.log 2>&1
python bench.py --config 4 --profile --steps 3 --warmup 2 > $out/plain_full_c4.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_lg -s 2 -c 1 -o $out/full_c4 \
      python bench.py --config 4 --profile --steps 3 --warmup 2 > $out/ncu_full_c4.log 2>&1
python bench.py --config 5 --profile --steps 2 --warmup 1 > $out/plain_full_c5.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_big_apply -s 1 -c 1 -o $out/full_c5 \
      python bench.py --config 5 --profile --steps 2 --warmup 1 > $out/ncu_full_c5.log 2>&1
python bench.py --config 3 --profile --steps 3 --warmup 2 > $out/plain_full_c3.log 2>&1 && \
  ncu --set full --clock-control none --import-source on -k regex:k_apply_stream -s 2 -c 1 -o $out/full_c3 \
      python bench.py --config 3 --profile --steps 3 --warmup 2 > $out/ncu_full_c3.log 2>&1
ls -la $out
