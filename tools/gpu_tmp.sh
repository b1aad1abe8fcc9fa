#!/bin/bash
timeout 600 python -m pytest tests/test_variants_gpu.py -q -x -k "c3" 2>&1 | tail -2
for k in stream_8x4_q6_i8 streaml_8x4_q6_i8 stream_8x4_q6_i8 streaml_8x4_q6_i8; do echo $k; timeout 60 python tools/dbg_time.py $k 3 20 1 2>&1 | tail -1; done
python bench.py --config 3 --profile --steps 3 --warmup 2 > /dev/null 2>&1
MIMO_FORCE_KERNEL=streaml_8x4_q6_i8 ncu --metrics gpu__time_duration.sum --clock-control none --csv python bench.py --config 3 --profile --steps 3 --warmup 2 2>/dev/null | grep "k_" | tail -2 | awk -F'","' '{print $5, $NF}'
