#!/bin/bash
timeout 60 python tools/dbg_size.py big8e6h_64x16_q6_i8 3276 40 big8e6_64x16_q6_i8 2>&1 | tail -1
for k in big8e6_64x16_q6_i8 big8e6h_64x16_q6_i8 big8e6_64x16_q6_i8 big8e6h_64x16_q6_i8; do echo $k; timeout 60 python tools/dbg_time.py $k 5 40 1 2>&1 | tail -1; done
python bench.py --config 5 --profile --steps 3 --warmup 2 > /dev/null 2>&1
for k in big8e6_64x16_q6_i8 big8e6h_64x16_q6_i8; do MIMO_FORCE_KERNEL=$k ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_big_setup --csv python bench.py --config 5 --profile --steps 3 --warmup 2 2>/dev/null | grep k_big_setup | tail -1 | awk -F'","' '{print $5, $NF}'; done
