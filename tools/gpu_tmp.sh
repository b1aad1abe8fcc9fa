#!/bin/bash
for k in big8_64x16_q6_i8 ablation_big8_noconv ablation_big8_noepi ablation_big8_none ablation_big8_mma1 big11_64x16_q6_i8 ablation_big11_noconv; do echo $k; timeout 60 python tools/dbg_time.py $k 5 40 1 2>&1 | tail -1; done
python bench.py --config 5 --profile --steps 3 --warmup 2 > /dev/null 2>&1
for k in big8_64x16_q6_i8 ablation_big8_noconv ablation_big8_none; do
MIMO_FORCE_KERNEL=$k ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_big_apply --csv python bench.py --config 5 --profile --steps 3 --warmup 2 2>/dev/null | grep k_big_apply | tail -1 | awk -F'","' '{print $NF}'
done
