#!/bin/bash
mkdir -p gpurun_out
timeout 120 python tools/dbg_size.py big4_64x16_q6_i8 3276 40 big4c_64x16_q6_i8 2>&1 | tail -1
for k in big4c_64x16_q6_i8 big4_64x16_q6_i8; do timeout 60 python tools/dbg_time.py $k 5 40 1 2>&1 | tail -1; done
timeout 900 python -m pytest tests/test_variants_gpu.py tests/test_parity_gpu.py -q -x -k "c5 or 5" 2>&1 | tail -3
timeout 300 bash tools/bench_variants.sh 5 big4c_64x16_q6_i8 big4_64x16_q6_i8
python bench.py --config 5 --profile --steps 3 --warmup 2 > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_big --csv python bench.py --config 5 --profile --steps 3 --warmup 2 2>/dev/null | grep -E "k_big" | tail -4 | cut -c1-250
