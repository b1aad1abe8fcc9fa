#!/bin/bash
timeout 600 python -m pytest tests/test_variants_gpu.py -q -x -k "c4" 2>&1 | tail -2
for k in lg3hp_16x8_q8_f16 lg3hq_16x8_q8_f16 lg3hp_16x8_q8_f16 lg3hq_16x8_q8_f16; do echo $k; timeout 60 python tools/dbg_time.py $k 4 20 1 2>&1 | tail -1; done
