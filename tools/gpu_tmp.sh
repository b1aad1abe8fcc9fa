#!/bin/bash
mkdir -p gpurun_out
timeout 60 python tools/dbg_time.py big4_64x16_q6_i8 5 2>&1 | tail -4
timeout 60 python tools/dbg_time.py big6_64x16_q6_i8 5 4 0 2>&1 | tail -4
timeout 60 python tools/dbg_time.py big6_64x16_q6_i8 5 40 0 2>&1 | tail -4
timeout 60 python tools/dbg_time.py big6_64x16_q6_i8 5 40 1 2>&1 | tail -4
