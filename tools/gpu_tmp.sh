#!/bin/bash
for k in big8e6_64x16_q6_i8 big8e6s6_64x16_q6_i8 big8e6s3_64x16_q6_i8 big8e6_64x16_q6_i8 big8e6s6_64x16_q6_i8; do echo $k; timeout 60 python tools/dbg_time.py $k 5 40 1 2>&1 | tail -1; done
