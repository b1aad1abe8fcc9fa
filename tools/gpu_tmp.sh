#!/bin/bash
timeout 600 python -m pytest tests/test_variants_gpu.py -q -x -k "c3" 2>&1 | tail -2
for k in stream_8x4_q6_i8 ring_s4m4 ring_s6m3 ring_s7m4 ring_s3m4 stream_8x4_q6_i8; do echo $k; timeout 60 python tools/dbg_time.py $k 3 20 1 2>&1 | tail -1; done
