#!/bin/bash
timeout 600 python -m pytest tests/test_parity_gpu.py tests/test_variants_gpu.py tests/test_edge_gpu.py -q -x -k "3 or c3 or stream" 2>&1 | tail -2
for k in stream_8x4_q6_i8 stream_8x4_q6_i8 stream_8x4_q6_i8; do echo $k; timeout 60 python tools/dbg_time.py $k 3 20 1 2>&1 | tail -1; done
