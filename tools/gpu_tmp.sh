#!/bin/bash
for k in stream_8x4_q6_i8 streamf_8x4_q6_i8 streamf32_8x4_q6_i8 stream_8x4_q6_i8 streamf_8x4_q6_i8 streamf32_8x4_q6_i8; do echo $k; timeout 60 python tools/dbg_time.py $k 3 20 1 2>&1 | tail -1; done
echo "no overlap"; for k in stream_8x4_q6_i8 streamf_8x4_q6_i8; do echo $k; timeout 60 python tools/dbg_time.py $k 3 20 0 2>&1 | tail -1; done
timeout 600 python -m pytest tests/test_variants_gpu.py -q -x -k "c3" 2>&1 | tail -2
