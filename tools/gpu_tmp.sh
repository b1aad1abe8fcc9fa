#!/bin/bash
for k in stream_8x4_q6_i8 stream_u32 stream_u64 stream_8x4_q6_i8 stream_u32 stream_u64; do echo $k; timeout 60 python tools/dbg_time.py $k 3 20 1 2>&1 | tail -1; done
timeout 300 bash tools/bench_variants.sh 3 stream_8x4_q6_i8 stream_u32
