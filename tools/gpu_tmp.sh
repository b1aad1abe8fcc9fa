#!/bin/bash
timeout 600 python -m pytest tests/test_variants_gpu.py -q -x -k "c3" 2>&1 | tail -3
timeout 300 bash tools/bench_variants.sh 3 stream_8x4_q6_i8 tma_8x4_q6_i8 tma_8x4_q6_i8_s3m4 tma_8x4_q6_i8_s6m2 tma_8x4_q6_i8_s2m6
