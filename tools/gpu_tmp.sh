#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -x -k "4 or c4 or lg" 2>&1 | tail -2
timeout 300 bash tools/bench_variants.sh 4 lg3hp_16x8_q8_f16 lg3hp_w2
