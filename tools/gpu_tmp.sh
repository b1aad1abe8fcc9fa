MIMO_FORCE_KERNEL=lg3h_16x8_q8_f16 timeout 300 python -m pytest tests/test_parity_gpu.py -x -q -k "config and 4" 2>&1 | tail -1
bash tools/bench_variants.sh 4 lg3_16x8_q8_f16 lg3h_16x8_q8_f16 2>&1
