mkdir -p gpurun_out/r15
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "config and (4 or 5)" > gpurun_out/r15/parity45.log 2>&1; echo "parity45 rc=$?"; tail -1 gpurun_out/r15/parity45.log
bash tools/bench_variants.sh 4 lg3_16x8_q8_f16 > gpurun_out/r15/var4.log 2>&1; cat gpurun_out/r15/var4.log
bash tools/bench_variants.sh 5 big4_64x16_q6_i8 > gpurun_out/r15/var5.log 2>&1; cat gpurun_out/r15/var5.log
MIMO_FORCE_KERNEL=big4_64x16_q6_i8 timeout 300 ncu --metrics gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/r15/launch5.csv python bench.py --config 5 --profile --steps 1 --warmup 1 > /dev/null 2>&1
grep "k_big_setup" gpurun_out/r15/launch5.csv | head -3 | awk -F'","' '{print $13, $15}'
