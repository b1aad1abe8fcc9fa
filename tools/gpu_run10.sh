mkdir -p gpurun_out/r10
export PYTHONUNBUFFERED=1
timeout 120 python tools/dbg_size.py big4_64x16_q6_i8 3276 4 big2_64x16_q6_i8 > gpurun_out/r10/sizes.log 2>&1 || echo FAIL >> gpurun_out/r10/sizes.log
grep -v "^big" gpurun_out/r10/sizes.log
bash tools/bench_variants.sh 5 big4_64x16_q6_i8 > gpurun_out/r10/var5.log 2>&1; cat gpurun_out/r10/var5.log
MIMO_FORCE_KERNEL=big4_64x16_q6_i8 timeout 300 ncu --metrics gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/r10/launch_big4.csv python bench.py --config 5 --profile --steps 1 --warmup 1 > gpurun_out/r10/ncu_big4.log 2>&1
grep -h "k_big_apply4" gpurun_out/r10/launch_big4.csv | head -4 | cut -c1-250
