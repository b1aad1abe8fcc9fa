mkdir -p gpurun_out/r4
timeout 120 python tools/dbg_tc.py big2_64x16_q6_i8 > gpurun_out/r4/dbg_big2.log 2>&1
cat gpurun_out/r4/dbg_big2.log | head -3
MIMO_FORCE_KERNEL=big2_64x16_q6_i8 timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "config and 5" > gpurun_out/r4/parity5.log 2>&1; tail -2 gpurun_out/r4/parity5.log
bash tools/bench_variants.sh 5 big_64x16_q6_i8 big2_64x16_q6_i8 > gpurun_out/r4/var5.log 2>&1; cat gpurun_out/r4/var5.log
for k in big_64x16_q6_i8 big2_64x16_q6_i8; do
  MIMO_FORCE_KERNEL=$k timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/r4/launch_$k.csv python bench.py --config 5 --profile --steps 2 --warmup 1 > gpurun_out/r4/ncu_$k.log 2>&1
done
timeout 300 python tools/lu_breakdown.py --reps 30 > gpurun_out/r4/lu_breakdown.log 2>&1; tail -20 gpurun_out/r4/lu_breakdown.log
cp profiles/r01/lu_breakdown.* gpurun_out/r4/ 2>/dev/null
