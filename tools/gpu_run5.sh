mkdir -p gpurun_out/r5
for sz in "120 1" "1200 1" "3276 1" "3276 4" "3276 40"; do
  timeout 120 python tools/dbg_size.py big2_64x16_q6_i8 $sz >> gpurun_out/r5/sizes.log 2>&1 || { echo "FAIL at $sz" >> gpurun_out/r5/sizes.log; break; }
done
cat gpurun_out/r5/sizes.log | grep -v "^big"
bash tools/bench_variants.sh 5 big2_64x16_q6_i8 big_64x16_q6_i8 > gpurun_out/r5/var5.log 2>&1; cat gpurun_out/r5/var5.log
for k in big_64x16_q6_i8 big2_64x16_q6_i8; do
  MIMO_FORCE_KERNEL=$k timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum --clock-control none --csv --log-file gpurun_out/r5/launch_$k.csv python bench.py --config 5 --profile --steps 2 --warmup 1 > gpurun_out/r5/ncu_$k.log 2>&1
done
