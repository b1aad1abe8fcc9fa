mkdir -p gpurun_out/r14
timeout 120 python tools/dbg_size.py big4_64x16_q6_i8 3276 4 big2_64x16_q6_i8 2>&1 | grep -v "^big"
for k in big4_64x16_q6_i8 ablation_big4_none; do
  MIMO_FORCE_KERNEL=$k timeout 300 python bench.py --config 5 --profile --steps 1 --warmup 1 > /dev/null 2>&1 || { echo "plain failed $k"; continue; }
  MIMO_FORCE_KERNEL=$k timeout 300 ncu --metrics gpu__time_duration.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,dram__throughput.avg.pct_of_peak_sustained_elapsed --clock-control none --csv --log-file gpurun_out/r14/launch_$k.csv python bench.py --config 5 --profile --steps 1 --warmup 1 > /dev/null 2>&1
  echo "== $k"; grep "k_big_apply4" gpurun_out/r14/launch_$k.csv | head -4 | awk -F'","' '{print $13, $15}'
done
bash tools/bench_variants.sh 5 big4_64x16_q6_i8 > gpurun_out/r14/var5.log 2>&1; cat gpurun_out/r14/var5.log
