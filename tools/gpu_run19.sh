mkdir -p gpurun_out/r19
timeout 120 python tools/dbg_size.py big5_64x16_q6_i8 120 1 big2_64x16_q6_i8 2>&1 | grep -v "^big"
timeout 120 python tools/dbg_size.py big5_64x16_q6_i8 3276 4 big2_64x16_q6_i8 2>&1 | grep -v "^big"
for k in big5_64x16_q6_i8 big5s3_64x16_q6_i8 ablation_big5_none big4_64x16_q6_i8; do
  MIMO_FORCE_KERNEL=$k timeout 300 python bench.py --config 5 --profile --steps 1 --warmup 1 > /dev/null 2>&1 || { echo "plain failed $k"; continue; }
  MIMO_FORCE_KERNEL=$k timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/r19/launch_$k.csv python bench.py --config 5 --profile --steps 1 --warmup 1 > /dev/null 2>&1
  echo "== $k $(grep k_big_apply4 gpurun_out/r19/launch_$k.csv | head -2 | awk -F'","' '{print $15}' | tr '\n' ' ')"
done
