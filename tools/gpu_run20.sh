mkdir -p gpurun_out/r20
timeout 120 python tools/dbg_size.py big5_64x16_q6_i8 3276 4 big2_64x16_q6_i8 2>&1 | grep -v "^big"
for k in big5_64x16_q6_i8 big4_64x16_q6_i8; do
  MIMO_FORCE_KERNEL=$k timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/r20/launch_$k.csv python bench.py --config 5 --profile --steps 1 --warmup 1 > /dev/null 2>&1
  echo "== $k $(grep k_big_apply4 gpurun_out/r20/launch_$k.csv | head -2 | awk -F'","' '{print $15}' | tr '\n' ' ')"
done
bash tools/bench_variants.sh 4 lg3_16x8_q8_f16 lg3_16x8_q8_f16_pf518 lg3_16x8_q8_f16_pf1036 lg3_16x8_q8_f16_pf2072 > gpurun_out/r20/var4.log 2>&1; cat gpurun_out/r20/var4.log
