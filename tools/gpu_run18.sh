mkdir -p gpurun_out/r18
for k in ablation_big4_none ablation_big4_mma1; do
  MIMO_FORCE_KERNEL=$k timeout 300 ncu --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/r18/launch_$k.csv python bench.py --config 5 --profile --steps 1 --warmup 1 > /dev/null 2>&1
  echo "== $k $(grep k_big_apply4 gpurun_out/r18/launch_$k.csv | head -2 | awk -F'","' '{print $15}' | tr '\n' ' ')"
done
