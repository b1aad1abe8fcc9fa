mkdir -p gpurun_out/r17
for k in big4_64x16_q6_i8 big4s5_64x16_q6_i8 big4s6_64x16_q6_i8 big4s3_64x16_q6_i8 big4e8_64x16_q6_i8; do
  MIMO_FORCE_KERNEL=$k timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r17/launch_$k.csv python bench.py --config 5 --profile --steps 1 --warmup 1 > /dev/null 2>&1
  echo "== $k $(grep k_big_apply4 gpurun_out/r17/launch_$k.csv | head -1 | awk -F'","' '{print $15}')"
done
