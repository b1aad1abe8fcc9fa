mkdir -p gpurun_out/r11
export PYTHONUNBUFFERED=1
for kk in big4_64x16_q6_i8 big4e8_64x16_q6_i8 big4s6_64x16_q6_i8 big4e8s6_64x16_q6_i8; do
  timeout 120 python tools/dbg_size.py $kk 3276 4 big2_64x16_q6_i8 > gpurun_out/r11/sizes_$kk.log 2>&1 || echo "FAIL $kk" >> gpurun_out/r11/sizes_$kk.log
  grep -v "^big" gpurun_out/r11/sizes_$kk.log
done
bash tools/bench_variants.sh 5 big4_64x16_q6_i8 big4e8_64x16_q6_i8 big4s6_64x16_q6_i8 big4e8s6_64x16_q6_i8 big4s4_64x16_q6_i8 > gpurun_out/r11/var5.log 2>&1; cat gpurun_out/r11/var5.log
