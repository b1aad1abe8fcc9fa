mkdir -p gpurun_out
(timeout 120 python tools/dbg_tc.py bigtc3_64x16_q6_i8; timeout 120 python tools/dbg_tc.py bigtc2_64x16_q6_i8) > gpurun_out/dbg_tc.log 2>&1
bash tools/bench_variants.sh 5 big_64x16_q6_i8 bigtc3_64x16_q6_i8 bigtc2_64x16_q6_i8 > gpurun_out/var5.log 2>&1
bash tools/bench_variants.sh 4 lg_16x8_q8_f16 lg_16x8_q8_f16_w1 lg_16x8_q8_f16_w4 > gpurun_out/var4.log 2>&1
cat gpurun_out/dbg_tc.log gpurun_out/var5.log gpurun_out/var4.log
