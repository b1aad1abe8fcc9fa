mkdir -p gpurun_out/r8
export PYTHONUNBUFFERED=1
for sz in "120 1" "3276 2" "3276 40"; do
  timeout 120 python tools/dbg_size.py big4_64x16_q6_i8 $sz big2_64x16_q6_i8 >> gpurun_out/r8/sizes.log 2>&1 || { echo "FAIL at $sz" >> gpurun_out/r8/sizes.log; break; }
done
grep -v "^big" gpurun_out/r8/sizes.log
if ! grep -q FAIL gpurun_out/r8/sizes.log; then
MIMO_FORCE_KERNEL=big4_64x16_q6_i8 timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "config and 5" > gpurun_out/r8/parity5.log 2>&1; echo "parity5 rc=$?"; tail -1 gpurun_out/r8/parity5.log
bash tools/bench_variants.sh 5 big4_64x16_q6_i8 big3_64x16_q6_i8 > gpurun_out/r8/var5.log 2>&1; cat gpurun_out/r8/var5.log
MIMO_FORCE_KERNEL=big4_64x16_q6_i8 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/r8/launch_big4.csv python bench.py --config 5 --profile --steps 2 --warmup 1 > gpurun_out/r8/ncu_big4.log 2>&1
fi
for kk in lg2_16x8_q8_f16_r14s2 lg2_16x8_q8_f16_r14s2w1; do
  MIMO_FORCE_KERNEL=$kk timeout 300 python -m pytest tests/test_parity_gpu.py -x -q -k "config and 4" > gpurun_out/r8/parity4_$kk.log 2>&1; echo "$kk parity rc=$?"
done
bash tools/bench_variants.sh 4 lg_16x8_q8_f16 lg2_16x8_q8_f16_r14 lg2_16x8_q8_f16_r14s2 lg2_16x8_q8_f16_r14s2w1 > gpurun_out/r8/var4.log 2>&1; cat gpurun_out/r8/var4.log
