mkdir -p gpurun_out/r6
export PYTHONUNBUFFERED=1
for kk in lg2_16x8_q8_f16 lg2_16x8_q8_f16_w1; do
  MIMO_FORCE_KERNEL=$kk timeout 300 python -m pytest tests/test_parity_gpu.py -x -q -k "config and 4" > gpurun_out/r6/parity4_$kk.log 2>&1; echo "$kk parity rc=$?"; tail -1 gpurun_out/r6/parity4_$kk.log
done
MIMO_FORCE_KERNEL=stream_8x4_q6_i8_b4 timeout 300 python -m pytest tests/test_parity_gpu.py -x -q -k "config and 3" > gpurun_out/r6/parity3.log 2>&1; echo "c3 b4 parity rc=$?"
bash tools/bench_variants.sh 4 lg_16x8_q8_f16 lg2_16x8_q8_f16 lg2_16x8_q8_f16_r3 lg2_16x8_q8_f16_r6 lg2_16x8_q8_f16_w1 lg2_16x8_q8_f16_w4 > gpurun_out/r6/var4.log 2>&1; cat gpurun_out/r6/var4.log
bash tools/bench_variants.sh 3 stream_8x4_q6_i8 stream_8x4_q6_i8_b4 stream_8x4_q6_i8_b5 stream_8x4_q6_i8_g1b4 stream_8x4_q6_i8_g7b6 > gpurun_out/r6/var3.log 2>&1; cat gpurun_out/r6/var3.log
timeout 600 python -m pytest tests/test_accuracy_gpu.py tests/test_lu_route_gpu.py -x -q > gpurun_out/r6/acc.log 2>&1; echo "acc rc=$?"; tail -2 gpurun_out/r6/acc.log
timeout 300 python tools/lu_breakdown.py --reps 20 --out gpurun_out/r6/lu_breakdown > /dev/null 2>&1; cat gpurun_out/r6/lu_breakdown.md
