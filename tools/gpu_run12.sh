mkdir -p gpurun_out/r12
export PYTHONUNBUFFERED=1
for kk in lg3_16x8_q8_f16 lg3_16x8_q8_f16_w1; do
  MIMO_FORCE_KERNEL=$kk timeout 300 python -m pytest tests/test_parity_gpu.py -x -q -k "config and 4" > gpurun_out/r12/parity4_$kk.log 2>&1; echo "$kk parity rc=$?"; tail -1 gpurun_out/r12/parity4_$kk.log
done
bash tools/bench_variants.sh 4 lg_16x8_q8_f16 lg3_16x8_q8_f16 lg3_16x8_q8_f16_w1 lg3_16x8_q8_f16_w4 > gpurun_out/r12/var4.log 2>&1; cat gpurun_out/r12/var4.log
MIMO_FORCE_KERNEL=big4_64x16_q6_i8 timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "5" > gpurun_out/r12/parity5.log 2>&1; echo "big4 parity rc=$?"; tail -1 gpurun_out/r12/parity5.log
