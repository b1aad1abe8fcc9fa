mkdir -p gpurun_out/r7
export PYTHONUNBUFFERED=1
for sz in "120 1" "3276 2"; do
  timeout 120 python tools/dbg_size.py big3_64x16_q6_i8 $sz big2_64x16_q6_i8 >> gpurun_out/r7/sizes.log 2>&1 || { echo "FAIL at $sz" >> gpurun_out/r7/sizes.log; break; }
done
grep -v "^big" gpurun_out/r7/sizes.log
MIMO_FORCE_KERNEL=big3_64x16_q6_i8 timeout 600 python -m pytest tests/test_parity_gpu.py -x -q -k "config and 5" > gpurun_out/r7/parity5.log 2>&1; echo "parity5 rc=$?"; tail -1 gpurun_out/r7/parity5.log
bash tools/bench_variants.sh 5 big3_64x16_q6_i8 big2_64x16_q6_i8 > gpurun_out/r7/var5.log 2>&1; cat gpurun_out/r7/var5.log
MIMO_FORCE_KERNEL=big3_64x16_q6_i8 timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/r7/launch_big3.csv python bench.py --config 5 --profile --steps 2 --warmup 1 > gpurun_out/r7/ncu_big3.log 2>&1
MIMO_FORCE_KERNEL=big3_64x16_q6_i8 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_big_apply3 -s 1 -c 1 -o gpurun_out/r7/full_big3 python bench.py --config 5 --profile --steps 2 --warmup 1 > gpurun_out/r7/ncu_full_big3.log 2>&1
