mkdir -p gpurun_out/r3
cd $GRAFT_REPO_ROOT
python - <<'PY'
# pre-generate nothing; just check LU route quickly first
PY
timeout 600 python -m pytest tests/test_lu_route_gpu.py -x -q -s > gpurun_out/r3/lu_tests.log 2>&1; echo "lu tests rc=$?"
for k in big_64x16_q6_i8 bigtc2_64x16_q6_i8 bigtc3_64x16_q6_i8; do
  MIMO_FORCE_KERNEL=$k timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/r3/launch_$k.csv python bench.py --config 5 --profile --steps 2 --warmup 1 > gpurun_out/r3/ncu_$k.log 2>&1
done
MIMO_FORCE_KERNEL=bigtc2_64x16_q6_i8 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_big_tc2 -s 1 -c 1 -o gpurun_out/r3/full_tc2 python bench.py --config 5 --profile --steps 2 --warmup 1 > gpurun_out/r3/ncu_full_tc2.log 2>&1
tail -5 gpurun_out/r3/lu_tests.log
