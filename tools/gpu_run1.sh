set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py > gpurun_out/bench_default.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/bench_default.log
bash tools/bench_variants.sh 5 big_64x16_q6_i8 bigtc3_64x16_q6_i8 bigtc2_64x16_q6_i8 bigtc_64x16_q6_i8 > gpurun_out/var5.log 2>&1
cat gpurun_out/var5.log
for k in 1 3 4; do timeout 300 python bench.py --config $k --no-e2e --no-cpu-baseline | tail -1; done > gpurun_out/bench_cfgs.log 2>&1
cat gpurun_out/bench_cfgs.log
