mkdir -p gpurun_out/r23
export PYTHONUNBUFFERED=1
timeout 600 python -m pytest tests/test_bfp_gpu.py -q -s 2>&1 | tail -8
timeout 300 python bench.py --config 3 --bfp 9 --no-e2e --no-cpu-baseline > gpurun_out/r23/bench_c3_bfp9.json 2>&1; tail -1 gpurun_out/r23/bench_c3_bfp9.json | cut -c1-1500
