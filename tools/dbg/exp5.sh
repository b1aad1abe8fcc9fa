mkdir -p gpurun_out/exp
bash tools/dbg/exp.sh tools/dbg/libmimo_prof.so > gpurun_out/exp/exp5.log 2>&1
timeout 600 python -m pytest tests/test_variants_gpu.py tests/test_edge_gpu.py tests/test_parity_gpu.py tests/test_shard_gpu.py tests/test_api_gpu.py -q -x > gpurun_out/exp/exp5_pytest.log 2>&1
timeout 300 python bench.py --steps 200 --warmup 20 > gpurun_out/exp/exp5_bench.json 2> gpurun_out/exp/exp5_bench.err
mkdir -p gpurun_out/exp/rng
timeout 600 ncu --profile-from-start off --cache-control none --clock-control none --csv --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --log-file gpurun_out/exp/rng/range_c5.csv python tools/traffic_range.py --config 5 --steps 8 > gpurun_out/exp/rng/ncu.log 2>&1
