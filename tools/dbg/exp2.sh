mkdir -p gpurun_out/exp
bash tools/dbg/exp.sh tools/dbg/libmimo_prof.so tools/dbg/libmimo_prof_gj3.so > gpurun_out/exp/exp2.log 2>&1
timeout 600 python -m pytest tests/test_variants_gpu.py tests/test_edge_gpu.py tests/test_parity_gpu.py -q -x -k "c5 or C5 or 5" > gpurun_out/exp/exp2_pytest.log 2>&1
timeout 300 python bench.py --steps 200 --warmup 20 > gpurun_out/exp/exp2_bench.json 2> gpurun_out/exp/exp2_bench.err
