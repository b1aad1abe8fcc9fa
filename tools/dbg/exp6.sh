mkdir -p gpurun_out/exp
for kn in lg3hp_16x8_q8_f16 lg3hq_16x8_q8_f16; do
  timeout 300 python bench.py --config 4 --kernel $kn --steps 400 --warmup 20 > gpurun_out/exp/exp6_$kn.json 2> gpurun_out/exp/exp6_$kn.err
done
timeout 600 python -m pytest tests/test_variants_gpu.py -q -x -k "C4 or c4 or 4" > gpurun_out/exp/exp6_pytest.log 2>&1
