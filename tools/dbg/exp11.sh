mkdir -p gpurun_out/exp/e11
for kn in stream_8x4_q6_i8 stream_8x4_q6_i8f stream_8x4_q6_i8 stream_8x4_q6_i8f; do
  timeout 300 python bench.py --config 3 --kernel $kn --steps 4000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/exp/e11/b_$kn.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/exp/e11/b_$kn.json').read().strip().splitlines()[-1]); print('$kn', round(d['ms_per_step']*1e3,2), d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
timeout 600 python -m pytest tests/test_variants_gpu.py tests/test_edge_gpu.py -q -x > gpurun_out/exp/e11/pytest.log 2>&1; tail -2 gpurun_out/exp/e11/pytest.log
