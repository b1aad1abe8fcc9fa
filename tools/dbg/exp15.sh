mkdir -p gpurun_out/exp/e15
for k in stream_8x4_q6_i8 stream_8x4_q6_i8_g3 stream_8x4_q6_i8_g4 stream_8x4_q6_i8 stream_8x4_q6_i8_g3 stream_8x4_q6_i8_g4; do
  timeout 300 python bench.py --config 3 --kernel $k --steps 4000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/exp/e15/b_$k.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/exp/e15/b_$k.json').read().strip().splitlines()[-1]); print('$k', round(d['ms_per_step']*1e3,2), d['roofline']['frac'], d['clocks']['sm_mhz'])"
done
timeout 600 python -m pytest tests/test_variants_gpu.py -q -x -k "3" > gpurun_out/exp/e15/pytest.log 2>&1; tail -1 gpurun_out/exp/e15/pytest.log
