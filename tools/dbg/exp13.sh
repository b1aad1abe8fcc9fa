mkdir -p gpurun_out/exp/e13
for k in c5_fused_64x16_q6_i8 c5_fused3_64x16_q6_i8 c5_fused_64x16_q6_i8 c5_fused3_64x16_q6_i8; do PROFLIB=tools/dbg/libmimo_prof_v5.so timeout 120 python tools/dbg/c5time.py $k; done
timeout 900 python -m pytest tests/test_variants_gpu.py tests/test_edge_gpu.py -q -x -k "5 or c5 or C5" > gpurun_out/exp/e13/pytest.log 2>&1; tail -2 gpurun_out/exp/e13/pytest.log
for k in c5_fused_64x16_q6_i8 c5_fused3_64x16_q6_i8 c5_fused_64x16_q6_i8 c5_fused3_64x16_q6_i8; do
  timeout 300 python bench.py --kernel $k --steps 4000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/exp/e13/bench_$k.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/exp/e13/bench_$k.json').read().strip().splitlines()[-1]); print('$k', round(d['ms_per_step']*1e3,1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
