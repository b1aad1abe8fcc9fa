mkdir -p gpurun_out/exp/e12
for v in v0 v4 v0 v4; do PROFLIB=tools/dbg/libmimo_prof_$v.so timeout 120 python tools/dbg/c5time.py; done
PROFLIB=tools/dbg/libmimo_prof_v4.so timeout 300 python tools/dbg/varcheck.py 2>&1 | tail -1 | cut -c1-250
timeout 900 python -m pytest tests/test_variants_gpu.py tests/test_edge_gpu.py tests/test_parity_gpu.py tests/test_shard_gpu.py tests/test_api_gpu.py -q -x -k "5 or c5 or C5" > gpurun_out/exp/e12/pytest.log 2>&1; tail -2 gpurun_out/exp/e12/pytest.log
for v in v0 v4 v0 v4; do
  cp tools/dbg/libmimo_prof_$v.so paper_2510_07843_b200/lib/libmimo.so
  timeout 300 python bench.py --steps 4000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/exp/e12/bench_$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/exp/e12/bench_$v.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step']*1e3,1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
