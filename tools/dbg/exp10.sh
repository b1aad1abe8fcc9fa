mkdir -p gpurun_out/exp/e10
cp paper_2510_07843_b200/lib/libmimo.so /tmp/libmimo_main.so
for v in v0 v1 v2 v3 v0 v1; do
  cp tools/dbg/libmimo_prof_$v.so paper_2510_07843_b200/lib/libmimo.so
  timeout 300 python bench.py --steps 4000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/exp/e10/bench_$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/exp/e10/bench_$v.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step']*1e3,1), d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
cp /tmp/libmimo_main.so paper_2510_07843_b200/lib/libmimo.so
