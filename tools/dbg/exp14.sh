mkdir -p gpurun_out/exp/e14
for v in c4m1 c4m6 c4m7 c4m1 c4m6 c4m7; do
  cp tools/dbg/libmimo_prof_$v.so paper_2510_07843_b200/lib/libmimo.so
  timeout 300 python bench.py --config 4 --steps 4000 --warmup 50 --no-cpu-baseline --no-e2e > gpurun_out/exp/e14/bench_$v.json 2>/dev/null
  python -c "
import json; d=json.loads(open('gpurun_out/exp/e14/bench_$v.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step']*1e3,2), d['roofline']['frac'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
done
