set -u
out=gpurun_out/${TAG:-t1}; mkdir -p $out
for kn in c5_fusedt1y_64x16_q6_i8 c5_fusedt1x_64x16_q6_i8; do
  timeout 300 python -m pytest tests/test_variants_gpu.py -x -q -k "$kn" > $out/pytest_$kn.log 2>&1; echo "rc=$?" >> $out/pytest_$kn.log
  echo $kn; tail -2 $out/pytest_$kn.log
done
for kn in ${KERNELS:-}; do
  timeout 300 python bench.py --config 5 --steps 300 --warmup 20 --no-cpu-baseline --no-e2e --kernel $kn > $out/b_$kn.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$out/b_$kn.json').read().strip().splitlines()[-1]); c=d['clocks']; print('$kn', round(d['ms_per_step']*1e3,2), round(d['roofline']['frac'],4), c['sm_mhz'], c.get('power_w'), round(d['ms_per_step']*1e3*c['sm_mhz']/1e3,1),'kcyc')" 2>/dev/null || echo "$kn bench failed"
done
