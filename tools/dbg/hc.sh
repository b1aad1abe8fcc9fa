set -u
out=gpurun_out/${TAG:-hc}; mkdir -p $out
timeout 300 python -m pytest tests/test_variants_gpu.py -x -q -k "fusedhc" > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
tail -3 $out/pytest.log
grep -q "rc=0" $out/pytest.log || exit 1
for k in ${PROFK:-}; do timeout 120 python tools/dbg/c5prof.py $k > $out/roles_$k.txt 2>&1; timeout 120 python tools/dbg/c5bprof.py $k > $out/setup_$k.txt 2>&1; done
for kn in ${KERNELS:-}; do
  timeout 300 python bench.py --config 5 --steps 300 --warmup 20 --no-cpu-baseline --no-e2e --kernel $kn > $out/b_$kn.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$out/b_$kn.json').read().strip().splitlines()[-1]); print('$kn', round(d['ms_per_step']*1e3,2), round(d['roofline']['frac'],4), d['clocks'])"
done
