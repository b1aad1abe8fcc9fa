set -u
out=gpurun_out/${TAG:-bi3}; mkdir -p $out
timeout 600 python -m pytest tests/test_variants_gpu.py -x -q -k "fusedbi" > $out/pytest.log 2>&1; echo "rc=$?" >> $out/pytest.log
tail -2 $out/pytest.log
for kn in ${KERNELS:-}; do
  timeout 300 python bench.py --config 5 --steps 300 --warmup 20 --no-cpu-baseline --no-e2e --kernel $kn > $out/b_$kn.json 2>/dev/null
  python -c "
import json; d=json.loads(open('$out/b_$kn.json').read().strip().splitlines()[-1]); print('$kn', round(d['ms_per_step']*1e3,2), round(d['roofline']['frac'],4), d['clocks']['sm_mhz'])"
done
for kn in ${TRAFFIC:-}; do
  timeout 600 ncu --profile-from-start off --cache-control none --clock-control none --csv \
      --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
      --log-file $out/range_$kn.csv python tools/traffic_range.py --config 5 --steps 8 --kernel $kn > $out/ncu_range_$kn.log 2>&1
  python - <<PY
import csv
rows=[r for r in csv.reader(open('$out/range_$kn.csv')) if len(r)>5]
hdr=rows[0]; idx={n:i for i,n in enumerate(hdr)}
tot={}
for r in rows[1:]:
    m=r[idx['Metric Name']]; v=float(r[idx['Metric Value']].replace(',',''))
    u=r[idx['Metric Unit']]
    scale={'byte':1,'Kbyte':1e3,'Mbyte':1e6,'Gbyte':1e9,'KB':1e3,'MB':1e6,'GB':1e9}.get(u,1)
    tot.setdefault(m,[]).append(v*scale)
for m,v in tot.items(): print('$kn', m, 'per launch mean', sum(v[1:])/max(1,len(v)-1))
PY
done
