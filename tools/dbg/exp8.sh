mkdir -p gpurun_out/exp/e8
for n in tbase tnod told tr8 tu80 tbase; do
  PROFLIB=tools/dbg/libmimo_prof_$n.so timeout 120 python tools/dbg/c5time.py
done
for n in tbase tnod tu80; do
  PROFLIB=tools/dbg/libmimo_prof_$n.so timeout 300 ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:k_c5_apply -s 6 -c 4 --csv --log-file gpurun_out/exp/e8/dram_$n.csv python tools/dbg/c5time.py > /dev/null 2>&1
done
timeout 600 python tools/time_varying.py --out gpurun_out/exp/e8/time_varying.jsonl
timeout 600 python -m pytest tests/test_parity_gpu.py -q -x -k "time_varying" > gpurun_out/exp/e8/pytest_tv.log 2>&1
