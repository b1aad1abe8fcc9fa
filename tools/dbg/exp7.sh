mkdir -p gpurun_out/exp
for lib in tools/dbg/libmimo_prof.so tools/dbg/libmimo_prof_h1.so tools/dbg/libmimo_prof_r32.so tools/dbg/libmimo_prof_u80.so; do
  echo "=== $lib"
  PROFLIB=$lib timeout 300 python tools/dbg/varcheck.py 2>&1 | tail -1 | cut -c1-200
  PROFLIB=$lib timeout 120 python tools/dbg/c5bprof.py c5_fused_64x16_q6_i8 2>&1 | tail -8
  PROFLIB=$lib timeout 120 python tools/dbg/c5prof.py c5_fused_64x16_q6_i8 2>&1 | tail -21
  PROFLIB=$lib timeout 300 ncu --cache-control none --clock-control none --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum -k regex:k_c5_apply -s 6 -c 3 --csv python tools/dbg/c5prof.py c5_fused_64x16_q6_i8 2>/dev/null | grep -E "dram__|gpu__time" | cut -c1-220
done
for kn in lg3hq_16x8_q8_f16 lg3hl_16x8_q8_f16 lg3hl2_16x8_q8_f16; do
  timeout 300 python bench.py --config 4 --kernel $kn --steps 400 --warmup 20 > gpurun_out/exp/exp7_$kn.json 2> gpurun_out/exp/exp7_$kn.err
done
timeout 600 python -m pytest tests/test_variants_gpu.py -q -x -k "C4 or c4 or 4" > gpurun_out/exp/exp7_pytest.log 2>&1
