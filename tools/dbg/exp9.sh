mkdir -p gpurun_out/exp/e9
for n in tt1 tt0 tc4 tc8 tt1 tt0; do
  PROFLIB=tools/dbg/libmimo_prof_$n.so timeout 120 python tools/dbg/c5time.py
done
PROFLIB=tools/dbg/libmimo_prof_tt1.so timeout 300 python tools/dbg/varcheck.py 2>&1 | tail -1 | cut -c1-250
bash tools/dbg/exp.sh tools/dbg/libmimo_prof.so
