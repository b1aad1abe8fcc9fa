#!/bin/bash
# Tuning experiment on the GPU box: parity + setup-group and apply role profiles of each tuning library.
mkdir -p gpurun_out/exp
for lib in "$@"; do
  echo "=== $lib"
  PROFLIB=$lib timeout 300 python tools/dbg/varcheck.py 2>&1 | tail -2
  PROFLIB=$lib timeout 120 python tools/dbg/c5bprof.py c5_fused_64x16_q6_i8 2>&1 | tail -9
  PROFLIB=$lib timeout 120 python tools/dbg/c5prof.py c5_fused_64x16_q6_i8 2>&1 | tail -21
done
