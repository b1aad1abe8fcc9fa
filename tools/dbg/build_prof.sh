#!/bin/bash
# Tuning build: libmimo with -DC5_PROFILE (per-role cycle accounting in k_c5.cu) and extra -D flags
# ($1) -> tools/dbg/libmimo_prof${2}.so
set -e
PROFDEF=${PROFDEF--DC5_PROFILE}  # PROFDEF= (empty) for a timing build without the cycle counters
cd "$(dirname "$0")/../.."
C=paper_2510_07843_b200/csrc
od=tools/dbg/obj$2
mkdir -p $od
for f in $C/*.cu; do
  o=$od/$(basename $f .cu).o
  tgt=${PROFFILE:-k_c5.cu}  # the file the extra flags apply to
  if [ "$(basename $f)" = "$tgt" ]; then extra="$PROFDEF $1"; else extra=; fi
  if [ "$(basename $f)" != "$tgt" ] && [ -f tools/dbg/obj/$(basename $f .cu).o ] && [ "$od" != "tools/dbg/obj" ]; then cp tools/dbg/obj/$(basename $f .cu).o $o; continue; fi
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Xcompiler -fPIC --expt-relaxed-constexpr -Iinclude -I$C $extra -c $f -o $o &
done
wait
nvcc -gencode arch=compute_100a,code=sm_100a -shared -cudart=static -Xcompiler -fPIC -o tools/dbg/libmimo_prof$2.so $od/*.o
