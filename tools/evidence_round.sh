#!/bin/bash
# Round-end evidence in one gpurun call: GPU suite, smoke, bench lines of every config (+ emulated
# scaling, BFP e2e, reference arm), then the ncu captures of tools/profile_round.sh.
# Usage: tools/evidence_round.sh <tag>   (outputs under gpurun_out/ev_<tag>/ and gpurun_out/prof_<tag>/)
set -u
tag=${1:-r02}
out=gpurun_out/ev_$tag; mkdir -p $out
timeout 900 python -m pytest tests -m gpu -q > $out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > $out/smoke.log 2>&1
timeout 1500 python bench.py --config all --emulate 2 4 8 > $out/bench_all.jsonl 2> $out/bench_all.err
timeout 300 python bench.py > $out/bench_default.json 2> $out/bench_default.err
timeout 300 python bench.py --config 3 --bfp 9 > $out/bench_c3_bfp9.json 2> $out/bench_c3_bfp9.err
timeout 300 python bench.py --impl reference --steps 5 --warmup 3 > $out/bench_reference.json 2> $out/bench_reference.err
bash tools/profile_round.sh $tag
ls -la $out
