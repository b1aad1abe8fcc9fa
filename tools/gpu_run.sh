#!/bin/bash
# generic round-2 GPU session: tests, then C5 bench lines per kernel variant
set -u
out=gpurun_out/${TAG:-g}; mkdir -p $out
timeout 900 python -m pytest ${PYARGS:-tests} -m gpu -x -q > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/pytest.log
for kn in ${KERNELS:-}; do
  timeout 300 python bench.py --config 5 --steps 200 --warmup 20 --no-cpu-baseline --no-e2e --kernel $kn > $out/bench_$kn.json 2> $out/bench_$kn.err
done
