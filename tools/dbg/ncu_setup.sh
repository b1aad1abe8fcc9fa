set -u
out=gpurun_out/$1; mkdir -p $out
python bench.py --config 5 --profile --steps 2 --warmup 1 > /dev/null 2>&1 || exit 1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:${2:-k_c5_setup} -s 1 -c 1 -o $out/full python bench.py --config 5 --profile --steps 2 --warmup 1 > $out/ncu.log 2>&1
