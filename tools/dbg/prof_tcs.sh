set -u
out=gpurun_out/g6; mkdir -p $out
python bench.py --config 5 --profile --steps 2 --warmup 1 --kernel c5_bf16_tcs_64x16_q6_i8 > $out/plain.log 2>&1 || exit 1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_c5_setup -s 1 -c 1 -o $out/tcs python bench.py --config 5 --profile --steps 2 --warmup 1 --kernel c5_bf16_tcs_64x16_q6_i8 > $out/ncu1.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_c5_apply -s 1 -c 1 -o $out/apply python bench.py --config 5 --profile --steps 2 --warmup 1 > $out/ncu2.log 2>&1
ls -la $out
