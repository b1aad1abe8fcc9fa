set -u
out=gpurun_out/g9; mkdir -p $out
K=${K:-c5_bf16_tcs_64x16_q6_i8}
python bench.py --config 5 --profile --steps 2 --warmup 1 --kernel $K > $out/plain.log 2>&1 || exit 1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $out/launches.csv python bench.py --config 5 --profile --steps 2 --warmup 1 --kernel $K > $out/ncu0.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_c5_setup -s 1 -c 1 -o $out/tcs python bench.py --config 5 --profile --steps 2 --warmup 1 --kernel $K > $out/ncu1.log 2>&1
ls -la $out
