mkdir -p gpurun_out/r9
MIMO_FORCE_KERNEL=big4_64x16_q6_i8 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_big_apply4 -s 1 -c 1 -o gpurun_out/r9/full_big4 python bench.py --config 5 --profile --steps 2 --warmup 1 > gpurun_out/r9/ncu_full_big4.log 2>&1
tail -3 gpurun_out/r9/ncu_full_big4.log
