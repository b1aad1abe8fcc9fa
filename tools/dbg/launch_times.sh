# ncu launch-time list of one C5 kernel variant: tools/dbg/launch_times.sh <kernel> <out>
set -u
python bench.py --config 5 --profile --steps 2 --warmup 1 --kernel $1 > /dev/null 2>&1 || { echo "plain run failed"; exit 1; }
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $2 python bench.py --config 5 --profile --steps 2 --warmup 1 --kernel $1 > /dev/null 2>&1
