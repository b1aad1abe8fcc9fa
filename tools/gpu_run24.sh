for G in 1 2 7 14; do
  MIMO_BFP_G=$G timeout 300 python bench.py --config 3 --bfp 9 --no-e2e --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('G', $G, round(d['roofline']['step_us'],2), 'us', round(d['roofline']['frac'],3))"
done
