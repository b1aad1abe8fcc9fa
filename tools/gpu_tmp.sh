#!/bin/bash
timeout 400 python bench.py 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['cpu_baseline'])"
