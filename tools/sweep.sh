#!/bin/bash
# Tuning sweep of bench.py over environment overrides (kernel launch shapes); one line per setting.
# usage: sweep.sh workload "ENV=.. ENV=.." ...
w=$1; shift
for cfg in "$@"; do
  v=$(env $cfg timeout 300 python bench.py --workload $w --steps 1 --warmup 1 --no-e2e --no-cpu --no-clocks 2>/dev/null | python -c "import json,sys
for l in sys.stdin:
    if l.startswith('{'): d=json.loads(l); print('%.1f'%d['value'], d['config']['grid'], d['config']['slots'], '%.1f'%d['ms_per_step'])")
  echo "$w [$cfg] $v"
done
