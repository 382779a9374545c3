#!/bin/bash
mkdir -p gpurun_out/s9
B="python bench.py --workload cfg2_sk2000 --steps 1 --warmup 1 --no-e2e --no-cpu --no-clocks"
for pf in 0 8 16; do for g in 148 110 96; do
  v=$(MARS_UMMA_PF=$pf MARS_UMMA_GRID=$g timeout 300 $B 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('%.0f'%d['value'], d['config']['grid'], '%.0f'%d['relax_ms'])")
  echo "pf=$pf grid=$g -> $v" >> gpurun_out/s9/sweep.log
done; done
echo done
