#!/bin/bash
# grid re-check with the final kernel (same box)
O=gpurun_out/g3; mkdir -p $O
B="python bench.py --workload cfg2_sk2000 --steps 3 --warmup 3 --no-e2e --no-cpu"
for rep in 1 2; do
  for g in 98 104 110 116; do
    MARS_UMMA_GRID=$g timeout 300 $B >> $O/grid$g.json 2>> $O/err.log
  done
done
echo done
