#!/bin/bash
# L2 prefetch of the state tiles ahead of the ring (MARS_UMMA_PF chunks) with evict_first tiles
O=gpurun_out/pf; mkdir -p $O
B="python bench.py --workload cfg2_sk2000 --steps 3 --warmup 3 --no-e2e --no-cpu"
for rep in 1 2; do
  for pf in 0 4 8; do
    MARS_UMMA_PF=$pf timeout 300 $B >> $O/pf$pf.json 2>> $O/err.log
  done
done
echo done
