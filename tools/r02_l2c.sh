#!/bin/bash
# same-box cfg2: grid sweep with the evict_first state tiles, and the coupling-tile policy
mkdir -p gpurun_out/l2c
B="python bench.py --workload cfg2_sk2000 --steps 3 --warmup 3 --no-e2e --no-cpu"
run() { timeout 300 env "$@" $B >> gpurun_out/l2c/$(echo "$@" | tr ' =' '__').json 2>> gpurun_out/l2c/err.log; }
run MARS_BASE=1
run MARS_UMMA_GRID=92
run MARS_UMMA_GRID=104
run MARS_UMMA_GRID=110
run MARS_UMMA_JPOL=0
run MARS_UMMA_SPOL=2 MARS_UMMA_JPOL=2
run MARS_BASE=2
echo done
