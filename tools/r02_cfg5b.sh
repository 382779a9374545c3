#!/bin/bash
# cfg5 full batches (8192 descents, N = 16384): default split 2 over 8192 slots, and split 4
# over 15 tiles (3840 slots: runs queue longest-first, the fast tiles take two runs each)
mkdir -p gpurun_out/c5b
B="python bench.py --workload cfg5_sk16384 --steps 1 --warmup 0 --no-e2e --no-cpu"
MARS_UMMA_DEBUG=1 timeout 1500 $B > gpurun_out/c5b/split2.json 2> gpurun_out/c5b/split2.err
MARS_UMMA_DEBUG=1 MARS_UMMA_SPLIT=4 MARS_UMMA_GRID=30 timeout 1500 $B > gpurun_out/c5b/split4_g30.json 2> gpurun_out/c5b/split4_g30.err
echo done
