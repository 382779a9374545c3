#!/bin/bash
# 64-element K stages with SWIZZLE_128B (kc64, 3 x 48 KB) vs 32-element SW64 stages (6 x 24 KB)
O=gpurun_out/kc; mkdir -p $O
MARS_HANG_S=30 MARS_B200_LIB=libmars_b200_kc64.so timeout 900 python -m pytest tests/test_gpu_trajectory.py -x -q -k "single_sweep or cfg2_prefix" > $O/pytest_kc64.log 2>&1; echo "rc=$?" >> $O/pytest_kc64.log
B="python bench.py --workload cfg2_sk2000 --steps 3 --warmup 3 --no-e2e --no-cpu"
for rep in 1 2; do
  for v in libmars_b200_kc64.so libmars_b200.so; do
    MARS_HANG_S=30 MARS_B200_LIB=$v timeout 300 $B >> $O/cfg2_$v.json 2>> $O/err.log
  done
done
MARS_B200_LIB=libmars_b200_kc64.so MARS_PROFILE=1 timeout 300 python bench.py --workload cfg2_sk2000 --steps 1 --warmup 1 --no-e2e --no-cpu --no-clocks > $O/prof_kc64.json 2> $O/prof_kc64.err
echo done
