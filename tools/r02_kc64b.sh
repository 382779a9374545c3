#!/bin/bash
# with 64-element K stages the helper binds: rebalance (kc64 = mma helper takes every rectangle,
# kc64f = + walker fold, kc64c = CUDA-core helper + fold)
O=gpurun_out/kcb; mkdir -p $O
for v in kc64f kc64c; do
  MARS_HANG_S=30 MARS_B200_LIB=libmars_b200_$v.so timeout 900 python -m pytest tests/test_gpu_trajectory.py -x -q -k "single_sweep or cfg2_prefix" > $O/pytest_$v.log 2>&1; echo "rc=$?" >> $O/pytest_$v.log
done
B="python bench.py --workload cfg2_sk2000 --steps 3 --warmup 3 --no-e2e --no-cpu"
for rep in 1 2; do
  for v in kc64 kc64f kc64c; do
    MARS_HANG_S=30 MARS_B200_LIB=libmars_b200_$v.so timeout 300 $B >> $O/cfg2_$v.json 2>> $O/err.log
  done
done
for v in kc64f kc64c; do
  MARS_B200_LIB=libmars_b200_$v.so MARS_PROFILE=1 timeout 300 python bench.py --workload cfg2_sk2000 --steps 1 --warmup 1 --no-e2e --no-cpu --no-clocks > $O/prof_$v.json 2> $O/prof_$v.err
done
echo done
