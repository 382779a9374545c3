#!/bin/bash
# walker-bound default: hoisting the fold's coupling loads (ho) vs not
O=gpurun_out/ho; mkdir -p $O
MARS_B200_LIB=libmars_b200_ho.so timeout 900 python -m pytest tests/test_gpu_trajectory.py -x -q -k "single_sweep or cfg2_prefix" > $O/pytest_ho.log 2>&1; echo "rc=$?" >> $O/pytest_ho.log
B="python bench.py --workload cfg2_sk2000 --steps 3 --warmup 3 --no-e2e --no-cpu"
for rep in 1 2; do
  for v in libmars_b200_ho.so libmars_b200.so; do
    MARS_B200_LIB=$v timeout 300 $B >> $O/cfg2_$v.json 2>> $O/err.log
  done
done
echo done
