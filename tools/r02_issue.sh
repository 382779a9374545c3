#!/bin/bash
# one elect per stage (current) vs one per MMA (si0): parity, then same-box A/B
O=gpurun_out/iss; mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_trajectory.py tests/test_gpu_umma.py -x -q -k "not quench_consistency" > $O/pytest.log 2>&1; echo "rc=$?" >> $O/pytest.log
B="python bench.py --workload cfg2_sk2000 --steps 3 --warmup 3 --no-e2e --no-cpu"
for rep in 1 2; do
  for v in libmars_b200_si0.so libmars_b200.so; do
    MARS_B200_LIB=$v timeout 300 $B >> $O/cfg2_$v.json 2>> $O/err.log
  done
done
echo done
