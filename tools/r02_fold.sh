#!/bin/bash
# walker fold (f1) vs every rectangle on the helper's mma path (current): parity, then same-box A/B
mkdir -p gpurun_out/fo
timeout 900 python -m pytest tests/test_gpu_trajectory.py tests/test_gpu_umma.py -x -q -k "not quench_consistency" > gpurun_out/fo/pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/fo/pytest.log
B="python bench.py --workload cfg2_sk2000 --steps 3 --warmup 3 --no-e2e --no-cpu"
for rep in 1 2; do
  for v in libmars_b200_f1.so libmars_b200.so; do
    MARS_B200_LIB=$v timeout 300 $B >> gpurun_out/fo/cfg2_$v.json 2>> gpurun_out/fo/err.log
  done
done
MARS_PROFILE=1 timeout 300 python bench.py --workload cfg2_sk2000 --steps 1 --warmup 1 --no-e2e --no-cpu --no-clocks > gpurun_out/fo/prof.json 2> gpurun_out/fo/prof.err
echo done
