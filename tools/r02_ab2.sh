#!/bin/bash
# same-box A/B: previous build (a) vs current, and current at several grids
mkdir -p gpurun_out/ab2
B="python bench.py --workload cfg2_sk2000 --steps 3 --warmup 3 --no-e2e --no-cpu"
run() { timeout 300 env "$@" $B >> gpurun_out/ab2/$(echo "$@" | tr ' =' '__').json 2>> gpurun_out/ab2/err.log; }
for rep in 1 2; do
  run MARS_B200_LIB=libmars_b200_a.so
  run MARS_B200_LIB=libmars_b200.so
  run MARS_UMMA_GRID=98
  run MARS_UMMA_GRID=104
done
timeout 600 python -m pytest tests/test_gpu_trajectory.py -x -q -k "split or single_sweep" > gpurun_out/ab2/pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/ab2/pytest.log
echo done
