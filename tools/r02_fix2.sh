#!/bin/bash
mkdir -p gpurun_out/f2
timeout 900 python -m pytest tests/test_gpu_trajectory.py -x -q -k "split" > gpurun_out/f2/pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/f2/pytest.log
B="python bench.py --workload cfg2_sk2000 --steps 3 --warmup 3 --no-e2e --no-cpu"
for v in libmars_b200_a.so libmars_b200.so libmars_b200_a.so libmars_b200.so; do
  MARS_B200_LIB=$v timeout 300 $B >> gpurun_out/f2/cfg2_$v.json 2>> gpurun_out/f2/cfg2_$v.err
done
for g in 80 86 98; do
  MARS_UMMA_GRID=$g timeout 300 $B >> gpurun_out/f2/cfg2_grid$g.json 2>> gpurun_out/f2/cfg2_grid$g.err
done
echo done
