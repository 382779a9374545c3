#!/bin/bash
# helper rectangles on mma.sync: parity first, then same-box A/B against the CUDA-core helper (h0)
mkdir -p gpurun_out/hm
timeout 900 python -m pytest tests/test_gpu_trajectory.py tests/test_gpu_umma.py -x -q -k "not quench_consistency" > gpurun_out/hm/pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/hm/pytest.log
B="python bench.py --workload cfg2_sk2000 --steps 3 --warmup 3 --no-e2e --no-cpu"
for rep in 1 2; do
  for v in libmars_b200_h0.so libmars_b200.so; do
    MARS_B200_LIB=$v timeout 300 $B >> gpurun_out/hm/cfg2_$v.json 2>> gpurun_out/hm/err.log
  done
done
MARS_PROFILE=1 timeout 300 python bench.py --workload cfg2_sk2000 --steps 1 --warmup 1 --no-e2e --no-cpu --no-clocks > gpurun_out/hm/prof.json 2> gpurun_out/hm/prof.err
MARS_PROFILE=1 MARS_B200_LIB=libmars_b200_h0.so timeout 300 python bench.py --workload cfg2_sk2000 --steps 1 --warmup 1 --no-e2e --no-cpu --no-clocks > gpurun_out/hm/prof_h0.json 2> gpurun_out/hm/prof_h0.err
echo done
