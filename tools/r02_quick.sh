#!/bin/bash
# quick check after a dense-kernel change: umma + trajectory tests, one cfg2 bench line with the profile
mkdir -p gpurun_out/q
timeout 900 python -m pytest tests/test_gpu_umma.py tests/test_gpu_trajectory.py -x -q -k "not quench_consistency" > gpurun_out/q/pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/q/pytest.log
MARS_PROFILE=1 timeout 300 python bench.py --workload cfg2_sk2000 --steps 1 --warmup 1 --no-e2e --no-cpu --no-clocks > gpurun_out/q/bench.json 2> gpurun_out/q/bench.err
echo done
