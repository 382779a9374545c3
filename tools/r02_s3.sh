#!/bin/bash
# walker/helper epilogue: correctness first (tests), then the full cfg2 profile line
mkdir -p gpurun_out/s3
timeout 600 python -m pytest tests/test_gpu_trajectory.py tests/test_gpu_umma.py -x -q -k "not prefix_against" > gpurun_out/s3/pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s3/pytest.log
MARS_PROFILE=1 timeout 300 python bench.py --workload cfg2_sk2000 --steps 1 --warmup 1 --no-e2e --no-cpu --no-clocks > gpurun_out/s3/bench.json 2> gpurun_out/s3/bench.err
echo done
