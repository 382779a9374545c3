#!/bin/bash
# split-K = 4 parity + cfg5 batch timings (split auto = 2 at 8192 runs, 4 at 1024 runs)
mkdir -p gpurun_out/sp4
timeout 900 python -m pytest tests/test_gpu_trajectory.py -x -q -k "single_sweep or split_k" > gpurun_out/sp4/pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/sp4/pytest.log
MARS_PROFILE=1 MARS_UMMA_SPLIT=4 timeout 300 python tools/cfg5_sweeps.py 1024 4 > gpurun_out/sp4/cfg5_1024_split4.log 2>&1
timeout 1500 python bench.py --workload cfg5_sk16384 --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/sp4/bench_cfg5.json 2> gpurun_out/sp4/bench_cfg5.err
echo "bench rc=$?" >> gpurun_out/sp4/bench_cfg5.err
timeout 900 python bench.py --workload cfg5_sk16384 --runs 1024 --steps 1 --warmup 0 --no-e2e --no-cpu > gpurun_out/sp4/bench_cfg5_1024.json 2> gpurun_out/sp4/bench_cfg5_1024.err
echo done
