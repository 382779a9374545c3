#!/bin/bash
mkdir -p gpurun_out/c5
timeout 900 python tools/sync_bench.py 8192 > gpurun_out/c5/sync_bench.log 2>&1
timeout 2400 python bench.py --workload cfg5_sk16384 --steps 1 --warmup 1 > gpurun_out/c5/bench_cfg5.json 2> gpurun_out/c5/bench_cfg5.err
timeout 600 ./tests/cuda/adapter_check > gpurun_out/c5/adapter_check.log 2>&1
echo done
