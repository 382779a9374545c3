#!/bin/bash
# Verify the exact-tanh sparse path on the GPU and measure its speed (tools only).
mkdir -p gpurun_out/r01v
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r01v/pytest_gpu.log 2>&1
for w in cfg3a_er800 cfg3b_er2000 cfg4_ea2d cfg4_ea3d; do
  timeout 600 python bench.py --workload $w --steps 3 --warmup 3 > gpurun_out/r01v/bench_$w.json 2> gpurun_out/r01v/bench_$w.err
done
timeout 600 python bench.py --workload cfg1_sk256_pm1 --kernel csr --steps 3 --warmup 3 > gpurun_out/r01v/bench_cfg1_csr.json 2> gpurun_out/r01v/bench_cfg1_csr.err
echo done
