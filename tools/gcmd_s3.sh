#!/bin/bash
mkdir -p gpurun_out/s3
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/s3/pytest_gpu.log 2>&1
for h in 0 1; do MARS_UMMA_L2HINT=$h timeout 600 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu > gpurun_out/s3/bench_cfg2_hint$h.json 2>&1; done
S=tools/sweep.sh
$S cfg4_ea2d "X=default" "MARS_STENCIL_THREADS=64" "MARS_STENCIL_THREADS=64 MARS_STENCIL_CTAS_PER_SM=16" > gpurun_out/s3/sweep.log 2>&1
$S cfg4_ea3d "X=default" "MARS_STENCIL_THREADS=128 MARS_STENCIL_CTAS_PER_SM=8" >> gpurun_out/s3/sweep.log 2>&1
$S cfg3b_er2000 "X=default" "MARS_SPARSE_CW=64" >> gpurun_out/s3/sweep.log 2>&1
timeout 300 python bench.py --workload cfg1_sk256_pm1 --kernel dense_simt --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/s3/bench_cfg1_simt.json 2>&1
SECS="--section SpeedOfLight --section MemoryWorkloadAnalysis --section ComputeWorkloadAnalysis --section Occupancy --section LaunchStats --section SchedulerStats --section WarpStateStats --section InstructionStats --section MemoryWorkloadAnalysis_Tables"
timeout 600 ncu $SECS --clock-control none -k regex:relax_spmm -c 1 -o gpurun_out/s3/ncu_spmm_cfg3b python bench.py --workload cfg3b_er2000 --steps 1 --warmup 0 --no-e2e --no-cpu --no-clocks > gpurun_out/s3/ncu_spmm_cfg3b.log 2>&1
timeout 600 ncu $SECS --clock-control none -k regex:relax_spmm -c 1 -o gpurun_out/s3/ncu_spmm_cfg3a python bench.py --workload cfg3a_er800 --steps 1 --warmup 0 --no-e2e --no-cpu --no-clocks > gpurun_out/s3/ncu_spmm_cfg3a.log 2>&1
timeout 600 ncu $SECS --clock-control none -k regex:relax_stencil -c 1 -o gpurun_out/s3/ncu_stencil_ea3d python bench.py --workload cfg4_ea3d --steps 1 --warmup 0 --no-e2e --no-cpu --no-clocks > gpurun_out/s3/ncu_stencil_ea3d.log 2>&1
echo done
