#!/bin/bash
# ncu captures of each config's dominant kernel at the bench workload (tools only).
# SourceCounters (SASS-patched per-instruction counts) is left out for the tcgen05 kernel:
# the instrumented replay is slow enough to trip the kernel's 20 s mbarrier watchdog.
mkdir -p gpurun_out/r01n
SECS="--section SpeedOfLight --section MemoryWorkloadAnalysis --section ComputeWorkloadAnalysis --section Occupancy --section LaunchStats --section SchedulerStats --section WarpStateStats --section InstructionStats --section MemoryWorkloadAnalysis_Tables"
timeout 1500 ncu $SECS --clock-control none -k regex:relax_dense_umma -c 1 -o gpurun_out/r01n/ncu_umma_cfg2 python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-clocks > gpurun_out/r01n/ncu_umma_cfg2.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:relax_spmm -c 1 -o gpurun_out/r01n/ncu_spmm_cfg3a python bench.py --workload cfg3a_er800 --steps 1 --warmup 0 --no-e2e --no-cpu --no-clocks > gpurun_out/r01n/ncu_spmm_cfg3a.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:relax_spmm -c 1 -o gpurun_out/r01n/ncu_spmm_cfg3b python bench.py --workload cfg3b_er2000 --steps 1 --warmup 0 --no-e2e --no-cpu --no-clocks > gpurun_out/r01n/ncu_spmm_cfg3b.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:relax_stencil -c 1 -o gpurun_out/r01n/ncu_stencil_ea2d python bench.py --workload cfg4_ea2d --steps 1 --warmup 0 --no-e2e --no-cpu --no-clocks > gpurun_out/r01n/ncu_stencil_ea2d.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:relax_stencil -c 1 -o gpurun_out/r01n/ncu_stencil_ea3d python bench.py --workload cfg4_ea3d --steps 1 --warmup 0 --no-e2e --no-cpu --no-clocks > gpurun_out/r01n/ncu_stencil_ea3d.log 2>&1
timeout 600 ncu $SECS --clock-control none -k regex:relax_dense_umma -c 1 -o gpurun_out/r01n/ncu_umma_cfg1 python bench.py --workload cfg1_sk256_pm1 --steps 1 --warmup 0 --no-e2e --no-cpu --no-clocks > gpurun_out/r01n/ncu_umma_cfg1.log 2>&1
echo done
