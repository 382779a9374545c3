#!/bin/bash
mkdir -p gpurun_out/n2
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:relax_dense_umma -c 1 -o gpurun_out/n2/ncu_umma_cfg2_1wave python bench.py --runs 18944 --steps 1 --warmup 0 --no-e2e --no-cpu --no-clocks > gpurun_out/n2/ncu_umma.log 2>&1
SECS="--section SpeedOfLight --section MemoryWorkloadAnalysis --section ComputeWorkloadAnalysis --section Occupancy --section LaunchStats --section SchedulerStats --section WarpStateStats"
timeout 900 ncu --replay-mode application $SECS --clock-control none -k regex:relax_stencil -c 1 -o gpurun_out/n2/ncu_stencil_ea3d python bench.py --workload cfg4_ea3d --steps 1 --warmup 0 --no-e2e --no-cpu --no-clocks > gpurun_out/n2/ncu_stencil_ea3d.log 2>&1
echo done
