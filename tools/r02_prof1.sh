#!/bin/bash
# Round-2 first look: per-phase counters of the tcgen05 kernel on cfg2 (MARS_PROFILE) at a few
# grids, then a metrics-only ncu pass (tensor pipe, DRAM, L2) on the same command.
mkdir -p gpurun_out/p1
B="python bench.py --workload cfg2_sk2000 --runs 14080 --steps 1 --warmup 1 --no-e2e --no-cpu --no-clocks"
for g in 110 148 74; do
  MARS_PROFILE=1 MARS_UMMA_GRID=$g timeout 300 $B > gpurun_out/p1/prof_g$g.json 2> gpurun_out/p1/prof_g$g.err
done
MARS_UMMA_GRID=110 timeout 300 $B > gpurun_out/p1/plain.json 2>&1 && \
MARS_UMMA_GRID=110 timeout 900 ncu --clock-control none -k regex:relax_dense_umma -c 1 \
  --metrics gpu__time_duration.sum,sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_subpipe_hmma_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_tensor_subpipe_hmma.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg,sm__cycles_elapsed.avg.per_second,sm__throughput.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_tc_wavefronts.sum \
  --csv --log-file gpurun_out/p1/ncu_metrics.csv $B > gpurun_out/p1/ncu.log 2>&1
echo done
