#!/bin/bash
# Full cfg2 batch (65536 descents): per-phase counters at 110/148 CTAs, then metrics-only ncu.
mkdir -p gpurun_out/p2
B="python bench.py --workload cfg2_sk2000 --steps 1 --warmup 1 --no-e2e --no-cpu --no-clocks"
for g in 110 148; do
  MARS_PROFILE=1 MARS_UMMA_GRID=$g timeout 300 $B > gpurun_out/p2/prof_g$g.json 2> gpurun_out/p2/prof_g$g.err
done
MARS_UMMA_GRID=110 timeout 300 $B > gpurun_out/p2/plain.json 2>&1 && \
MARS_UMMA_GRID=110 timeout 900 ncu --clock-control none -k regex:relax_dense_umma -c 1 \
  --metrics gpu__time_duration.sum,sm__inst_executed_pipe_tensor_subpipe_hmma.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg,sm__cycles_elapsed.avg.per_second,lts__throughput.avg.pct_of_peak_sustained_elapsed,dram__throughput.avg.pct_of_peak_sustained_elapsed \
  --csv --log-file gpurun_out/p2/ncu_metrics.csv $B > gpurun_out/p2/ncu.log 2>&1
echo done
