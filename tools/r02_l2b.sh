#!/bin/bash
# same-box: state-tile L2 policy evict_normal (0) vs evict_first (2), alternating, plus DRAM bytes of each (ncu metrics)
mkdir -p gpurun_out/l2b
B="python bench.py --workload cfg2_sk2000 --steps 3 --warmup 3 --no-e2e --no-cpu"
for rep in 1 2 3; do
  for sp in 0 2; do
    MARS_UMMA_SPOL=$sp timeout 300 $B >> gpurun_out/l2b/spol$sp.json 2>> gpurun_out/l2b/err.log
  done
done
M="python bench.py --workload cfg2_sk2000 --steps 1 --warmup 0 --no-e2e --no-cpu --no-clocks"
for sp in 0 2; do
  MARS_UMMA_SPOL=$sp timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:relax_dense_umma --csv --log-file gpurun_out/l2b/ncu_spol$sp.csv $M > gpurun_out/l2b/ncu_spol$sp.log 2>&1
done
echo done
