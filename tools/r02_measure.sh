#!/bin/bash
# Round-2 measurement session: every BASELINE config's bench line, the cfg2 launch list and
# DRAM traffic of the full workload, the adapter check.  Outputs under gpurun_out/m/.
mkdir -p gpurun_out/m
for w in cfg2_sk2000 cfg1_sk256_pm1 cfg3a_er800 cfg3b_er2000 cfg4_ea2d cfg4_ea3d; do
  timeout 900 python bench.py --workload $w > gpurun_out/m/bench_$w.json 2> gpurun_out/m/bench_$w.err
done
timeout 600 python tests/cuda/adapter_check > gpurun_out/m/adapter_check.log 2>&1 || timeout 600 ./tests/cuda/adapter_check > gpurun_out/m/adapter_check.log 2>&1
B="python bench.py --workload cfg2_sk2000 --steps 1 --warmup 0 --no-e2e --no-cpu --no-clocks"
timeout 300 $B > gpurun_out/m/plain.json 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__inst_executed_pipe_tensor_subpipe_hmma.sum,sm__cycles_elapsed.avg,sm__cycles_elapsed.avg.per_second --clock-control none --csv --log-file gpurun_out/m/ncu_cfg2_launches.csv $B > gpurun_out/m/ncu.log 2>&1
echo done
