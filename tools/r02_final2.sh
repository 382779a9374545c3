#!/bin/bash
# refresh of the dense-kernel measurements for the final default (64-element stages, CUDA-core
# helper): cfg2 line with the per-phase counters, cfg2 launch list + batch ncu metrics, cfg5 line
O=gpurun_out/fin2; mkdir -p $O
MARS_PROFILE=1 timeout 300 python bench.py --workload cfg2_sk2000 --steps 1 --warmup 1 --no-e2e --no-cpu --no-clocks > $O/prof_cfg2.json 2> $O/prof_cfg2.err
B="python bench.py --workload cfg2_sk2000 --steps 2 --warmup 1 --no-cpu --no-clocks"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/ncu_cfg2_launches.csv $B > $O/ncu_launches.log 2>&1
M="python bench.py --workload cfg2_sk2000 --steps 1 --warmup 0 --no-e2e --no-cpu --no-clocks"
timeout 900 ncu --clock-control none -k regex:relax_dense_umma -c 1 --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__ops_path_tensor_op_utchmma_src_fp16_dst_fp32_sparsity_off.sum.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_tc_wavefronts_mem_shared.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum --csv --log-file $O/ncu_cfg2_batch_metrics.csv $M > $O/ncu_batch.log 2>&1
timeout 1800 python bench.py --workload cfg5_sk16384 --steps 1 --warmup 0 > $O/bench_cfg5_sk16384.json 2> $O/bench_cfg5_sk16384.err
echo done
