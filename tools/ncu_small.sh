#!/bin/bash
# ncu evidence for cfg1's dominant kernel (relax_small.cu): launch list + one full capture.
mkdir -p gpurun_out/n3
timeout 300 python bench.py --workload cfg1_sk256_pm1 --steps 3 --warmup 3 > gpurun_out/n3/bench_cfg1.json 2> gpurun_out/n3/bench_cfg1.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/n3/launches_cfg1.csv python bench.py --workload cfg1_sk256_pm1 --steps 2 --warmup 1 --no-cpu --no-clocks > gpurun_out/n3/ncu_launch.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:relax_small -c 1 -o gpurun_out/n3/ncu_small_cfg1 python bench.py --workload cfg1_sk256_pm1 --steps 1 --warmup 0 --no-e2e --no-cpu --no-clocks > gpurun_out/n3/ncu_full.log 2>&1
echo done
