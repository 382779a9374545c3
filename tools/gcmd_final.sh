#!/bin/bash
# One GPU session: tests, per-config bench lines, launch list, ncu captures (tools only).
mkdir -p gpurun_out/r01
timeout 1200 python -m pytest tests -m gpu -q > gpurun_out/r01/pytest_gpu.log 2>&1
timeout 900 python bench.py > gpurun_out/r01/bench_default.json 2> gpurun_out/r01/bench_default.err
for w in cfg1_sk256_pm1 cfg3a_er800 cfg3b_er2000 cfg4_ea2d cfg4_ea3d; do
  timeout 600 python bench.py --workload $w --steps 3 --warmup 3 > gpurun_out/r01/bench_$w.json 2> gpurun_out/r01/bench_$w.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r01/launches_default.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 1200 ncu --set full --import-source on --clock-control none -k regex:relax_dense_umma -c 1 -o gpurun_out/r01/ncu_umma_cfg2 python bench.py --runs 18944 --steps 1 --warmup 0 --no-e2e --no-cpu --no-clocks > gpurun_out/r01/ncu_umma_cfg2.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:relax_spmm -c 1 -o gpurun_out/r01/ncu_spmm_cfg3b python bench.py --workload cfg3b_er2000 --runs 3848 --steps 1 --warmup 0 --no-e2e --no-cpu --no-clocks > gpurun_out/r01/ncu_spmm_cfg3b.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:relax_stencil -c 1 -o gpurun_out/r01/ncu_stencil_ea2d python bench.py --workload cfg4_ea2d --runs 1184 --steps 1 --warmup 0 --no-e2e --no-cpu --no-clocks > gpurun_out/r01/ncu_stencil_ea2d.log 2>&1
timeout 600 ncu --set full --clock-control none -k regex:energy -c 1 -o gpurun_out/r01/ncu_energy_cfg2 python bench.py --runs 18944 --steps 1 --warmup 0 --no-e2e --no-cpu --no-clocks > gpurun_out/r01/ncu_energy_cfg2.log 2>&1
echo done
