#!/bin/bash
mkdir -p gpurun_out/fin4
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/fin4/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fin4/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/fin4/bench_cfg2_sk2000.json 2> gpurun_out/fin4/bench_cfg2.err
timeout 300 python bench.py --workload cfg1_sk256_pm1 > gpurun_out/fin4/bench_cfg1_sk256_pm1.json 2> gpurun_out/fin4/bench_cfg1.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fin4/launches_cfg2.csv python bench.py --steps 2 --warmup 1 --no-cpu --no-clocks > gpurun_out/fin4/ncu_launch.log 2>&1
echo done
