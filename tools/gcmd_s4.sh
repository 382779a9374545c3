#!/bin/bash
mkdir -p gpurun_out/s4
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/s4/pytest_gpu.log 2>&1
timeout 600 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s4/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/s4/bench_cfg2_default.json 2> gpurun_out/s4/bench_cfg2_default.err
for w in cfg1_sk256_pm1 cfg3a_er800 cfg3b_er2000 cfg4_ea2d cfg4_ea3d; do
  timeout 600 python bench.py --workload $w --steps 3 --warmup 3 > gpurun_out/s4/bench_$w.json 2> gpurun_out/s4/bench_$w.err
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/s4/launches_default.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu > /dev/null 2>&1
timeout 900 ncu --replay-mode application --section SpeedOfLight --section MemoryWorkloadAnalysis --clock-control none -k regex:relax_spmm -c 1 -o gpurun_out/s4/ncu_spmm_cfg3b python bench.py --workload cfg3b_er2000 --steps 1 --warmup 0 --no-e2e --no-cpu --no-clocks > gpurun_out/s4/ncu_spmm_cfg3b.log 2>&1
echo done
