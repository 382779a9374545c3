#!/bin/bash
# Standard GPU validation session (run through gpurun): GPU tests, smoke(), default bench, cfg1 bench.
mkdir -p gpurun_out/fin
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/fin/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fin/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/fin/bench_cfg2_default.json 2> gpurun_out/fin/bench_cfg2_default.err
timeout 300 python bench.py --workload cfg1_sk256_pm1 > gpurun_out/fin/bench_cfg1_sk256_pm1.json 2> gpurun_out/fin/bench_cfg1.err
echo done
