#!/bin/bash
timeout 800 python -m pytest tests -m gpu -q > gpurun_out/s9_pytest.log 2>&1
timeout 300 python bench.py --workload cfg1_sk256_pm1 --steps 3 --warmup 3 > gpurun_out/s9_cfg1.json 2>&1
MARS_DENSE_SMALL=0 timeout 300 python bench.py --workload cfg1_sk256_pm1 --steps 3 --warmup 3 --no-cpu --no-e2e > gpurun_out/s9_cfg1_umma.json 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/s9_smoke.log 2>&1
echo done
