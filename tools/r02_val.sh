#!/bin/bash
# validation session: full GPU test suite, smoke, default bench line
mkdir -p gpurun_out/val
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/val/pytest_gpu.log 2>&1
echo "rc=$?" >> gpurun_out/val/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/val/smoke.log 2>&1
echo "rc=$?" >> gpurun_out/val/smoke.log
timeout 900 python bench.py > gpurun_out/val/bench.json 2> gpurun_out/val/bench.err
echo done
