#!/bin/bash
mkdir -p gpurun_out/sp
timeout 900 python -m pytest tests/test_gpu_trajectory.py -x -q -k "single_sweep or split_k" > gpurun_out/sp/pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/sp/pytest.log
for sp in 1 2; do MARS_PROFILE=1 MARS_UMMA_SPLIT=$sp timeout 600 python tools/cfg5_sweeps.py 8192 4 > gpurun_out/sp/cfg5_split$sp.log 2>&1; done
echo done
