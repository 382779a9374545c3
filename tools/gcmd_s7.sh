#!/bin/bash
timeout 800 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "launch_shapes or exact" > gpurun_out/s7_pytest.log 2>&1
S=tools/sweep.sh
$S cfg3b_er2000 "X=default" "MARS_SPMM_R=2" > gpurun_out/s7_sweep.log 2>&1
$S cfg3a_er800 "X=default" "MARS_SPMM_R=2" >> gpurun_out/s7_sweep.log 2>&1
echo done
