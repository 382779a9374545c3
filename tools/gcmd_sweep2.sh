#!/bin/bash
timeout 900 python -m pytest tests -m gpu -q -k "sparse or tanh or launch_shapes or workload_prefix" > gpurun_out/sweep2_pytest.log 2>&1
S=tools/sweep.sh
$S cfg4_ea2d "X=default" "MARS_STENCIL_THREADS=64" "MARS_STENCIL_THREADS=64 MARS_STENCIL_CTAS_PER_SM=16" "MARS_STENCIL_THREADS=96" > gpurun_out/sweep2.log 2>&1
$S cfg4_ea3d "X=default" "MARS_STENCIL_THREADS=128 MARS_STENCIL_CTAS_PER_SM=8" "MARS_STENCIL_THREADS=192 MARS_STENCIL_CTAS_PER_SM=6" >> gpurun_out/sweep2.log 2>&1
$S cfg3b_er2000 "X=default" "MARS_SPARSE_CW=64" "MARS_SPARSE_CW=64 MARS_SPMM_RING_KB=16" >> gpurun_out/sweep2.log 2>&1
$S cfg3a_er800 "X=default" "MARS_SPARSE_CW=32 MARS_SPMM_H=2" >> gpurun_out/sweep2.log 2>&1
$S cfg1_sk256_pm1 "X=default" "--kernel-simt" >> gpurun_out/sweep2.log 2>&1
timeout 300 python bench.py --workload cfg1_sk256_pm1 --kernel dense_simt --steps 3 --warmup 3 --no-cpu >> gpurun_out/sweep2.log 2>&1
echo done
