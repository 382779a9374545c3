#!/bin/bash
# same-box cfg2 experiments on the L2 policy of the state tiles and the persisting-L2 carve-out
mkdir -p gpurun_out/l2
B="python bench.py --workload cfg2_sk2000 --steps 3 --warmup 3 --no-e2e --no-cpu"
run() { timeout 300 env MARS_UMMA_DEBUG=1 "$@" $B >> gpurun_out/l2/$(echo "$@" | tr ' =' '__').json 2>> gpurun_out/l2/err.log; }
run MARS_BASE=1
run MARS_UMMA_SPOL=1
run MARS_UMMA_SPOL=2
run MARS_L2_PERSIST=1
run MARS_L2_PERSIST=1 MARS_UMMA_SPOL=1
run MARS_L2_PERSIST=2
run MARS_BASE=2
echo done
# the large-N split / tile choice (short schedule)
MARS_UMMA_DEBUG=1 timeout 600 python bench.py --workload cfg5_sk16384 --steps 1 --warmup 0 --no-e2e --no-cpu --no-clocks --tmax 4 > gpurun_out/l2/cfg5_t4.json 2> gpurun_out/l2/cfg5_t4.err
MARS_UMMA_DEBUG=1 timeout 600 python bench.py --workload cfg5_sk16384 --runs 1024 --steps 1 --warmup 0 --no-e2e --no-cpu --no-clocks --tmax 4 > gpurun_out/l2/cfg5_1024_t4.json 2> gpurun_out/l2/cfg5_1024_t4.err
timeout 600 python -m pytest tests/test_gpu_trajectory.py -x -q -k "split" > gpurun_out/l2/pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/l2/pytest.log
