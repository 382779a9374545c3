#!/bin/bash
# after the host refactor of the split choice: full GPU tests + the large-N choice on the GPU
O=gpurun_out/chk2; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
B="python bench.py --workload cfg5_sk16384 --steps 1 --warmup 0 --no-e2e --no-cpu --no-clocks --tmax 4"
MARS_UMMA_DEBUG=1 timeout 600 $B > $O/cfg5_t4.json 2> $O/cfg5_t4.err
MARS_UMMA_DEBUG=1 timeout 600 $B --runs 1024 > $O/cfg5_1024_t4.json 2> $O/cfg5_1024_t4.err
MARS_UMMA_DEBUG=1 timeout 600 python bench.py --workload cfg5_sk16384 --steps 1 --warmup 0 --no-e2e --no-cpu --no-clocks --tmax 30 > $O/cfg5_t30.json 2> $O/cfg5_t30.err
echo done
