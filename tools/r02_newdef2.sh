#!/bin/bash
# the new default (64-element SW128 stages, CUDA-core helper + walker fold): full GPU suite,
# smoke, default bench, reference arm, cfg5 large-N choices
O=gpurun_out/nd3; mkdir -p $O
MARS_HANG_S=60 timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "rc=$?" >> $O/bench_default.err
MARS_UMMA_DEBUG=1 timeout 900 python bench.py --workload cfg5_sk16384 --steps 1 --warmup 0 --no-e2e --no-cpu --no-clocks --tmax 30 > $O/cfg5_t30.json 2> $O/cfg5_t30.err
MARS_HANG_S=30 MARS_SYNC_CHECK=1 timeout 900 python tools/split_stress.py 2 6144,8192,1024 > $O/stress.log 2>&1; echo "rc=$?" >> $O/stress.log
echo done
