timeout 1500 python bench.py --workload cfg5_sk16384 --steps 1 --warmup 0 --no-e2e > gpurun_out/bench_cfg5.log 2>&1
echo rc=$? >> gpurun_out/bench_cfg5.log
echo done
