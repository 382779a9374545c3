#!/bin/bash
# post-change check of the driver-facing entry points: default bench, the reference arm, smoke
O=gpurun_out/chk; mkdir -p $O
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "rc=$?" >> $O/bench_default.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err; echo "rc=$?" >> $O/bench_reference.err
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
timeout 900 python -m pytest tests/test_gpu_trajectory.py -q -s -k "cfg5_short or cfg2_prefix" > $O/prefix.log 2>&1; echo "rc=$?" >> $O/prefix.log
echo done
