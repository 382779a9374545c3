#!/bin/bash
# End-of-round validation: GPU tests, smoke, one bench line per config (cfg5 excluded: ~1000 s
# per step), the reference arm on the headline config, and a small-kernel warps sweep.
mkdir -p gpurun_out/fin2
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/fin2/pytest_gpu.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/fin2/smoke.log 2>&1
for w in cfg2_sk2000 cfg1_sk256_pm1 cfg3a_er800 cfg3b_er2000 cfg4_ea2d cfg4_ea3d; do
  timeout 900 python bench.py --workload $w > gpurun_out/fin2/bench_$w.json 2> gpurun_out/fin2/bench_$w.err
done
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/fin2/ref_cfg2_sk2000.json 2> gpurun_out/fin2/ref.err
for wv in 4 5 10; do
  MARS_SMALL_WARPS=$wv timeout 200 python bench.py --workload cfg1_sk256_pm1 --no-cpu > gpurun_out/fin2/small_w$wv.json 2>&1
done
echo done
