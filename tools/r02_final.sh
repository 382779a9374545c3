#!/bin/bash
# Round-2 final session: full GPU tests, smoke, every config's bench line (cfg5 included), the
# reference-side adapter check, NMFA/SimCIM throughput, cfg2 launch list + batch metrics (ncu),
# one full ncu capture of the tcgen05 kernel, MARS_PROFILE counters.  Outputs: gpurun_out/fin/
O=gpurun_out/fin; mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "rc=$?" >> $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "rc=$?" >> $O/smoke.log
for w in cfg2_sk2000 cfg1_sk256_pm1 cfg3a_er800 cfg3b_er2000 cfg4_ea2d cfg4_ea3d; do
  timeout 900 python bench.py --workload $w > $O/bench_$w.json 2> $O/bench_$w.err
done
timeout 600 ./tests/cuda/adapter_check > $O/adapter_check.log 2>&1
timeout 900 python tools/sync_bench.py 8192 > $O/sync_bench.log 2>&1
MARS_PROFILE=1 timeout 300 python bench.py --workload cfg2_sk2000 --steps 1 --warmup 1 --no-e2e --no-cpu --no-clocks > $O/prof_cfg2.json 2> $O/prof_cfg2.err
B="python bench.py --workload cfg2_sk2000 --steps 2 --warmup 1 --no-cpu --no-clocks"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/ncu_cfg2_launches.csv $B > $O/ncu_launches.log 2>&1
M="python bench.py --workload cfg2_sk2000 --steps 1 --warmup 0 --no-e2e --no-cpu --no-clocks"
timeout 900 ncu --clock-control none -k regex:relax_dense_umma -c 1 --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_tc_wavefronts_mem_shared.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum --csv --log-file $O/ncu_cfg2_batch_metrics.csv $M > $O/ncu_batch.log 2>&1
cat > /tmp/exp_fin.py <<'PY'
import os, sys, numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import paper_1907_05124_b200 as mb
p = mb.IsingProblem.dense(2000, mb.gen_sk_gaussian(2000, 7))
s0 = np.random.default_rng(1).uniform(-1, 1, (98 * 128, 2000)).astype(np.float32)
out, k = mb.debug_sweep(p, s0, 20.0, 10)
print(k, float(np.abs(out).mean()))
PY
timeout 300 python /tmp/exp_fin.py > $O/plain_sweeps.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:relax_dense_umma -c 1 -o $O/umma_full python /tmp/exp_fin.py > $O/ncu_full.log 2>&1
timeout 1800 python bench.py --workload cfg5_sk16384 --steps 1 --warmup 0 > $O/bench_cfg5_sk16384.json 2> $O/bench_cfg5_sk16384.err
echo done
