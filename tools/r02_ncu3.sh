#!/bin/bash
# full ncu capture of the current tcgen05 kernel on fixed-T sweeps (98 CTAs x 128 runs, SK2000, 10 sweeps)
mkdir -p gpurun_out/n3c
cat > /tmp/exp_n3.py <<'PY'
import os, sys, numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import paper_1907_05124_b200 as mb
p = mb.IsingProblem.dense(2000, mb.gen_sk_gaussian(2000, 7))
s0 = np.random.default_rng(1).uniform(-1, 1, (98 * 128, 2000)).astype(np.float32)
out, k = mb.debug_sweep(p, s0, 20.0, 10)
print(k, float(np.abs(out).mean()))
PY
MARS_PROFILE=1 timeout 300 python /tmp/exp_n3.py > gpurun_out/n3c/plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:relax_dense_umma -c 1 \
  -o gpurun_out/n3c/umma_full python /tmp/exp_n3.py > gpurun_out/n3c/ncu.log 2>&1
echo done
# metrics of the whole cfg2 batch launch (tensor pipe, shared-memory pipe, DRAM)
M="python bench.py --workload cfg2_sk2000 --steps 1 --warmup 0 --no-e2e --no-cpu --no-clocks"
timeout 900 ncu --clock-control none -k regex:relax_dense_umma -c 1 --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_elapsed,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_tc_wavefronts_mem_shared.sum,l1tex__data_bank_reads.avg.pct_of_peak_sustained_elapsed,l1tex__data_bank_writes.avg.pct_of_peak_sustained_elapsed,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,smsp__inst_executed.sum --csv --log-file gpurun_out/n3c/ncu_cfg2_batch_metrics.csv $M > gpurun_out/n3c/ncu_batch.log 2>&1
echo done2
