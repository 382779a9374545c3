#!/bin/bash
# timing experiment: how much of a block is the write-back coupling (GEMM(b+1)'s last chunks wait
# for walker(b))?  Fixed-T sweeps (98 x 128 runs, 30 sweeps) with the per-phase counters, with and
# without the producers' write-back waits (MARS_UMMA_NOWB=1: results wrong, timing only).
O=gpurun_out/nowb; mkdir -p $O
cat > /tmp/exp_nowb.py <<'PY'
import os, sys, time, numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import paper_1907_05124_b200 as mb
p = mb.IsingProblem.dense(2000, mb.gen_sk_gaussian(2000, 7))
s0 = np.random.default_rng(1).uniform(-1, 1, (98 * 128, 2000)).astype(np.float32)
for it in range(2):
    t = time.perf_counter(); out, k = mb.debug_sweep(p, s0, 20.0, 30); print(k, time.perf_counter() - t, flush=True)
PY
for v in 0 1 0 1; do
  MARS_UMMA_NOWB=$v MARS_PROFILE=1 timeout 300 python /tmp/exp_nowb.py >> $O/nowb$v.log 2>&1
done
echo done
