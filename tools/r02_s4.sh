#!/bin/bash
# experiment: is the tcgen05 GEMM SMEM-port bound?  fixed-temperature sweeps isolate per-block cost
mkdir -p gpurun_out/s4
cat > /tmp/exp.py <<'PY'
import os, sys, time, numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import paper_1907_05124_b200 as mb
J = mb.gen_sk_gaussian(2000, 7)
p = mb.IsingProblem.dense(2000, J)
s0 = np.random.default_rng(1).uniform(-1, 1, (110 * 128, 2000)).astype(np.float32)
for it in range(2):
    t = time.perf_counter()
    out, k = mb.debug_sweep(p, s0, 20.0, 50)
    dt = time.perf_counter() - t
print(os.environ.get("MARS_UMMA_EXP", "0"), k, "50 sweeps x 14080 runs: %.3f s" % dt, flush=True)
PY
for e in 0 1 2 3; do MARS_PROFILE=1 MARS_UMMA_EXP=$e timeout 300 python /tmp/exp.py >> gpurun_out/s4/exp.log 2>&1; done
echo done
