#!/bin/bash
# one ncu --set full capture of the final-default tcgen05 kernel (fixed-T sweeps, 98 x 128 runs)
O=gpurun_out/fin3; mkdir -p $O
cat > /tmp/exp_f3.py <<'PY'
import os, sys, numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import paper_1907_05124_b200 as mb
p = mb.IsingProblem.dense(2000, mb.gen_sk_gaussian(2000, 7))
s0 = np.random.default_rng(1).uniform(-1, 1, (98 * 128, 2000)).astype(np.float32)
out, k = mb.debug_sweep(p, s0, 20.0, 10)
print(k, float(np.abs(out).mean()))
PY
timeout 300 python /tmp/exp_f3.py > $O/plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:relax_dense_umma -c 1 -o $O/umma_full python /tmp/exp_f3.py > $O/ncu.log 2>&1
echo done
