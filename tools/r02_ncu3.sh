#!/bin/bash
# full ncu capture of the current tcgen05 kernel on fixed-T sweeps (92 CTAs x 128 runs, SK2000, 10 sweeps)
mkdir -p gpurun_out/n3b
cat > /tmp/exp_n3.py <<'PY'
import os, sys, numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import paper_1907_05124_b200 as mb
p = mb.IsingProblem.dense(2000, mb.gen_sk_gaussian(2000, 7))
s0 = np.random.default_rng(1).uniform(-1, 1, (92 * 128, 2000)).astype(np.float32)
out, k = mb.debug_sweep(p, s0, 20.0, 10)
print(k, float(np.abs(out).mean()))
PY
MARS_PROFILE=1 timeout 300 python /tmp/exp_n3.py > gpurun_out/n3b/plain.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:relax_dense_umma -c 1 \
  -o gpurun_out/n3b/umma_full python /tmp/exp_n3.py > gpurun_out/n3b/ncu.log 2>&1
echo done
