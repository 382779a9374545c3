#!/bin/bash
# per-block cycles of one CTA pair alone (no L2 / DRAM / power contention) vs the full grid
O=gpurun_out/alone; mkdir -p $O
cat > /tmp/exp_alone.py <<'PY'
import os, sys, time, numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import paper_1907_05124_b200 as mb
ctas = int(sys.argv[1])
p = mb.IsingProblem.dense(2000, mb.gen_sk_gaussian(2000, 7))
s0 = np.random.default_rng(1).uniform(-1, 1, (ctas * 128, 2000)).astype(np.float32)
for it in range(2):
    t = time.perf_counter(); out, k = mb.debug_sweep(p, s0, 20.0, 30); print(ctas, k, time.perf_counter() - t, flush=True)
PY
for g in 2 8 32 98; do
  MARS_UMMA_GRID=$g MARS_PROFILE=1 timeout 300 python /tmp/exp_alone.py $g > $O/grid$g.log 2>&1
done
echo done
