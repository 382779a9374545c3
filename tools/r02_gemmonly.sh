#!/bin/bash
# timing only: the GEMM's per-block time with the helpers' mma.sync rectangles skipped (and with
# the write-back decoupled too), one CTA pair alone and the full grid
O=gpurun_out/gemmonly; mkdir -p $O
cat > /tmp/exp_alone.py <<'PY'
import os, sys, time, numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import paper_1907_05124_b200 as mb
ctas = int(sys.argv[1])
p = mb.IsingProblem.dense(2000, mb.gen_sk_gaussian(2000, 7))
s0 = np.random.default_rng(1).uniform(-1, 1, (ctas * 128, 2000)).astype(np.float32)
out, k = mb.debug_sweep(p, s0, 20.0, 30)
print(ctas, k, flush=True)
PY
for g in 2 98; do
  for v in "MARS_UMMA_GEMMONLY=1 MARS_UMMA_NOWB=1"; do
    env $v MARS_HANG_S=20 MARS_UMMA_GRID=$g MARS_PROFILE=1 timeout 300 python /tmp/exp_alone.py $g >> $O/g$g.log 2>&1
    echo "-- $v" >> $O/g$g.log
  done
done
echo done
