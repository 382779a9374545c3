#!/bin/bash
mkdir -p gpurun_out/s7
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
timeout 300 python -m pytest tests/test_gpu_trajectory.py -x -q -k "pm256 and umma" > gpurun_out/s7/pytest0.log 2>&1
echo "rc=$?" >> gpurun_out/s7/pytest0.log
timeout 900 python -m pytest tests/test_gpu_umma.py tests/test_gpu_trajectory.py -x -q -k "not quench_consistency" > gpurun_out/s7/pytest.log 2>&1
echo "pytest rc=$?" >> gpurun_out/s7/pytest.log
for e in 0; do MARS_PROFILE=1 MARS_UMMA_EXP=$e timeout 300 python /tmp/exp.py >> gpurun_out/s7/exp.log 2>&1; done
MARS_PROFILE=1 timeout 300 python bench.py --workload cfg2_sk2000 --steps 1 --warmup 1 --no-e2e --no-cpu --no-clocks > gpurun_out/s7/bench.json 2> gpurun_out/s7/bench.err
echo done
