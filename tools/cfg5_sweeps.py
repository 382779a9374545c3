"""cfg5 (SK N=16384) throughput probe: fixed-temperature sweeps of 8192 runs through the
tcgen05 kernel (mars_debug_sweeps) -> sweep-runs/s, and the same per kernel launch shape
(grid, clocks) -- the full 8192-descent batch takes ~10^4 sweeps per descent."""
import os, sys, time
import numpy as np
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1907_05124_b200 as mb

runs = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
sweeps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
t0 = time.time()
J = mb.gen_sk_gaussian(16384, 7)
p = mb.IsingProblem.dense(16384, J)
print(f"instance + problem {time.time() - t0:.1f}s kernel {p.kernel()}", flush=True)
s0 = np.random.default_rng(1).uniform(-1, 1, (runs, 16384)).astype(np.float32)
for it in range(2):
    t = time.perf_counter()
    out, k = mb.debug_sweep(p, s0, 60.0, sweeps)
    dt = time.perf_counter() - t
    print(f"{runs} runs x {sweeps} sweeps: {dt:.2f} s -> {runs * sweeps / dt:.0f} sweep-runs/s "
          f"(incl. upload/turnover sweeps)", flush=True)
