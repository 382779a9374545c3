"""Stress the split-K tcgen05 path: one N=16384 problem, repeated short batches (t_max 4) at
several run counts until one fails; prints each batch's time and the error (with the hang
detector's record when a barrier wait timed out)."""
import dataclasses, os, sys, time
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1907_05124_b200 as mb
from paper_1907_05124_b200.workloads import WORKLOADS, build_problem

w = dataclasses.replace(WORKLOADS["cfg5_sk16384"], t_max=float(os.environ.get("TMAX", "4")))
t0 = time.time()
p = build_problem(w)
print(f"problem {time.time() - t0:.1f}s", flush=True)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 6
sizes = [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "6144,8192,4096").split(",")]
for rep in range(reps):
    for runs in sizes:
        t = time.perf_counter()
        try:
            rec = mb.run_shard(p, mb.BatchSpec(w.params(), runs, w.base_seed + rep), 0, runs)
        except Exception as e:
            print(f"rep {rep} runs {runs}: FAILED after {time.perf_counter() - t:.1f}s: {e}", flush=True)
            sys.exit(1)
        print(f"rep {rep} runs {runs}: {time.perf_counter() - t:.1f}s ok", flush=True)
