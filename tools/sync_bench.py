"""Throughput of the GPU synchronous baselines (NMFA / SimCIM, jacobi_umma.cu) on cfg2's
instance: iterations of whole-run GEMM + fused update per second, and runs/s, next to the
reference's own run_batch on a bounded CPU sample (oracle/_ref, all host threads)."""
import json, os, sys, time
import numpy as np
ROOT = os.environ.get("GRAFT_REPO_ROOT", os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import paper_1907_05124_b200 as mb

n, runs, iters = 2000, int(sys.argv[1]) if len(sys.argv) > 1 else 8192, 1000
J = mb.gen_sk_gaussian(n, 7)
p = mb.IsingProblem.dense(n, J)
out = {}
for name, prm in (("nmfa", mb.nmfa_defaults(iters)), ("simcim", mb.simcim_defaults(iters))):
    mb.run_batch(p, mb.BatchSpec(prm, 256, 1))                     # warm-up
    t = time.perf_counter()
    st = mb.run_batch(p, mb.BatchSpec(prm, runs, 1))
    dt = time.perf_counter() - t
    flops = 2.0 * n * n * iters * runs
    out[name] = {"runs": runs, "iters": iters, "seconds": dt, "runs_per_s": runs / dt,
                 "algorithmic_tflops": flops / dt / 1e12, "best_energy": st.best_energy,
                 "mean_energy": st.mean_energy}
    print(name, json.dumps(out[name]), flush=True)
try:
    from oracle.oracle import Oracle
    R = Oracle("ref")
    rp = R.problem_dense(J)
    cores = os.cpu_count()
    for name, prm in (("nmfa", mb.nmfa_defaults(iters)), ("simcim", mb.simcim_defaults(iters))):
        k = cores
        t = time.perf_counter()
        if name == "nmfa":
            rp.run_sync("nmfa", prm.noise_sigma, prm.alpha, iters, prm.schedule, k, 1)
        else:
            rp.run_sync("simcim", prm.step_size, prm.noise_sigma, iters, prm.pump_schedule, k, 1)
        dt = time.perf_counter() - t
        out[name]["cpu_reference_runs_per_s"] = k / dt
        out[name]["cpu_sample"] = f"first {k} runs, {cores} workers, {dt:.1f} s"
        print(name, "cpu", k / dt, flush=True)
except Exception as e:  # the oracle travels as a prebuilt .so
    print("cpu reference unavailable:", e)
print(json.dumps(out))
