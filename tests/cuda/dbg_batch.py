import sys, time, numpy as np
sys.path.insert(0, "/root/repo")
import paper_1907_05124_b200 as mb
n = int(sys.argv[1]); tmax = float(sys.argv[2]); runs = int(sys.argv[3]); kernel = sys.argv[4]
p = mb.IsingProblem.dense(n, mb.gen_sk_gaussian(n, 7), kernel=kernel)
spec = mb.BatchSpec(mb.MarsParams(0, tmax, 1, 1, 1e-4, mb.StartMode.UniformRandom), runs, 1, keep_spins=False)
b = mb.DeviceBatch(p, spec); b.upload()
t = b.execute()
rec, best, _ = b.fetch()
it = rec.descent_iters
print(kernel, n, tmax, runs, "relax_ms", round(t["relax_ms"],1), "status", np.bincount(rec.status, minlength=3), "iters mean", it.mean(), "max", it.max(), "argmax", it.argmax(), "best", rec.energy[rec.status==0].min(), flush=True)
