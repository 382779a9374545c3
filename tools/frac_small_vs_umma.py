import os, sys, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1907_05124_b200 as mb
from oracle.oracle import Oracle, params
port = Oracle("port")
for n, h in [(37, False), (100, True), (200, False), (256, True), (256, False)]:
    J = port.gen_sk_pm1(n, 40 + n)
    hv = np.where(np.arange(n) % 3 == 0, 1.0, -1.0) if h else None
    t = float(int(np.sqrt(n)) + 2)
    ob = (port.problem_dense(J, hv) if h else port.problem_dense(J)).run_batch(params(0, t, 1, 1, 1e-4, uniform=True), 256, 3)
    out = []
    for small in ("1", "0"):
        os.environ["MARS_DENSE_SMALL"] = small
        p = mb.IsingProblem.dense(n, J, hv)
        st = mb.run_batch(p, mb.BatchSpec(mb.MarsParams(0, t, 1, 1, 1e-4, mb.StartMode.UniformRandom), 256, 3, keep_spins=True))
        same = np.all(st.records.spins == ob.spins, axis=1)
        out.append((round(same.mean(), 3), st.best_energy))
    print(n, h, "small", out[0], "umma", out[1], "oracle best", ob.stats["best_energy"], flush=True)
