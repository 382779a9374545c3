"""Phase timings for the N=16384 dense workload (tools only)."""
import sys, time
sys.path.insert(0, ".")
t = time.perf_counter()
def lap(msg):
    global t
    now = time.perf_counter()
    print(f"{now - t:8.2f}s  {msg}", flush=True)
    t = now
import paper_1907_05124_b200 as mb
from paper_1907_05124_b200.workloads import WORKLOADS
lap("import")
w = WORKLOADS["cfg5_sk16384"]
J = mb.gen_sk_gaussian(w.n, w.seed)
lap("gen_sk_gaussian")
p = mb.IsingProblem.dense(w.n, J)
lap(f"IsingProblem.dense kernel={p.kernel()}")
runs = int(sys.argv[1]) if len(sys.argv) > 1 else 256
spec = mb.BatchSpec(w.params(), w.runs, w.base_seed)
b = mb.DeviceBatch(p, spec, 0, runs)
lap(f"DeviceBatch({runs})")
b.upload()
lap("upload")
tm = b.execute()
lap(f"execute relax {tm['relax_ms']:.0f} ms energy {tm['energy_ms']:.0f} ms sweeps {tm['total_sweeps']} grid {tm['grid']}")
