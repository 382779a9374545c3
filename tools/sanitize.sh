#!/bin/bash
# compute-sanitizer memcheck / racecheck over smoke() (tcgen05, small-instance and sparse kernels)
mkdir -p gpurun_out/san
timeout 1200 compute-sanitizer --tool memcheck --print-limit 20 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san/memcheck.log 2>&1; echo "memcheck rc=$?" >> gpurun_out/san/memcheck.log
MARS_DENSE_SMALL=1 timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python -c "
import paper_1907_05124_b200 as mb
J = mb.gen_sk_pm1(100, 3)
p = mb.IsingProblem.dense(100, J)
s = mb.run_batch(p, mb.BatchSpec(mb.MarsParams(0, 6, 1, 1, 1e-4, mb.StartMode.UniformRandom), 32, 1))
print('best', s.best_energy)" > gpurun_out/san/racecheck_small.log 2>&1; echo "racecheck rc=$?" >> gpurun_out/san/racecheck_small.log
timeout 300 python -m pytest tests -m gpu -q -k ragged > gpurun_out/san/ragged.log 2>&1
echo done
