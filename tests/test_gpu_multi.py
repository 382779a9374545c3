"""mars_run_batch_multi (multi-GPU inside one C-ABI call) on the GPU.

This pool gives one GPU per call, so the N-device exchange is exercised as a single-rank NCCL
communicator (MARS_MULTI_FORCE=1 keeps the NCCL path for one replica): NCCL loaded at run
time, ncclCommInitAll, the four collectives on device buffers, the packed record AllGather and
its unpacking.  The rank logic for N > 1 is covered on CPU by
tests/test_distributed.py::test_native_multi_gpu_exchange_logic (same C++ code, host transport)."""
import numpy as np
import pytest

import paper_1907_05124_b200 as mb
from conftest import gpu_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]


@pytest.mark.parametrize("kernel", ["dense_umma", "csr"])
def test_multi_call_equals_run_batch(kernel, monkeypatch):
    if kernel == "csr":
        p = mb.IsingProblem.from_edges(400, mb.gen_er(400, 0.02, 3))
        prm = mb.MarsParams(0, 12, 1, 1, 1e-4, mb.StartMode.UniformRandom)
    else:
        p = mb.IsingProblem.dense(300, mb.gen_sk_gaussian(300, 5))
        prm = mb.MarsParams(0, 20, 1, 1, 1e-4, mb.StartMode.UniformRandom)
    spec = mb.BatchSpec(prm, 300, 7, keep_spins=True)
    one = mb.run_batch(p, spec)
    monkeypatch.setenv("MARS_MULTI_FORCE", "1")
    multi = mb.run_batch_multi([p], spec)
    for name in ("status", "energy", "cut", "descent_iters", "start_temp", "spins"):
        assert np.array_equal(getattr(multi.records, name), getattr(one.records, name)), name
    assert multi.best_index == one.best_index and multi.best_energy == one.best_energy
    assert np.array_equal(multi.best_result.spins, one.best_result.spins)


def test_replica_is_the_same_problem():
    p = mb.IsingProblem.dense(64, mb.gen_sk_pm1(64, 2))
    q = p.replicate(0)
    assert q.size() == 64 and q.kernel() == p.kernel() and q.coupling_sum() == p.coupling_sum()
    s = np.where(np.arange(64) % 3 == 0, 1, -1).astype(np.int8)
    assert mb.energy(q, s) == mb.energy(p, s)
