"""The tcgen05 dense relaxation kernel (kernel="dense_umma") against the reference (GPU).

Same bars as tests/test_gpu_parity.py.  The state is an fp16 pair (22-23 significant bits)
and J_hi*S_hi + J_hi*S_lo + J_lo*S_hi is accumulated in fp32 (fp32-accurate split)."""
import numpy as np
import pytest

import paper_1907_05124_b200 as mb
from conftest import golden, gpu_available
from test_gpu_parity import SPIN_FRACTION, SPIN_FRACTION_FP32_SK2000, compare_records, uniform
from paper_1907_05124_b200.workloads import WORKLOADS, build_problem

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]


@pytest.fixture(autouse=True)
def _tensor_core_kernel_only(monkeypatch):
    # small integer batches would otherwise go to the warp-per-run kernel (relax_small.cu)
    monkeypatch.setenv("MARS_DENSE_SMALL", "0")


def test_umma_cfg1_full_batch(port):
    w = WORKLOADS["cfg1_sk256_pm1"]
    g = golden("cfg1")
    p = build_problem(w, kernel="dense_umma")
    assert p.kernel() == "dense_umma"
    stats = mb.run_batch(p, mb.BatchSpec(w.params(), w.runs, w.base_seed, keep_spins=True))
    compare_records(stats, g, w.n)
    assert stats.best_energy == -6120.0
    pp = port.problem_dense(port.gen_sk_pm1(w.n, w.seed))
    for k in range(0, w.runs, 11):
        assert stats.records.energy[k] == pp.energy(stats.records.spins[k])


@pytest.mark.parametrize("case", ["grid12", "grid24", "grid60", "int20"])
def test_umma_small_cases(case):
    g = golden("small")
    if case == "grid12":
        n, p = 12, mb.IsingProblem.dense(12, mb.gen_sk_gaussian(12, 4001), kernel="dense_umma")
        spec = mb.BatchSpec(mb.MarsParams(0, 10, 0.05), 1, 99, keep_spins=True)
    elif case == "grid24":
        n, p = 24, mb.IsingProblem.dense(24, mb.gen_sk_gaussian(24, 71), kernel="dense_umma")
        spec = mb.BatchSpec(mb.MarsParams(0, 12, 1), 1, 9, keep_spins=True)
    elif case == "grid60":
        n, p = 60, mb.IsingProblem.dense(60, mb.gen_sk_gaussian(60, 99), kernel="dense_umma")
        spec = mb.BatchSpec(mb.MarsParams(0, 16, 0.25), 1, 41, keep_spins=True)
    else:
        n, p = 20, mb.IsingProblem.dense(20, g["int20_J"], g["int20_h"], kernel="dense_umma")
        spec = mb.BatchSpec(uniform(20), 256, 3, keep_spins=True)
    stats = mb.run_batch(p, spec)
    compare_records(stats, g, n, prefix=case + "_")
    assert stats.best_energy == g[case + "_stats"][0]


def test_umma_cfg2_prefix():
    g = golden("cfg2_sk2000_prefix")
    w = WORKLOADS["cfg2_sk2000"]
    p = build_problem(w, kernel="dense_umma")
    k = len(g["status"])
    rec = mb.run_shard(p, mb.BatchSpec(w.params(), w.runs, w.base_seed, keep_spins=True), 0, k)
    compare_records(rec, g, w.n, frac=SPIN_FRACTION_FP32_SK2000)


def test_umma_shard_invariance():
    p = mb.IsingProblem.dense(300, mb.gen_sk_gaussian(300, 3), kernel="dense_umma")
    spec = mb.BatchSpec(uniform(20), 400, 8, keep_spins=True)
    full = mb.run_batch(p, spec)
    parts = [mb.run_shard(p, spec, f, c) for f, c in [(0, 129), (129, 271)]]
    assert np.array_equal(np.concatenate([x.energy for x in parts]), full.records.energy)
    assert np.array_equal(np.concatenate([x.spins for x in parts]), full.records.spins)
