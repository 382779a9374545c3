"""NMFA and SimCIM on the GPU (solvers.cpp:374-443) against the compiled
reference, through the C-ABI (mars_run_batch_nmfa / _simcim).

Bars:
  * the device noise stream is the reference's Rng: engine outputs bit-exact, Box-Muller draws
    within 4 ulp (device fp64 log / sincos vs glibc);
  * noise-free NMFA (deterministic) reaches the reference's final spins on every run, energies
    bit-exact;
  * with noise, each run consumes the reference's own noise sequence; with the fp32-accurate
    state the runs end on the reference's final spins (measured: every run of every case;
    gated at 95%), energies bit-exact where they agree, mean energy within 1% and the best
    energy equal to or better than the reference's;
  * validation errors before any run, with the reference's messages.
"""
import numpy as np
import pytest

import paper_1907_05124_b200 as mb
from conftest import golden, gpu_available

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]


def test_device_stream_is_the_reference_rng():
    import ctypes as C
    from paper_1907_05124_b200._native import lib
    g = golden("rng")
    seeds = np.array([0, 1, 42], np.uint64)
    cnt = g["draw_u64"].shape[1]
    u = np.zeros((3, cnt), np.uint64)
    z = np.zeros((3, cnt))
    assert lib.mars_debug_rng(seeds.ctypes.data_as(C.c_void_p), 3, cnt, u.ctypes.data_as(C.c_void_p),
                              z.ctypes.data_as(C.c_void_p)) == 0
    assert np.array_equal(u, g["draw_u64"])
    ulp = np.abs(z - g["draw_gaussian"]) / np.spacing(np.abs(g["draw_gaussian"]))
    assert ulp.max() <= 4, ulp.max()


def _ref(J, h=None):
    from oracle.oracle import Oracle
    R = Oracle("ref")
    return R.problem_dense(J, h)


def _compare(dev, ref, frac, n):
    same = np.all(dev.records.spins == ref.spins, axis=1)
    assert np.array_equal(dev.records.status, ref.status)
    assert same.mean() >= frac, same.mean()
    assert np.array_equal(dev.records.energy[same], ref.energy[same])
    assert np.array_equal(dev.records.descent_iters, ref.descent_iters)
    assert np.array_equal(dev.records.start_temp, ref.start_temp)
    return same.mean()


def test_nmfa_noise_free_matches_reference():
    rng = np.random.default_rng(4)
    n = 200
    J = mb.gen_sk_gaussian(n, 12)
    h = rng.standard_normal(n)
    prm = mb.NmfaParams(0.0, 0.15, mb.linear_schedule(2.0, 0.02, 64), 300)
    dev = mb.run_batch(mb.IsingProblem.dense(n, J, h), mb.BatchSpec(prm, 64, 3, keep_spins=True))
    ref = _ref(J, h).run_sync("nmfa", 0.0, 0.15, 300, prm.schedule, 64, 3)
    _compare(dev, ref, 1.0, n)
    assert dev.best_energy == ref.stats["best_energy"]


@pytest.mark.parametrize("solver", ["nmfa", "simcim"])
@pytest.mark.parametrize("n,kind", [(256, "gauss"), (300, "pm1")])
def test_noisy_baselines_match_reference(solver, n, kind):
    J = mb.gen_sk_gaussian(n, 21) if kind == "gauss" else mb.gen_sk_pm1(n, 22)
    iters, runs, seed = 400, 256, 9
    if solver == "nmfa":
        prm = mb.nmfa_defaults(iters)
        ref = _ref(J).run_sync("nmfa", prm.noise_sigma, prm.alpha, iters, prm.schedule, runs, seed)
    else:
        prm = mb.simcim_defaults(iters)
        ref = _ref(J).run_sync("simcim", prm.step_size, prm.noise_sigma, iters, prm.pump_schedule, runs, seed)
    dev = mb.run_batch(mb.IsingProblem.dense(n, J), mb.BatchSpec(prm, runs, seed, keep_spins=True))
    frac = _compare(dev, ref, 0.95, n)
    assert abs(dev.mean_energy / ref.stats["mean_energy"] - 1.0) < 0.01
    assert dev.best_energy <= ref.stats["best_energy"] + (0.0 if kind == "pm1" else 1e-9)
    print(f"{solver} {kind} N={n}: {frac:.3f} of runs on the reference's spins; best {dev.best_energy} "
          f"(reference {ref.stats['best_energy']}), mean {dev.mean_energy:.2f} ({ref.stats['mean_energy']:.2f})")


def test_sparse_storage_runs_on_dense_planes():
    # a G-set-shape (CSR-stored) instance: the baselines build the fp16 planes on demand
    u, v, w = mb.gen_er(400, 0.02, 5)
    p = mb.IsingProblem.from_edges(400, (u, v, w))
    assert p.uses_adjacency()
    prm = mb.simcim_defaults(300)
    dev = mb.run_batch(p, mb.BatchSpec(prm, 128, 2, keep_spins=True))
    from oracle.oracle import Oracle
    ref = Oracle("ref").problem_edges(400, u, v, w).run_sync("simcim", prm.step_size, prm.noise_sigma, 300,
                                                             prm.pump_schedule, 128, 2)
    _compare(dev, ref, 0.95, 400)


def test_baseline_validation_errors():
    p = mb.IsingProblem.dense(2, [0, -1, -1, 0])
    for bad, msg in [(mb.NmfaParams(0.15, 0.0, [1.0], 10), "alpha"),
                     (mb.NmfaParams(-1.0, 0.1, [1.0], 10), "noise_sigma"),
                     (mb.NmfaParams(0.1, 0.1, [1.0], 0), "iters"),
                     (mb.NmfaParams(0.1, 0.1, [], 10), "schedule"),
                     (mb.NmfaParams(0.1, 0.1, [-1.0], 10), "temperatures"),
                     (mb.SimCimParams(0.0, 0.1, [1.0], 10), "step_size"),
                     (mb.SimCimParams(0.1, 0.1, [], 10), "pump")]:
        with pytest.raises(mb.InputError, match=msg):
            mb.run_batch(p, mb.BatchSpec(bad, 4, 1))
