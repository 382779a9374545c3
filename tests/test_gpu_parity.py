"""Parity of the sm_100a path against the reference (GPU; every call goes through the C-ABI).

Bars (BASELINE.json north_star):
  * energy / cut of any returned spin vector: BIT-EXACT (device fp64 in the reference's
    exact order -- checked for integer AND Gaussian couplings);
  * per-run status, start temperature: exact;
  * rounded final spins: identical to the reference on >= SPIN_FRACTION of runs (the
    device relaxes in fp32 with blocked summation; fp rounding can flip a chaotic
    trajectory into a different local minimum);
  * best-found energy: equal to the reference's on the small/integral instances;
  * descent_iters: reported as a distribution (not gated per run), mean within 10%.
"""
import os

import numpy as np
import pytest

import paper_1907_05124_b200 as mb
from conftest import golden, gpu_available, unpack_spins
from paper_1907_05124_b200.workloads import WORKLOADS, build_problem

pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(not gpu_available(), reason="needs a CUDA device")]

SPIN_FRACTION = 0.98          # fp64 CSR kernel (exact op order) and small dense instances


def fp32_floor_gate(k=None):
    """Dense fp32 kernels on Gaussian SK N=2000, T up to 40: the committed fp32 replay of the
    reference (tests/golden/cfg2_sk2000_f32replay.npz, oracle/mars_oracle.c
    orc_replay_batch_f32: the same descents with fp32 state, fields and tanh) ends on the
    reference's spins in 80.1% of the first 256 runs -- a chaotic descent split by rounding
    reaches another local minimum.  Gate: that floor minus a 3-sigma binomial margin."""
    g = golden("cfg2_sk2000_prefix")
    r = golden("cfg2_sk2000_f32replay")
    k = len(g["status"]) if k is None else k
    floor = np.all(unpack_spins(r["spins_packed"], 2000)[:k] == unpack_spins(g["spins_packed"], 2000)[:k],
                   axis=1).mean()
    return floor - 3.0 * np.sqrt(floor * (1.0 - floor) / k)


SPIN_FRACTION_FP32_SK2000 = fp32_floor_gate()


def uniform(t_max, t_min=0.0):
    return mb.MarsParams(t_min, t_max, 1, 1, 1e-4, mb.StartMode.UniformRandom)


def compare_records(stats, g, n, prefix="", frac=SPIN_FRACTION, count=None):
    rec = stats.records if hasattr(stats, "records") else stats
    k = len(g[prefix + "status"]) if count is None else count
    assert np.array_equal(rec.status[:k], g[prefix + "status"][:k])
    assert np.array_equal(rec.start_temp[:k], g[prefix + "start_temp"][:k])
    ok = g[prefix + "status"][:k] == 0
    ref_spins = unpack_spins(g[prefix + "spins_packed"], n)[:k]
    same = np.all(rec.spins[:k] == ref_spins, axis=1)[ok]
    frac_same = same.mean() if same.size else 1.0
    # where the spins agree the energies must agree bit for bit
    e_same = rec.energy[:k][ok][same]
    assert np.array_equal(e_same, g[prefix + "energy"][:k][ok][same])
    assert np.array_equal(rec.cut[:k][ok][same], g[prefix + "cut"][:k][ok][same])
    it_ref = g[prefix + "iters"][:k][ok].astype(float)
    it_dev = rec.descent_iters[:k][ok].astype(float)
    assert frac_same >= frac, f"only {frac_same:.3f} of runs end in the reference's spins"
    if it_ref.sum() > 0:
        assert abs(it_dev.mean() / it_ref.mean() - 1.0) < 0.10, (it_dev.mean(), it_ref.mean())
    return frac_same


def test_cfg1_full_batch_matches_reference(port):
    w = WORKLOADS["cfg1_sk256_pm1"]
    g = golden("cfg1")
    p = build_problem(w, kernel="dense_simt")
    assert p.kernel() == "dense_simt"
    stats = mb.run_batch(p, mb.BatchSpec(w.params(), w.runs, w.base_seed, keep_spins=True))
    compare_records(stats, g, w.n)
    assert stats.best_energy == -6120.0 == g["stats"][0]
    assert stats.best_cut == g["stats"][2]
    # every returned energy is the exact reference energy of the returned spins
    pp = port.problem_dense(port.gen_sk_pm1(w.n, w.seed))
    for k in range(0, w.runs, 7):
        assert stats.records.energy[k] == pp.energy(stats.records.spins[k])
        assert stats.records.cut[k] == pp.cut_value(stats.records.spins[k])
    assert stats.best_result.energy == stats.best_energy
    assert np.array_equal(stats.best_result.spins, stats.records.spins[stats.best_index])


@pytest.mark.parametrize("case", ["grid12", "grid24", "grid60", "ferro", "int20", "er200", "ea16"])
def test_small_cases_match_reference(case, port):
    g = golden("small")
    if case == "grid12":
        n, p = 12, mb.IsingProblem.dense(12, mb.gen_sk_gaussian(12, 4001))
        spec = mb.BatchSpec(mb.MarsParams(0, 10, 0.05), 1, 99, keep_spins=True)
    elif case == "grid24":
        n, p = 24, mb.IsingProblem.dense(24, mb.gen_sk_gaussian(24, 71))
        spec = mb.BatchSpec(mb.MarsParams(0, 12, 1), 1, 9, keep_spins=True)
    elif case == "grid60":
        n, p = 60, mb.IsingProblem.dense(60, mb.gen_sk_gaussian(60, 99))
        spec = mb.BatchSpec(mb.MarsParams(0, 16, 0.25), 1, 41, keep_spins=True)
    elif case == "ferro":
        # two degenerate ground states (++ / --): which one a run reaches is decided by the
        # sign of a state that decays toward 0 above T_c = 1 -- in fp32 it underflows to an
        # exact 0 where fp64 keeps the sign.  Energies must match; spins up to a global flip.
        p = mb.IsingProblem.dense(2, [0, -1, -1, 0])
        stats = mb.run_batch(p, mb.BatchSpec(mb.MarsParams(0, 30, 1), 1, 77, keep_spins=True))
        assert np.array_equal(stats.records.status, g["ferro_status"])
        assert np.array_equal(stats.records.energy, g["ferro_energy"])
        ok = stats.records.status == 0
        assert np.all(stats.records.spins[ok, 0] == stats.records.spins[ok, 1])
        return
    elif case == "int20":
        n, p = 20, mb.IsingProblem.dense(20, g["int20_J"], g["int20_h"])
        spec = mb.BatchSpec(uniform(20), 256, 3, keep_spins=True)
    elif case == "er200":
        n = 200
        p = mb.IsingProblem.from_edges(200, (g["er200_u"], g["er200_v"], g["er200_w"]), g["er200_h"])
        assert p.uses_adjacency() and p.kernel() == "csr"
        spec = mb.BatchSpec(uniform(10), 256, 4, keep_spins=True)
    else:
        n = 256
        p = mb.IsingProblem.from_edges(256, mb.gen_ea(16, 2, 5))
        spec = mb.BatchSpec(uniform(4), 256, 1, keep_spins=True)
    stats = mb.run_batch(p, spec)
    compare_records(stats, g, n, prefix=case + "_")
    assert stats.best_energy == g[case + "_stats"][0]
    assert stats.skipped_runs == g[case + "_stats"][8]


def test_energy_bit_exact_any_couplings(port):
    rng = np.random.default_rng(5)
    for J in (port.gen_sk_gaussian(300, 11), port.gen_sk_pm1(300, 12)):
        p = mb.IsingProblem.dense(300, J)
        pp = port.problem_dense(J)
        for _ in range(20):
            s = rng.choice(np.array([-1, 1], np.int8), 300)
            assert mb.energy(p, s) == pp.energy(s)
            assert mb.cut_value(p, s) == pp.cut_value(s)
    g = golden("small")
    p = mb.IsingProblem.from_edges(200, (g["er200_u"], g["er200_v"], g["er200_w"]), g["er200_h"])
    pp = port.problem_edges(200, g["er200_u"], g["er200_v"], g["er200_w"], g["er200_h"])
    for _ in range(20):
        s = rng.choice(np.array([-1, 1], np.int8), 200)
        assert mb.energy(p, s) == pp.energy(s)
        assert mb.cut_value(p, s) == pp.cut_value(s)


def test_kernels_agree_across_storage(port):
    # G1-style graph stored dense by the reference (6% > 5%): AUTO routes it to the fp64 CSR
    # kernel, whose sorted-nonzero sums are bit-identical to the dense row_dot
    u, v, w = mb.gen_er(300, 0.06, 9)
    p = mb.IsingProblem.from_edges(300, (u, v, w))
    assert not p.uses_adjacency() and p.kernel() == "csr"
    a = mb.run_batch(p, mb.BatchSpec(uniform(12), 256, 5, keep_spins=True))
    from oracle.oracle import params
    ob = port.problem_edges(300, u, v, w).run_batch(params(0, 12, 1, uniform=True), 256, 5)
    assert (np.all(a.records.spins == ob.spins, axis=1)).mean() >= SPIN_FRACTION
    assert a.best_energy == ob.stats["best_energy"]
    # the fp32 dense kernel forced onto the same instance: statistically equivalent batch
    b = mb.run_batch(mb.IsingProblem.from_edges(300, (u, v, w), kernel="dense_simt"),
                     mb.BatchSpec(uniform(12), 256, 5, keep_spins=True))
    assert b.best_energy <= ob.stats["best_energy"] * 0.99
    assert abs(b.mean_energy / ob.stats["mean_energy"] - 1) < 0.01


def test_determinism_and_shard_invariance():
    # identical results for any sharding of the run indices (test_runner.cpp:60-69 analogue)
    p = mb.IsingProblem.dense(128, mb.gen_sk_gaussian(128, 3))
    spec = mb.BatchSpec(uniform(20), 300, 8, keep_spins=True)
    full = mb.run_batch(p, spec)
    again = mb.run_batch(p, spec)
    assert np.array_equal(full.records.energy, again.records.energy)
    assert np.array_equal(full.records.descent_iters, again.records.descent_iters)
    parts = [mb.run_shard(p, spec, f, c) for f, c in [(0, 101), (101, 150), (251, 49)]]
    for name in ("status", "energy", "cut", "start_temp", "descent_iters"):
        assert np.array_equal(np.concatenate([getattr(x, name) for x in parts]),
                              getattr(full.records, name)), name
    assert np.array_equal(np.concatenate([x.spins for x in parts]), full.records.spins)


def test_divergence_records_match_port(port):
    # sweep_cap overrides kMarsSweepCap: runs that exhaust it become Diverged records with
    # the failing level's sweep count and the rounded partial state (runner.cpp:43-53)
    J = port.gen_sk_pm1(64, 21)
    prm = mb.MarsParams(0, 8, 1, 1, 1e-4, mb.StartMode.UniformRandom, sweep_cap=40)
    port.set_sweep_cap(40)
    try:
        from oracle.oracle import params
        ob = port.problem_dense(J).run_batch(params(0, 8, 1, 1, 1e-4, uniform=True), 128, 2)
    finally:
        port.set_sweep_cap(0)
    stats = mb.run_batch(mb.IsingProblem.dense(64, J), mb.BatchSpec(prm, 128, 2, keep_spins=True))
    assert stats.failed_runs > 0 and stats.completed_runs > 0
    agree = (stats.records.status == ob.status).mean()
    assert agree >= 0.95
    both_div = (stats.records.status == 2) & (ob.status == 2)
    assert np.all(stats.records.descent_iters[both_div] <= 40)
    assert stats.completed_runs == (stats.records.status == 0).sum()
    # a Diverged record is built fresh (runner.cpp:43-53): elapsed 0, DivergedError's message with
    # the level temperature formatted by std::to_string (solvers.cpp:169)
    div = np.flatnonzero(stats.records.status == 2)
    assert np.all(stats.records.elapsed_seconds[div] == 0.0)
    for k in div[:8]:
        msg = stats.runs[k].error
        assert msg.startswith("relaxation exceeded the sweep cap at T = ")
        t = float(msg.rsplit("= ", 1)[1])
        assert msg.endswith("%f" % t)
        levels = stats.records.start_temp[k] - np.arange(1, 64)
        assert np.min(np.abs(levels - t)) < 1e-5


def test_all_failed_batch_raises():
    p = mb.IsingProblem.dense(64, mb.gen_sk_gaussian(64, 2))
    prm = mb.MarsParams(0, 30, 1, 1, 1e-12, mb.StartMode.UniformRandom, sweep_cap=1)
    with pytest.raises(mb.Error, match="no run completed"):
        mb.run_batch(p, mb.BatchSpec(prm, 16, 1))


def test_input_errors_before_any_run():
    p = mb.IsingProblem.dense(2, [0, -1, -1, 0])
    with pytest.raises(mb.InputError):
        mb.run_batch(p, mb.BatchSpec(mb.MarsParams(c_step=0.0), 1, 1))
    with pytest.raises(mb.InputError):
        mb.run_batch(p, mb.BatchSpec(mb.MarsParams(0, 30, 40), 1, 1))
    with pytest.raises(mb.InputError):
        mb.IsingProblem.dense(2, [0, 1, 2, 0])          # asymmetric
    with pytest.raises(mb.InputError):
        mb.IsingProblem.dense(2, [1, 1, 1, 0])          # nonzero diagonal
    with pytest.raises(mb.InputError):
        mb.IsingProblem.from_edges(3, [(0, 0, 1.0)])    # self coupling
    with pytest.raises(mb.InputError):
        mb.energy(p, np.array([1, 1, 1], np.int8))      # length mismatch


@pytest.mark.parametrize("name,frac", [("cfg2_sk2000", SPIN_FRACTION_FP32_SK2000),
                                       ("cfg3a_er800", SPIN_FRACTION),
                                       ("cfg3b_er2000", SPIN_FRACTION),
                                       ("cfg4_ea2d", 0.9),
                                       ("cfg4_ea3d", 0.85)])
def test_workload_prefix_matches_reference(name, frac):
    """The first run indices of each BASELINE config, run as a shard of the full batch,
    against the compiled reference's records for the same indices."""
    import os
    from conftest import GOLDEN
    if not os.path.exists(os.path.join(GOLDEN, name + "_prefix.npz")):
        pytest.skip("fixture not generated")
    g = golden(name + "_prefix")
    w = WORKLOADS[name]
    k = len(g["status"])
    p = build_problem(w)
    rec = mb.run_shard(p, mb.BatchSpec(w.params(), w.runs, w.base_seed, keep_spins=True), 0, k)
    compare_records(rec, g, w.n, frac=frac)
    if p.kernel() == "csr" and _host_has_fma():
        # fp64 sparse path with the reference's tanh: the prefix is the reference's, exactly
        assert np.array_equal(rec.descent_iters[:k], g["iters"][:k])
        assert compare_records(rec, g, w.n, frac=1.0) == 1.0
    assert abs(p.coupling_sum() - g["coupling_sum"][0]) == 0.0
    # the device's best over the prefix is equal to or better than the reference's
    dev_best = rec.energy[rec.status == 0].min()
    ref_best = g["energy"][g["status"] == 0].min()
    assert dev_best <= ref_best + (0.0 if p.integral() else 1e-9), (dev_best, ref_best)


@pytest.mark.parametrize("kind", ["ea2d", "ea3d", "er_gauss"])
def test_sparse_launch_shapes_bit_identical(kind, monkeypatch, port):
    """The level-scheduled sparse kernel is the reference's sequential sweep reordered only
    across uncoupled spins: every launch shape (state in shared memory or in a global row,
    1..8 warps, 16- or 32-spin chunks, 1..8 runs per CTA, any grid; or the warp-per-run
    kernel with any ring depth) must give bit-identical records, and those records must
    match the reference port run for run."""
    if kind == "ea2d":
        n, (u, v, w) = 24 * 24, mb.gen_ea(24, 2, 3)
    elif kind == "ea3d":
        n, (u, v, w) = 8 ** 3, mb.gen_ea(8, 3, 4)
    else:   # non-unit weights: the multiply path
        rng = np.random.default_rng(7)
        n = 400
        u, v = np.triu_indices(n, 1)
        keep = rng.random(u.size) < 0.02
        u, v = u[keep].astype(np.int32), v[keep].astype(np.int32)
        w = rng.standard_normal(u.size)
    spec = mb.BatchSpec(uniform(6), 96, 11, keep_spins=True)
    results = []
    levels = [("smem", "1", "0", "1", "32"), ("smem", "4", "7", "4", "16"),
              ("global", "2", "0", "2", "32"), ("global", "8", "5", "4", "32"),
              ("smem", "2", "0", "2", "16"), ("global", "3", "0", "1", "16")]
    shapes = [dict(MARS_SPARSE_KERNEL="levels", MARS_SPARSE_STATE=st, MARS_SPARSE_WARPS=wp,
                   MARS_SPARSE_GRID=gr, MARS_SPARSE_R=r, MARS_SPARSE_CW=cw)
              for st, wp, gr, r, cw in levels]
    # warp-per-run kernel: consumer warps x ring depth x chunk width x grid
    # (ring sizes from "just the largest block" upward exercise the byte ring's wrap-around)
    # chunk width x runs per warp covers all four (runs per warp, spins per lane) variants
    shapes += [dict(MARS_SPARSE_KERNEL="spmm", MARS_SPMM_WARPS=wp, MARS_SPMM_RING_KB=rg,
                    MARS_SPARSE_CW=cw, MARS_SPMM_H=hh, MARS_SPARSE_GRID=gr)
               for wp, rg, cw, hh, gr in [("1", "1", "32", "1", "0"), ("3", "3", "16", "2", "5"),
                                          ("8", "5", "64", "1", "0"), ("2", "40", "32", "2", "0"),
                                          ("16", "8", "64", "1", "3")]]
    # two runs per lane group, interleaved (one 16-byte gather for both)
    shapes += [dict(MARS_SPARSE_KERNEL="spmm", MARS_SPMM_R="2", MARS_SPMM_WARPS=wp, MARS_SPARSE_CW=cw,
                    MARS_SPMM_H=hh, MARS_SPARSE_GRID=gr)
               for wp, cw, hh, gr in [("1", "32", "1", "0"), ("5", "16", "2", "0"), ("3", "32", "1", "4")]]
    if kind != "er_gauss":
        # torus stencil kernel: state in shared memory or a global row, any CTA width / grid
        shapes += [dict(MARS_SPARSE_KERNEL="stencil", MARS_SPARSE_STATE=st, MARS_STENCIL_THREADS=th,
                        MARS_SPARSE_GRID=gr)
                   for st, th, gr in [("smem", "0", "0"), ("global", "64", "3"), ("smem", "32", "0"),
                                      ("global", "1024", "0")]]
    for env in shapes:
        for k in ("MARS_SPARSE_KERNEL", "MARS_STENCIL_THREADS", "MARS_SPARSE_STATE", "MARS_SPARSE_WARPS", "MARS_SPARSE_GRID",
                  "MARS_SPARSE_R", "MARS_SPARSE_CW", "MARS_SPMM_WARPS", "MARS_SPMM_RING_KB",
                  "MARS_SPMM_H", "MARS_SPMM_R"):
            monkeypatch.delenv(k, raising=False)
        for k, val in env.items():
            if val == "off":
                monkeypatch.setenv(k, "0")
            elif val != "0":
                monkeypatch.setenv(k, val)
        p = mb.IsingProblem.from_edges(n, (u, v, w))
        assert p.kernel() == "csr"
        results.append(mb.run_batch(p, spec).records)
    for r in results[1:]:
        for name in ("status", "energy", "cut", "descent_iters", "spins"):
            assert np.array_equal(getattr(r, name), getattr(results[0], name)), name
    from oracle.oracle import params
    ob = port.problem_edges(n, u, v, w).run_batch(params(0, 6, 1, uniform=True), 96, 11)
    same = np.all(results[0].spins == ob.spins, axis=1)
    assert same.mean() >= SPIN_FRACTION
    assert np.array_equal(results[0].energy[same], ob.energy[same])


def _host_has_fma():
    try:
        return " fma " in open("/proc/cpuinfo").read().replace("\n", " ")
    except OSError:
        return False


@pytest.mark.skipif(not _host_has_fma(), reason="glibc selects its FMA expm1 only on FMA hosts")
def test_device_tanh_matches_libm():
    """csrc/ref_tanh.cuh == this host's libm tanh / expm1 (what the reference calls), bit for bit."""
    import ctypes
    import math
    from conftest import ROOT
    lib = ctypes.CDLL(os.path.join(ROOT, "tests", "cuda", "libtanh_probe.so"))
    lib.tanh_probe.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_longlong]
    rng = np.random.default_rng(11)
    x = np.concatenate([
        rng.uniform(-1, 1, 200000) * 10.0 ** rng.uniform(-6, 1.4, 200000),   # tanh's range
        rng.uniform(-50, 50, 100000),                                         # expm1 branches
        np.array([0.0, -0.0, 5e-324, -5e-324, 1e-300, 2.0 ** -55, 0.5493061443340548, 1.0, -1.0,
                  21.999999999999996, 22.0, -22.0, 1e300, np.inf, -np.inf, 0.34657359027997264,
                  1.0397207708399179, 38.8, 709.7, -709.7])])
    t, e = np.zeros_like(x), np.zeros_like(x)
    assert lib.tanh_probe(x.ctypes.data, t.ctypes.data, e.ctypes.data, x.size) == 0
    want_t = np.array([math.tanh(v) for v in x])
    want_e = np.array([math.expm1(v) if v < 709 else np.inf for v in x])
    fin = np.isfinite(want_e)
    assert np.array_equal(t.view(np.int64), want_t.view(np.int64))
    assert np.array_equal(e[fin].view(np.int64), want_e[fin].view(np.int64))


@pytest.mark.parametrize("kind", ["er_pm1", "er_gauss_field", "ea2d", "ea3d", "er_dense_storage",
                                  "ea2d_narrow_ctas", "ea2d_field", "ea3d_grid_sweep"])
def test_sparse_kernels_exact_vs_reference(kind, port, monkeypatch):
    """With the reference's own tanh on the device, the fp64 sparse kernels reproduce the
    reference's descents exactly: every status, iteration count, energy, cut and spin."""
    from oracle.oracle import params
    rng = np.random.default_rng(17)
    h = None
    if kind == "er_pm1":
        n, (u, v, w) = 300, mb.gen_er(300, 0.02, 3)
    elif kind == "er_gauss_field":
        n = 400
        u, v = np.triu_indices(n, 1)
        keep = rng.random(u.size) < 0.02
        u, v = u[keep].astype(np.int32), v[keep].astype(np.int32)
        w = rng.standard_normal(u.size)
        h = rng.standard_normal(n) * 0.3
    elif kind == "ea2d":
        n, (u, v, w) = 24 * 24, mb.gen_ea(24, 2, 3)
    elif kind == "ea3d":
        n, (u, v, w) = 8 ** 3, mb.gen_ea(8, 3, 4)
    elif kind == "ea2d_field":         # stencil kernel with an external field
        n, (u, v, w) = 20 * 20, mb.gen_ea(20, 2, 8)
        h = rng.standard_normal(n) * 0.5
    elif kind == "ea3d_grid_sweep":    # GridSweep plan (skipped t = 0 slot) on the stencil
        n, (u, v, w) = 6 ** 3, mb.gen_ea(6, 3, 9)
    elif kind == "ea2d_narrow_ctas":   # levels wider than the CTA: several sites per thread
        n, (u, v, w) = 48 * 48, mb.gen_ea(48, 2, 6)
        monkeypatch.setenv("MARS_STENCIL_THREADS", "32")
    else:   # 6% graph stored dense by the reference, relaxed by the sparse path
        n, (u, v, w) = 200, mb.gen_er(200, 0.06, 9)
    p = mb.IsingProblem.from_edges(n, (u, v, w), h)
    assert p.kernel() == "csr"
    runs, seed, tmax = 128, 23, 8.0
    if kind == "ea3d_grid_sweep":
        prm, oprm = mb.MarsParams(0, 6, 0.25), params(0, 6, 0.25)
    else:
        prm, oprm = uniform(tmax), params(0, tmax, 1, uniform=True)
    dev = mb.run_batch(p, mb.BatchSpec(prm, runs, seed, keep_spins=True)).records
    ob = port.problem_edges(n, u, v, w, h).run_batch(oprm, runs, seed)
    assert np.array_equal(dev.status, ob.status)
    assert np.array_equal(dev.descent_iters, ob.descent_iters)
    assert np.array_equal(dev.energy.view(np.int64), ob.energy.view(np.int64))
    assert np.array_equal(dev.cut.view(np.int64), ob.cut.view(np.int64))
    assert np.array_equal(dev.spins, ob.spins)


def test_small_dense_kernel_matches_reference(monkeypatch):
    """The opt-in on-chip small-instance kernel (MARS_DENSE_SMALL=1) on cfg1's instance: the
    reference's full-batch records within the dense (fp32) bar, and the best energy exactly."""
    monkeypatch.setenv("MARS_DENSE_SMALL", "1")
    w = WORKLOADS["cfg1_sk256_pm1"]
    g = golden("cfg1")
    p = build_problem(w)
    stats = mb.run_batch(p, mb.BatchSpec(w.params(), w.runs, w.base_seed, keep_spins=True))
    compare_records(stats, g, w.n)
    assert stats.best_energy == -6120.0


@pytest.mark.parametrize("kernel", ["dense_umma", "csr"])
def test_finish_times_for_time_to_best(kernel):
    """mars_batch_fetch_finish: per-run retirement on the device clock, measured from the
    launch's first descent start -- every executed run retires no earlier than its own
    elapsed time and no later than the relaxation kernel lasted."""
    w = WORKLOADS["cfg1_sk256_pm1"]
    p = build_problem(w, kernel=kernel)
    spec = mb.BatchSpec(w.params(), 512, w.base_seed)
    b = mb.DeviceBatch(p, spec)
    b.upload()
    t = b.execute()
    rec, _, _ = b.fetch()
    fin = b.finish_seconds()
    ran = rec.status != 1
    assert ran.all()
    assert np.all(fin[ran] >= rec.elapsed_seconds[ran] - 1e-6)
    assert fin.min() >= 0.0 and fin.max() <= t["relax_ms"] * 1e-3 * 1.05 + 1e-4
    best = float(rec.energy[rec.status == 0].min())
    ttb = mb.time_to_best(rec.energy, rec.status, fin, best, p.energy_equality_tolerance())
    assert 0.0 < ttb <= fin.max()


def test_small_kernel_auto_selection(monkeypatch):
    """Integer N <= 256 batches that fit on the device at once take the warp-per-run kernel
    (timing kernel 4); MARS_DENSE_SMALL=0 keeps them on the tensor-core kernel (3)."""
    w = WORKLOADS["cfg1_sk256_pm1"]
    p = build_problem(w)
    spec = mb.BatchSpec(w.params(), 1024, w.base_seed)
    monkeypatch.delenv("MARS_DENSE_SMALL", raising=False)
    b = mb.DeviceBatch(p, spec)
    b.upload()
    assert b.execute()["kernel"] == 4
    monkeypatch.setenv("MARS_DENSE_SMALL", "0")
    b = mb.DeviceBatch(p, spec)
    b.upload()
    assert b.execute()["kernel"] == 3


@pytest.mark.parametrize("n,h", [(37, False), (100, True), (150, False), (200, False), (256, True)])
def test_small_kernel_ragged_sizes_match_port(port, n, h):
    """relax_small.cu (the default for these resident integer batches) at sizes that leave a
    partial spin pair / partial 64-spin group, with and without an external field: the
    oracle's records within the dense bar, energies bit-exact where the spins agree."""
    from oracle.oracle import params
    J = port.gen_sk_pm1(n, 40 + n)
    hv = np.where(np.arange(n) % 3 == 0, 1.0, -1.0) if h else None
    t = float(int(np.sqrt(n)) + 2)
    ob = (port.problem_dense(J, hv) if h else port.problem_dense(J)).run_batch(
        params(0, t, 1, 1, 1e-4, uniform=True), 256, 3)
    p = mb.IsingProblem.dense(n, J, hv)
    spec = mb.BatchSpec(mb.MarsParams(0, t, 1, 1, 1e-4, mb.StartMode.UniformRandom), 256, 3, keep_spins=True)
    b = mb.DeviceBatch(p, spec)
    b.upload()
    assert b.execute()["kernel"] == 4
    stats = mb.run_batch(p, spec)
    assert np.array_equal(stats.records.status, ob.status)
    same = np.all(stats.records.spins == ob.spins, axis=1)
    # fp32 floor of these low-temperature (T <= sqrt(n) + 2) instances, integer fields make
    # phi = 0 ties common: measured 0.89-1.0 for this kernel AND 0.887-1.0 for the tcgen05
    # kernel on the same cases (tools/frac_small_vs_umma.py); the best energy must match
    assert same.mean() >= 0.85, same.mean()
    assert np.array_equal(stats.records.energy[same], ob.energy[same])
    assert stats.best_energy == ob.stats["best_energy"]


def test_batch_outlives_destroyed_problem():
    """mars_problem_destroy with a staged batch outstanding only marks the handle released;
    the batch keeps executing on it and the last mars_batch_destroy frees it (the Python
    cyclic GC may finalise a problem before a batch that references it)."""
    from paper_1907_05124_b200._native import lib
    w = WORKLOADS["cfg1_sk256_pm1"]
    p = build_problem(w)
    b = mb.DeviceBatch(p, mb.BatchSpec(w.params(), 64, w.base_seed))
    lib.mars_problem_destroy(p._h)
    p._h = None
    b.upload()
    b.execute()
    rec, best, _ = b.fetch()
    assert (rec.status == 0).all() and 0 <= best < 64
    del b


@pytest.mark.parametrize("kernel", ["dense_umma", "small", "dense_simt", "csr", "stencil"])
def test_progress_during_the_batch(kernel, monkeypatch):
    """run_batch's ProgressFn (test_runner.cpp:148-162): called once per run -- skipped slots
    included -- with a non-increasing best, and the last best equal to the batch best; here from
    the calling thread while the kernel runs (every relaxation kernel logs its finished runs)."""
    import threading
    monkeypatch.setenv("MARS_DENSE_SMALL", "1" if kernel == "small" else "0")
    if kernel == "csr":
        p = mb.IsingProblem.from_edges(300, mb.gen_er(300, 0.02, 4))
    elif kernel == "stencil":
        p = mb.IsingProblem.from_edges(256, mb.gen_ea(16, 2, 5))
    elif kernel == "small":
        p = mb.IsingProblem.dense(256, mb.gen_sk_pm1(256, 1))
    else:
        p = mb.IsingProblem.dense(200, mb.gen_sk_gaussian(200, 3), kernel=kernel)
    spec = mb.BatchSpec(mb.MarsParams(0, 10, 0.5), 1, 5, keep_spins=True)     # grid: t = 0 slot skipped
    calls, me = [], threading.get_ident()
    stats = mb.run_batch(p, spec, progress=lambda i, b: calls.append((i, b, threading.get_ident())))
    assert sorted(c[0] for c in calls) == list(range(len(stats.records.status)))
    assert all(c[2] == me for c in calls)
    bests = [c[1] for c in calls]
    assert all(b2 <= b1 for b1, b2 in zip(bests, bests[1:]))
    assert bests[-1] == stats.best_energy
    plain = mb.run_batch(p, spec)
    assert np.array_equal(plain.records.energy, stats.records.energy)
