"""Generates the committed golden fixtures in tests/golden/ from the REFERENCE itself.

    make -C oracle && python tests/golden/make_golden.py

Every vector here is an output of oracle/_ref/libmars_ref.so -- the reference's own
model.cpp / solvers.cpp / runner.cpp compiled from /root/reference/proj/src -- run in this
container (the reference does not exist on the GPU box, so its outputs travel as these
fixtures).  The reference ships no golden vectors of its own; its one
frozen constant, splitmix64(0) == 0xE220A8397B1DCDAF (tests/test_io.cpp:157), is included.
"""
from __future__ import annotations

import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import Oracle, params  # noqa: E402
from paper_1907_05124_b200.workloads import WORKLOADS, build_oracle_problem  # noqa: E402

R = Oracle("ref")


def save(name, **arrays):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrays)
    print(f"{name}.npz  {os.path.getsize(path) / 1024:.1f} KiB")


def batch_arrays(prefix, b, n_spins_keep=None):
    out = {
        prefix + "status": b.status, prefix + "energy": b.energy, prefix + "cut": b.cut,
        prefix + "start_temp": b.start_temp, prefix + "iters": b.descent_iters,
    }
    if b.spins is not None:
        sp = b.spins if n_spins_keep is None else b.spins[:n_spins_keep]
        out[prefix + "spins_packed"] = np.packbits(sp > 0, axis=1)
    st = b.stats
    out[prefix + "stats"] = np.array([st["best_energy"], st["mean_energy"], st["best_cut"],
                                      st["mean_cut"], st["hit_count"], st["success_probability"],
                                      st["best_index"], st["completed_runs"], st["skipped_runs"],
                                      st["failed_runs"]], np.float64)
    return out


def rng():
    out = {"splitmix_in": np.array([0, 1, 2, 12345, 2**63, 2**64 - 1], np.uint64)}
    out["splitmix_out"] = np.array([R.splitmix64(int(x)) for x in out["splitmix_in"]], np.uint64)
    out["sub_seed"] = np.array([[R.sub_seed(b, i) for i in range(16)] for b in (0, 1, 7, 99)],
                               np.uint64)
    for kind, name in enumerate(["u64", "open01", "open_sym", "gaussian", "coin"]):
        out["draw_" + name] = np.stack([R.draws(s, kind, 1000) for s in (0, 1, 42)])
    out["draw_below7"] = np.stack([R.draws(s, 5, 1000, 7) for s in (0, 1, 42)])
    pu = params(0, 16, 1, 1, 1e-4, uniform=True)
    pg = params(0, 10, 0.05, 1, 1e-4)
    out["plan_uniform"] = np.array([R.run_plan(pu, 1, k) for k in range(1024)],
                                   dtype=[("skipped", "?"), ("t", "f8"), ("seed", "u8")])
    out["plan_grid"] = np.array([R.run_plan(pg, 99, k) for k in range(201)],
                                dtype=[("skipped", "?"), ("t", "f8"), ("seed", "u8")])
    out["init_state_seed"] = np.array([R.sub_seed(1, k) for k in range(4)], np.uint64)
    out["init_state"] = np.stack([R.initial_state(int(s), 2000) for s in out["init_state_seed"]])
    save("rng", **out)


def instances():
    out = {}
    J1 = R.gen_sk_pm1(256, 1)
    out["cfg1_J_packed"] = np.packbits(J1 > 0, axis=1)
    J2 = R.gen_sk_gaussian(2000, 7)
    out["cfg2_rowsum"] = J2.sum(axis=1)
    out["cfg2_corner"] = np.concatenate([J2[0, :64], J2[1999, -64:], J2[1000, 900:964]])
    for name in ("cfg3a_er800", "cfg3b_er2000"):
        w = WORKLOADS[name]
        u, v, wt = R.gen_er(w.n, w.prob, w.seed)
        out[name + "_uv"] = np.stack([u, v])
    for name in ("cfg4_ea2d", "cfg4_ea3d"):
        w = WORKLOADS[name]
        u, v, wt = R.gen_ea(w.L, w.dims, w.seed)
        out[name + "_w_packed"] = np.packbits(wt > 0)
        out[name + "_v_head"] = v[:4096]
    out["sk12_4001"] = R.gen_sk_gaussian(12, 4001)
    save("instances", **out)


def cfg1():
    w = WORKLOADS["cfg1_sk256_pm1"]
    p = build_oracle_problem(R, w)
    pr = params(0, w.t_max, 1, 1, 1e-4, uniform=True)
    t = time.time()
    b = p.run_batch(pr, w.runs, w.base_seed, workers=0)
    print(f"cfg1 reference batch {time.time() - t:.1f}s best {b.stats['best_energy']}")
    out = batch_arrays("", b)
    out["coupling_sum"] = np.array([p.coupling_sum])
    save("cfg1", **out)


def prefix(name, runs, keep=None, t_max=None, tag="_prefix"):
    w = WORKLOADS[name]
    p = build_oracle_problem(R, w)
    pr = params(0, w.t_max if t_max is None else t_max, 1, 1, 1e-4, uniform=True)
    t = time.time()
    b = p.run_batch(pr, runs, w.base_seed, workers=0)
    print(f"{name} prefix {runs} runs {time.time() - t:.1f}s best {b.stats['best_energy']} "
          f"mean iters {b.descent_iters.mean():.1f} adjacency {p.uses_adjacency}")
    out = batch_arrays("", b, keep)
    out["coupling_sum"] = np.array([p.coupling_sum])
    out["wall_seconds"] = np.array([time.time() - t])
    save(name + tag, **out)


def small():
    out = {}
    # test_solvers.cpp:150-173 -- generate_sk(12, 4001), grid [0,10] step 0.05, seed 99
    p = R.problem_dense(R.gen_sk_gaussian(12, 4001))
    out.update(batch_arrays("grid12_", p.run_batch(params(0, 10, 0.05), 1, 99)))
    # test_runner.cpp:60-69 -- generate_sk(24, 71), grid [0,12] step 1, seed 9
    p = R.problem_dense(R.gen_sk_gaussian(24, 71))
    out.update(batch_arrays("grid24_", p.run_batch(params(0, 12, 1), 1, 9)))
    # acceptance.cpp:262-297 -- generate_sk(60, 99), grid [0,16] step 0.25, seed 41
    p = R.problem_dense(R.gen_sk_gaussian(60, 99))
    out.update(batch_arrays("grid60_", p.run_batch(params(0, 16, 0.25), 1, 41)))
    # ferromagnetic pair (test_solvers.cpp:71-81)
    p = R.problem_dense(np.array([[0.0, -1.0], [-1.0, 0.0]]))
    out.update(batch_arrays("ferro_", p.run_batch(params(0, 30, 1), 1, 77)))
    # integer couplings in [-3,3] with an integer field in [-2,2] (support.hpp:64-77 shape)
    n = 20
    dj = R.draws(5, 5, n * (n - 1) // 2, 7).astype(np.int64) - 3
    J = np.zeros((n, n))
    J[np.triu_indices(n, 1)] = dj
    J = J + J.T
    h = (R.draws(6, 5, n, 5).astype(np.int64) - 2).astype(np.float64)
    out["int20_J"] = J
    out["int20_h"] = h
    p = R.problem_dense(J, h)
    out.update(batch_arrays("int20_", p.run_batch(params(0, 20, 1, uniform=True), 256, 3)))
    # sparse storage with a field: ER(200, 2%) +-1 weights, h +-1
    u, v, _ = R.gen_er(200, 0.02, 31)
    wts = R.draws(32, 4, len(u))
    hs = R.draws(33, 4, 200)
    out["er200_u"], out["er200_v"], out["er200_w"], out["er200_h"] = u, v, wts, hs
    p = R.problem_edges(200, u, v, wts, hs)
    assert p.uses_adjacency
    out.update(batch_arrays("er200_", p.run_batch(params(0, 10, 1, uniform=True), 256, 4)))
    # EA 2D L=16 (CSR)
    u, v, wts = R.gen_ea(16, 2, 5)
    p = R.problem_edges(256, u, v, wts)
    out.update(batch_arrays("ea16_", p.run_batch(params(0, 4, 1, uniform=True), 256, 1)))
    # single-sweep unit checks at high T: one relax_sweep from a seeded state
    J2 = R.gen_sk_gaussian(2000, 7)
    p2 = R.problem_dense(J2)
    for T in (40.0, 20.0):
        s = R.initial_state(4242, 2000)
        d = p2.relax_sweep(s, T)
        out[f"sweep2000_T{int(T)}"] = s
        out[f"sweep2000_T{int(T)}_d"] = np.array([d])
    p1 = R.problem_dense(R.gen_sk_pm1(256, 1))
    s = R.initial_state(4242, 256)
    out["sweep256_T16_d"] = np.array([p1.relax_sweep(s, 16.0)])
    out["sweep256_T16"] = s
    save("small", **out)


def sweeps():
    """Single-sweep trajectory fixtures (SURVEY.md 8(c) "per-sweep unit check"): one
    mars_relax_sweep (solvers.cpp:150-161) of the reference from fp32-representable states
    (so the device, which takes fp32 states, starts from the identical point), at the
    temperatures of the cfg1 / cfg2 / cfg5 schedules.  Inputs are regenerated from the seeds
    with mars_initial_state (pinned by rng.npz); outputs are stored as fp32 (the gate is 5e-5)."""
    out = {}
    cases = [("sk2000", lambda: R.gen_sk_gaussian(2000, 7), 2000, (40.0, 20.0, 5.0), 8),
             ("pm256", lambda: R.gen_sk_pm1(256, 1), 256, (16.0, 8.0, 1.0), 8),
             ("sk16384", lambda: R.gen_sk_gaussian(16384, 7), 16384, (115.0, 60.0), 2)]
    for name, gen, n, temps, nseeds in cases:
        t = time.time()
        p = R.problem_dense(gen())
        seeds = np.array([R.sub_seed(4242, k) for k in range(nseeds)], np.uint64)
        out[name + "_seeds"] = seeds
        out[name + "_temps"] = np.array(temps)
        res = np.zeros((len(temps), nseeds, n), np.float32)
        ds = np.zeros((len(temps), nseeds))
        for ti, T in enumerate(temps):
            for k, sd in enumerate(seeds):
                s = R.initial_state(int(sd), n).astype(np.float32).astype(np.float64)
                ds[ti, k] = p.relax_sweep(s, T)
                res[ti, k] = s
        out[name + "_out"] = res
        out[name + "_d"] = ds
        # the fp32 floor: the same sweep in fp32 (C port, ascending-j fp32 row dots, tanhf)
        P = Oracle("port")
        pp = P.problem_dense(gen())
        f32 = np.zeros((len(temps), nseeds))
        for ti, T in enumerate(temps):
            for k, sd in enumerate(seeds):
                s = R.initial_state(int(sd), n).astype(np.float32)
                pp.relax_sweep_f32(s, T)
                f32[ti, k] = np.abs(s.astype(np.float64) - res[ti, k]).max()
        out[name + "_f32err"] = f32
        print(f"sweeps {name}: {time.time() - t:.1f}s")
    save("sweeps", **out)


def replay_f32():
    """The fp32 floor of the dense Gaussian path: the reference's first 256 cfg2 descents
    replayed by the C port with fp32 state/fields/tanh (oracle/mars_oracle.c
    orc_replay_batch_f32) -- how many end on the reference's spins when only the arithmetic
    precision changes.  The device gate in tests/test_gpu_parity.py is set from this."""
    P = Oracle("port")
    w = WORKLOADS["cfg2_sk2000"]
    p = build_oracle_problem(P, w)
    pr = params(0, w.t_max, 1, 1, 1e-4, uniform=True)
    t = time.time()
    st, it, sp = p.replay_f32(pr, 256, w.base_seed, 0, 0)
    print(f"cfg2 fp32 replay 256 runs {time.time() - t:.1f}s")
    save("cfg2_sk2000_f32replay", status=st, iters=it, spins_packed=np.packbits(sp > 0, axis=1))


if __name__ == "__main__":
    which = sys.argv[1:] or ["rng", "instances", "small", "cfg1", "prefixes"]
    if "rng" in which:
        rng()
    if "instances" in which:
        instances()
    if "small" in which:
        small()
    if "cfg1" in which:
        cfg1()
    if "sweeps" in which:
        sweeps()
    if "replay" in which:
        replay_f32()
    if "cfg2" in which:
        prefix("cfg2_sk2000", 256)
    if "cfg5" in which:
        # cfg5's instance (N = 16384) on a short schedule (t_max = 3): the first 16 descents of
        # the reference (~1 min per descent per core)
        prefix("cfg5_sk16384", 16, t_max=3.0, tag="_t3_prefix")
    if "prefixes" in which:
        prefix("cfg2_sk2000", 256)
        prefix("cfg3a_er800", 256)
        prefix("cfg3b_er2000", 256)
        prefix("cfg4_ea2d", 16)
        prefix("cfg4_ea3d", 8)
