"""Product host logic that needs no GPU: seeding, plan, generators, validation and the
reference's aggregation (runner.cpp:126-167), checked against the golden fixtures and the
CPU oracle.  The device itself is never touched here."""
import numpy as np
import pytest

import paper_1907_05124_b200 as mb
from conftest import golden
from oracle.oracle import params
from paper_1907_05124_b200.mars import RunResult, RunStatus
from paper_1907_05124_b200.workloads import WORKLOADS


def test_seeding_matches_reference():
    g = golden("rng")
    assert mb.splitmix64(0) == 0xE220A8397B1DCDAF
    assert [mb.splitmix64(int(x)) for x in g["splitmix_in"]] == list(g["splitmix_out"])
    for b, row in zip((0, 1, 7, 99), g["sub_seed"]):
        assert [mb.sub_seed(b, i) for i in range(16)] == list(row)
    for s, row in zip(g["init_state_seed"], g["init_state"]):
        assert np.array_equal(mb.initial_state(int(s), 2000), row)


def test_plan_matches_reference():
    g = golden("rng")
    pu = mb.MarsParams(0, 16, 1, 1, 1e-4, mb.StartMode.UniformRandom)
    pg = mb.MarsParams(0, 10, 0.05, 1, 1e-4, mb.StartMode.GridSweep)
    for k, rec in enumerate(g["plan_uniform"]):
        p = mb.mars_run_plan(pu, 1, k)
        assert (p.skipped, p.start_temp, p.seed) == (bool(rec["skipped"]), float(rec["t"]), int(rec["seed"]))
    for k, rec in enumerate(g["plan_grid"]):
        p = mb.mars_run_plan(pg, 99, k)
        assert (p.skipped, p.start_temp, p.seed) == (bool(rec["skipped"]), float(rec["t"]), int(rec["seed"]))
    assert mb.mars_run_count(pg, 1) == 201                        # test_solvers.cpp:150-158
    assert mb.mars_grid_count(mb.MarsParams(0, 30, 1)) == 31       # test_solvers.cpp:129-134


def test_generators_match_oracle(port):
    assert np.array_equal(mb.gen_sk_pm1(256, 1), port.gen_sk_pm1(256, 1))
    assert np.array_equal(mb.gen_sk_gaussian(300, 7), port.gen_sk_gaussian(300, 7))
    for name in ("cfg3a_er800", "cfg3b_er2000"):
        w = WORKLOADS[name]
        for a, b in zip(mb.gen_er(w.n, w.prob, w.seed), port.gen_er(w.n, w.prob, w.seed)):
            assert np.array_equal(a, b)
    for name in ("cfg4_ea2d", "cfg4_ea3d"):
        w = WORKLOADS[name]
        for a, b in zip(mb.gen_ea(w.L, w.dims, w.seed), port.gen_ea(w.L, w.dims, w.seed)):
            assert np.array_equal(a, b)


@pytest.mark.parametrize("bad", [dict(t_min=-1.0), dict(t_max=0.0), dict(t_step=0.0),
                                 dict(c_step=0.0), dict(d_min=0.0)])
def test_validate_rejects_like_reference(bad, port):
    prm = mb.MarsParams(**bad)
    with pytest.raises(mb.InputError):
        mb.validate(prm)
    from oracle.oracle import OracleError
    with pytest.raises(OracleError):
        port.validate(params(prm.t_min, prm.t_max, prm.t_step, prm.c_step, prm.d_min))


def test_run_count_errors():
    with pytest.raises(mb.InputError):          # test_solvers.cpp:189-193, empty grid
        mb.mars_run_count(mb.MarsParams(0, 30, 40), 1)
    assert mb.mars_run_count(mb.MarsParams(3, 30, 40), 1) == 1
    with pytest.raises(mb.InputError):          # UniformRandom needs runs >= 1
        mb.mars_run_count(mb.MarsParams(2, 6, start_mode=mb.StartMode.UniformRandom), 0)


def test_aggregation_failure_injection():
    # test_runner.cpp:115-146: diverged idx 3, skipped idx 5, exception idx 7
    def run(idx):
        if idx == 3:
            return RunResult(status=RunStatus.Diverged, energy=-1e9)
        if idx == 5:
            return RunResult(status=RunStatus.Skipped)
        if idx == 7:
            raise RuntimeError("boom")
        return RunResult(energy=-float(idx % 4), cut=float(idx), spins=np.ones(6, np.int8))
    s = mb.run_batch_with(6, run, 10)
    assert (s.completed_runs, s.failed_runs, s.skipped_runs) == (7, 2, 1)
    ok = [k for k in range(10) if k not in (3, 5, 7)]
    energies = [-float(k % 4) for k in ok]
    assert list(s.energies) == energies
    assert s.best_energy == -2.0
    assert s.best_index == 2            # first strict minimum among completed (runner.cpp:147)
    assert s.mean_energy == sum(energies) / 7
    assert s.hit_count == 2 and s.success_probability == 2 / 7
    assert s.best_cut == 9.0
    assert s.records.status[7] == RunStatus.Diverged


def test_aggregation_all_failed_raises():
    with pytest.raises(mb.Error, match="no run completed"):
        mb.run_batch_with(4, lambda i: RunResult(status=RunStatus.Diverged), 3)


def test_aggregation_matches_reference_stats():
    # the oracle's stats of cfg1, recomputed from its records by the product aggregation
    g = golden("cfg1")
    rec = mb.Records(g["status"].copy(), g["energy"].copy(), g["cut"].copy(),
                     g["start_temp"].copy(), g["iters"].copy(), np.zeros(len(g["status"])))
    s = mb.aggregate(rec, 0.0, 0.0)
    st = g["stats"]
    assert [s.best_energy, s.mean_energy, s.best_cut, s.mean_cut, s.hit_count,
            s.success_probability, s.best_index, s.completed_runs, s.skipped_runs,
            s.failed_runs] == list(st)


def test_progress_callback_order():
    seen = []
    mb.run_batch_with(2, lambda i: RunResult(energy=float(5 - i)), 5,
                      progress=lambda i, b: seen.append((i, b)))
    assert seen == [(0, 5.0), (1, 4.0), (2, 3.0), (3, 2.0), (4, 1.0)]


def test_shard_ranges_cover_batch():
    for runs in (1, 7, 65536, 8193):
        for world in (1, 2, 3, 8):
            spans = [mb.shard_range(runs, r, world) for r in range(world)]
            assert spans[0][0] == 0
            for (f, c), (f2, _) in zip(spans, spans[1:]):
                assert f + c == f2
            assert sum(c for _, c in spans) == runs
