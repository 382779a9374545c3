"""The named workloads of BASELINE.json ``configs`` as frozen in SURVEY.md 8(d).

Instances are built only from the reference's seeded Rng primitives (product-side
generators in the native library, pinned bit-for-bit against the reference's own Rng by
tests/test_host.py), so the oracle and the device see identical couplings.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Workload:
    name: str
    kind: str          # "sk_pm1" | "sk_gauss" | "er" | "ea"
    n: int
    seed: int
    t_max: float
    runs: int
    base_seed: int = 1
    prob: float = 0.0  # er
    L: int = 0         # ea
    dims: int = 0      # ea
    note: str = ""

    def params(self):
        from .mars import MarsParams, StartMode
        return MarsParams(t_min=0.0, t_max=self.t_max, t_step=1.0, c_step=1.0, d_min=1e-4,
                          start_mode=StartMode.UniformRandom)

    def flops_per_sweep_run(self, nnz: int = 0) -> float:
        """Algorithmic flops of one Gauss-Seidel sweep of one run:
        2*N^2 dense (row_dot touches every column), 2*nnz sparse."""
        if self.kind in ("sk_pm1", "sk_gauss"):
            return 2.0 * self.n * self.n
        return 2.0 * nnz


WORKLOADS = {
    "cfg1_sk256_pm1": Workload("cfg1_sk256_pm1", "sk_pm1", 256, 1, 16.0, 1024,
                               note="SK N=256 +-1, 1024 descents (reference CPU parity case)"),
    "cfg2_sk2000": Workload("cfg2_sk2000", "sk_gauss", 2000, 7, 40.0, 65536,
                            note="dense SK N=2000 Gaussian, 65536 descents"),
    "cfg3a_er800": Workload("cfg3a_er800", "er", 800, 11, 30.0, 65536, prob=0.06,
                            note="G1-shape ER(800, 6%), dense storage"),
    "cfg3b_er2000": Workload("cfg3b_er2000", "er", 2000, 22, 40.0, 65536, prob=0.01,
                             note="G22-shape ER(2000, 1%), CSR storage"),
    "cfg4_ea2d": Workload("cfg4_ea2d", "ea", 128 * 128, 5, 4.0, 4096, L=128, dims=2,
                          note="EA +-J 2D torus L=128"),
    "cfg4_ea3d": Workload("cfg4_ea3d", "ea", 32 ** 3, 5, 6.0, 4096, L=32, dims=3,
                          note="EA +-J 3D torus L=32"),
    "cfg5_sk16384": Workload("cfg5_sk16384", "sk_gauss", 16384, 7, 115.0, 8192,
                             note="dense SK N=16384 Gaussian"),
}


def build_problem(w: Workload, device: int = 0, kernel: str = "auto"):
    """The workload's instance as a device-resident IsingProblem."""
    from . import mars as M
    if w.kind == "sk_pm1":
        return M.IsingProblem.dense(w.n, M.gen_sk_pm1(w.n, w.seed), device=device, kernel=kernel)
    if w.kind == "sk_gauss":
        return M.IsingProblem.dense(w.n, M.gen_sk_gaussian(w.n, w.seed), device=device, kernel=kernel)
    if w.kind == "er":
        return M.IsingProblem.from_edges(w.n, M.gen_er(w.n, w.prob, w.seed), device=device, kernel=kernel)
    if w.kind == "ea":
        return M.IsingProblem.from_edges(w.n, M.gen_ea(w.L, w.dims, w.seed), device=device, kernel=kernel)
    raise ValueError(w.kind)


def build_oracle_problem(orc, w: Workload):
    """The same instance in a CPU oracle (tests / CPU baseline only)."""
    if w.kind == "sk_pm1":
        return orc.problem_dense(orc.gen_sk_pm1(w.n, w.seed))
    if w.kind == "sk_gauss":
        return orc.problem_dense(orc.gen_sk_gaussian(w.n, w.seed))
    if w.kind == "er":
        return orc.problem_edges(w.n, *orc.gen_er(w.n, w.prob, w.seed))
    if w.kind == "ea":
        return orc.problem_edges(w.n, *orc.gen_ea(w.L, w.dims, w.seed))
    raise ValueError(w.kind)


def time_to_best(energy: np.ndarray, status: np.ndarray, finish: np.ndarray, best: float,
                 tol: float = 0.0) -> float:
    """Time-to-best: the earliest retirement among the completed runs whose
    energy is within ``tol`` of ``best`` (the reference's hit rule, runner.cpp:160-162);
    inf when none of these runs reaches it.  Pure numpy: bench.py's CPU reference arm uses it
    without loading the native library."""
    hit = (status == 0) & (np.abs(energy - best) <= tol)
    return float(finish[hit].min()) if hit.any() else float("inf")
