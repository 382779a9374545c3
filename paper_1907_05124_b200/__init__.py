"""B200-native MARS (Mean-field Annealing from a Random State, arXiv 1907.05124).

The hot path -- a massively parallel batch of independent MARS mean-field descents -- as
hand-written sm_100a CUDA behind a C-ABI (include/mars_b200.h), with this package as the
host-side mirror of the reference's solver API (model.hpp / solvers.hpp / runner.hpp).
"""
from .mars import (  # noqa: F401
    BatchSpec, BatchStats, CudaError, GroundState, brute_force_ground_state, DeviceBatch, DivergedError, Error, InputError,
    IsingProblem, MarsParams, MarsRunPlan, Records, RunResult, RunStatus, StartMode,
    aggregate, cut_value, distributed_batch, energy, gen_ea, gen_er, gen_sk_gaussian,
    gen_sk_pm1, generate_sk, initial_state, mars_grid_count, mars_grid_temp, mars_run_count,
    mars_run_plan, mars_sweep, round_spins, run_batch, run_batch_with, run_shard, shard_range,
    splitmix64, sub_seed, time_to_best, validate,
)
from . import io  # noqa: F401,E402  (instance I/O and result documents, io.hpp mirror)
