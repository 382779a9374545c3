"""B200-native MARS (Mean-field Annealing from a Random State, arXiv 1907.05124).

The hot path -- a massively parallel batch of independent MARS mean-field descents -- as
hand-written sm_100a CUDA behind a C-ABI (include/mars_b200.h), with this package as the
host-side mirror of the reference's solver API (model.hpp / solvers.hpp / runner.hpp).

The native library is loaded on first use of any solver name (PEP 562 module
``__getattr__``), so pure-Python helpers such as ``paper_1907_05124_b200.workloads`` can be
imported by the CPU reference arm of bench.py without mapping libmars_b200.so.  There is no
fallback: the first solver access raises ImportError when the library is missing.
"""
import importlib

_MARS_NAMES = (
    "BatchSpec", "BatchStats", "CudaError", "GroundState", "brute_force_ground_state", "DeviceBatch",
    "DivergedError", "Error", "InputError", "IsingProblem", "MarsParams", "MarsRunPlan", "Records",
    "RunResult", "RunStatus", "StartMode", "aggregate", "cut_value", "distributed_batch", "energy",
    "gen_ea", "gen_er", "gen_sk_gaussian", "gen_sk_pm1", "generate_sk", "initial_state",
    "mars_grid_count", "mars_grid_temp", "mars_run_count", "mars_run_plan", "mars_sweep",
    "round_spins", "run_batch", "run_batch_with", "run_shard", "shard_range",
    "splitmix64", "sub_seed", "time_to_best", "validate", "debug_sweep",
    "NmfaParams", "SimCimParams", "run_batch_multi", "debug_exchange", "nmfa_defaults", "simcim_defaults", "linear_schedule", "schedule_at",
    "debug_choose_split",
)

__all__ = list(_MARS_NAMES) + ["io", "mars", "workloads"]


def __getattr__(name):
    if name in ("io", "mars", "workloads", "_native"):
        return importlib.import_module(f".{name}", __name__)
    if name in _MARS_NAMES:
        return getattr(importlib.import_module(".mars", __name__), name)
    raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
