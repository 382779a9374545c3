"""ctypes binding of the C-ABI in include/mars_b200.h (libmars_b200.so, built in-tree).

There is no fallback: if the native library is missing this module raises ImportError,
and every compute entry point runs the sm_100a kernels (problem creation fails with a
CUDA error when no device is present).
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# MARS_B200_LIB names an alternative build next to this file (A/B kernel experiments)
LIB_PATH = os.path.join(HERE, os.path.basename(os.environ.get("MARS_B200_LIB") or "libmars_b200.so"))

if not os.path.exists(LIB_PATH):
    raise ImportError(f"{LIB_PATH} is missing: build it with "
                      "`python -m paper_1907_05124_b200._build` (nvcc, sm_100a)")

lib = C.CDLL(LIB_PATH)

MARS_OK, MARS_ERR_INPUT, MARS_ERR_RUNTIME, MARS_ERR_CUDA, MARS_ERR_NCCL, MARS_ERR_ALL_FAILED = range(6)
MARS_KERNEL_AUTO, MARS_KERNEL_DENSE_SIMT, MARS_KERNEL_CSR, MARS_KERNEL_DENSE_UMMA = range(4)


class mars_params_t(C.Structure):
    _fields_ = [("t_min", C.c_double), ("t_max", C.c_double), ("t_step", C.c_double),
                ("c_step", C.c_double), ("d_min", C.c_double), ("start_mode", C.c_int32),
                ("reserved", C.c_int32), ("sweep_cap", C.c_int64)]


class mars_problem_info_t(C.Structure):
    _fields_ = [("n", C.c_int32), ("uses_adjacency", C.c_int32), ("integral", C.c_int32),
                ("has_field", C.c_int32), ("coupling_sum", C.c_double), ("nonzeros", C.c_int64),
                ("device", C.c_int32), ("kernel", C.c_int32), ("levels", C.c_int32),
                ("reserved", C.c_int32)]


class mars_records_t(C.Structure):
    _fields_ = [("status", C.c_void_p), ("energy", C.c_void_p), ("cut", C.c_void_p),
                ("start_temp", C.c_void_p), ("descent_iters", C.c_void_p),
                ("elapsed_seconds", C.c_void_p), ("spins", C.c_void_p), ("fail_temp", C.c_void_p)]


class mars_stats_t(C.Structure):
    _fields_ = [("best_energy", C.c_double), ("mean_energy", C.c_double),
                ("best_cut", C.c_double), ("mean_cut", C.c_double), ("hit_count", C.c_int64),
                ("success_probability", C.c_double), ("total_seconds", C.c_double),
                ("mean_seconds_per_run", C.c_double), ("best_index", C.c_int64),
                ("completed_runs", C.c_int64), ("skipped_runs", C.c_int64),
                ("failed_runs", C.c_int64)]


class mars_timing_t(C.Structure):
    _fields_ = [("relax_ms", C.c_double), ("energy_ms", C.c_double), ("reduce_ms", C.c_double),
                ("total_ms", C.c_double), ("launches", C.c_int64), ("total_sweeps", C.c_int64),
                ("grid", C.c_int32), ("slots", C.c_int32), ("kernel", C.c_int32), ("split", C.c_int32)]


class mars_nmfa_params_t(C.Structure):
    _fields_ = [("noise_sigma", C.c_double), ("alpha", C.c_double), ("iters", C.c_int64),
                ("schedule", C.c_void_p), ("schedule_len", C.c_int64)]


class mars_simcim_params_t(C.Structure):
    _fields_ = [("step_size", C.c_double), ("noise_sigma", C.c_double), ("iters", C.c_int64),
                ("pump_schedule", C.c_void_p), ("pump_schedule_len", C.c_int64)]


vp, i32, i64, u64, dbl = C.c_void_p, C.c_int32, C.c_int64, C.c_uint64, C.c_double
PROGRESS_FN = C.CFUNCTYPE(None, C.c_int64, C.c_double, C.c_void_p)   # progress(index, best, user)
P_params = C.POINTER(mars_params_t)

# name -> (restype, argtypes): exactly the declarations of include/mars_b200.h
SIGNATURES = {
    "mars_last_error": (C.c_char_p, []),
    "mars_device_count": (C.c_int, [vp]),
    "mars_problem_dense": (C.c_int, [i32, vp, vp, i32, i32, C.POINTER(vp)]),
    "mars_problem_from_edges": (C.c_int, [i32, i64, vp, vp, vp, vp, i32, i32, C.POINTER(vp)]),
    "mars_problem_destroy": (None, [vp]),
    "mars_problem_info": (C.c_int, [vp, C.POINTER(mars_problem_info_t)]),
    "mars_problem_hash": (C.c_int, [vp, vp]),
    "mars_instance_hash": (C.c_int, [i32, vp, i64, vp, vp, vp, vp, vp]),
    "mars_problem_rows": (C.c_int, [vp, vp]),
    "mars_brute_force": (C.c_int, [vp, i32, vp, vp]),
    "mars_energy": (C.c_int, [vp, vp, vp, vp]),
    "mars_validate_params": (C.c_int, [P_params]),
    "mars_run_count": (C.c_int, [P_params, i64, vp]),
    "mars_run_plan": (C.c_int, [P_params, u64, i64, vp, vp, vp]),
    "mars_initial_state": (C.c_int, [u64, i32, vp]),
    "mars_splitmix64": (u64, [u64]),
    "mars_sub_seed": (u64, [u64, u64]),
    "mars_run_batch": (C.c_int, [vp, P_params, i64, u64, C.POINTER(mars_records_t),
                                 C.POINTER(mars_stats_t), vp]),
    "mars_run_shard": (C.c_int, [vp, P_params, i64, u64, i64, i64, C.POINTER(mars_records_t)]),
    "mars_aggregate": (C.c_int, [i64, vp, vp, vp, vp, dbl, dbl, C.POINTER(mars_stats_t)]),
    "mars_batch_create": (C.c_int, [vp, P_params, i64, u64, i64, i64, C.POINTER(vp)]),
    "mars_batch_upload": (C.c_int, [vp]),
    "mars_batch_execute": (C.c_int, [vp, C.POINTER(mars_timing_t)]),
    "mars_debug_sweeps": (C.c_int, [vp, i64, vp, vp, i32, vp, vp]),
    "mars_debug_rng": (C.c_int, [vp, i32, i32, vp, vp]),
    "mars_run_batch_progress": (C.c_int, [vp, P_params, i64, u64, vp, vp, vp, vp, vp]),
    "mars_problem_replicate": (C.c_int, [vp, i32, C.POINTER(vp)]),
    "mars_run_batch_multi": (C.c_int, [vp, i32, P_params, i64, u64, vp, vp, vp]),
    "mars_debug_exchange": (C.c_int, [i32, i64, i32, vp, vp, vp, vp, vp, vp, dbl, vp, vp, vp]),
    "mars_debug_choose_split": (C.c_int, [vp, i64, P_params, i32, vp, i32, i32, i32, vp, vp]),
    "mars_run_batch_nmfa": (C.c_int, [vp, C.POINTER(mars_nmfa_params_t), i64, u64, vp, vp, vp]),
    "mars_run_batch_simcim": (C.c_int, [vp, C.POINTER(mars_simcim_params_t), i64, u64, vp, vp, vp]),
    "mars_batch_fetch": (C.c_int, [vp, C.POINTER(mars_records_t), vp, vp]),
    "mars_batch_fetch_finish": (C.c_int, [vp, vp]),
    "mars_batch_destroy": (None, [vp]),
    "mars_gen_sk_gaussian": (None, [i32, u64, vp]),
    "mars_gen_sk_pm1": (None, [i32, u64, vp]),
    "mars_gen_er": (i64, [i32, dbl, u64, vp, vp, vp]),
    "mars_gen_ea": (i64, [i32, i32, u64, vp, vp, vp]),
}

for _name, (_res, _args) in SIGNATURES.items():
    _fn = getattr(lib, _name)
    _fn.restype = _res
    _fn.argtypes = _args


def last_error() -> str:
    return (lib.mars_last_error() or b"").decode()


def ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)
