"""Host-side mirror of the reference's MARS solver API, driving the B200 kernels.

Same names, argument meaning and error behaviour as the reference headers
(/root/reference/proj/include/mars/{model,solvers,runner}.hpp), so a caller of
``mars::run_batch(problem, spec)`` finds the same call here:

    problem = IsingProblem.dense(n, J)            # model.hpp:41   (copies J to the GPU)
    spec = BatchSpec(MarsParams(t_min=0, t_max=40, start_mode=StartMode.UniformRandom),
                     runs=65536, base_seed=1)     # runner.hpp:19-24
    stats = run_batch(problem, spec)              # runner.hpp:55  -> BatchStats

Every descent runs in the persistent sm_100a relaxation kernel, energies in the exact-order
fp64 kernel, and best-of-R in the device reduction; this module only plans, marshals and
aggregates (runner.cpp:126-167, via the native ``mars_aggregate``).  Under
``torch.distributed`` with world_size > 1, ``run_batch`` shards the run indices
contiguously over the ranks (one GPU per process), gathers the per-run records and
broadcasts the winning spins (NCCL over NVLink when the backend is nccl).
"""
from __future__ import annotations

import ctypes as C
import enum
import time
from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np

from . import _native as N
from ._native import lib, ptr
from .workloads import time_to_best  # noqa: F401  (pure numpy; re-exported)


# ---------------------------------------------------------------- errors (errors.hpp:11-50)

class Error(RuntimeError):
    """mars::Error -- base class of everything the library raises on purpose."""


class InputError(Error):
    """mars::InputError -- invalid arguments or parameters."""


class CudaError(Error):
    """The device path failed (no device, launch or memory error)."""


class DivergedError(Error):
    """mars::DivergedError -- a relaxation exhausted its sweep budget."""

    def __init__(self, msg, partial_state=None, sweeps=0):
        super().__init__(msg)
        self.partial_state = partial_state
        self.sweeps = sweeps


def _check(rc: int):
    if rc == N.MARS_OK:
        return
    msg = N.last_error()
    if rc == N.MARS_ERR_INPUT:
        raise InputError(msg)
    if rc == N.MARS_ERR_CUDA:
        raise CudaError(msg)
    raise Error(msg)


# ------------------------------------------------------- parameters (solvers.hpp:18-35)

class StartMode(enum.IntEnum):
    GridSweep = 0
    UniformRandom = 1


class RunStatus(enum.IntEnum):
    Ok = 0
    Skipped = 1
    Diverged = 2


K_MARS_SWEEP_CAP = 1_000_000  # solvers.hpp:116


@dataclass
class MarsParams:
    """solvers.hpp:20-27 (defaults identical).  ``sweep_cap`` overrides kMarsSweepCap."""
    t_min: float = 0.0
    t_max: float = 30.0
    t_step: float = 1.0
    c_step: float = 1.0
    d_min: float = 1e-4
    start_mode: StartMode = StartMode.GridSweep
    sweep_cap: int = 0

    def _c(self) -> N.mars_params_t:
        return N.mars_params_t(float(self.t_min), float(self.t_max), float(self.t_step),
                               float(self.c_step), float(self.d_min), int(self.start_mode), 0,
                               int(self.sweep_cap))


# ------------------------------------- synchronous baselines (solvers.hpp:62-91)

def linear_schedule(start: float, stop: float, points: int) -> list:
    """linear_schedule (solvers.cpp:105-116): evenly spaced, both ends included."""
    if points < 1:
        raise InputError("schedule needs at least one point")
    if points == 1:
        return [float(start)]
    return [start + (stop - start) * k / (points - 1) for k in range(points)]


def schedule_at(schedule, k: int, iters: int) -> float:
    """schedule_at (solvers.cpp:118-123): the sequence stretched / compressed by index."""
    n = len(schedule)
    if n == iters:
        return float(schedule[k])
    return float(schedule[min(n - 1, k * n // iters)])


@dataclass
class NmfaParams:
    """solvers.hpp:62-67 -- noisy mean-field annealing (run on the GPU Jacobi kernel)."""
    noise_sigma: float = 0.15
    alpha: float = 0.15
    schedule: list = field(default_factory=list)
    iters: int = 1000

    def _c(self):
        self._sched = np.ascontiguousarray(self.schedule, np.float64)
        return N.mars_nmfa_params_t(float(self.noise_sigma), float(self.alpha), int(self.iters),
                                    ptr(self._sched) if len(self._sched) else None, len(self._sched))


@dataclass
class SimCimParams:
    """solvers.hpp:74-79 -- simulated coherent Ising machine (run on the GPU Jacobi kernel)."""
    step_size: float = 0.1
    noise_sigma: float = 0.03
    pump_schedule: list = field(default_factory=list)
    iters: int = 1000

    def _c(self):
        self._sched = np.ascontiguousarray(self.pump_schedule, np.float64)
        return N.mars_simcim_params_t(float(self.step_size), float(self.noise_sigma), int(self.iters),
                                      ptr(self._sched) if len(self._sched) else None, len(self._sched))


def nmfa_defaults(iters: int = 1000) -> NmfaParams:
    """nmfa_defaults (solvers.cpp:125-132)."""
    return NmfaParams(0.15, 0.15, linear_schedule(2.0, 0.02, 64), iters)


def simcim_defaults(iters: int = 1000) -> SimCimParams:
    """simcim_defaults (solvers.cpp:134-141)."""
    return SimCimParams(0.1, 0.03, linear_schedule(-2.0, 1.0, 64), iters)


def _validate_sync(params) -> None:
    """validate(NmfaParams) / validate(SimCimParams) (solvers.cpp:89-103), same messages."""
    if isinstance(params, NmfaParams):
        if not (0.0 < params.alpha <= 1.0):
            raise InputError("nmfa: alpha must lie in (0,1]")
        if not (params.noise_sigma >= 0.0):
            raise InputError("nmfa: noise_sigma must be >= 0")
        if params.iters < 1:
            raise InputError("nmfa: iters must be >= 1")
        if len(params.schedule) == 0:
            raise InputError("nmfa: temperature schedule must not be empty")
        if any(not (t >= 0.0) for t in params.schedule):
            raise InputError("nmfa: schedule temperatures must be >= 0")
    else:
        if not (params.step_size > 0.0):
            raise InputError("simcim: step_size must be positive")
        if not (params.noise_sigma >= 0.0):
            raise InputError("simcim: noise_sigma must be >= 0")
        if params.iters < 1:
            raise InputError("simcim: iters must be >= 1")
        if len(params.pump_schedule) == 0:
            raise InputError("simcim: pump schedule must not be empty")


def validate(params) -> None:
    """validate(MarsParams) -- solvers.cpp:35-41 (or the NMFA / SimCIM validators); raises
    InputError."""
    if isinstance(params, (NmfaParams, SimCimParams)):
        _validate_sync(params)
        return
    _check(lib.mars_validate_params(C.byref(params._c())))


def mars_grid_count(p: MarsParams) -> int:
    """solvers.cpp:43-48."""
    import math
    slots = math.floor((p.t_max - p.t_min) / p.t_step)
    if not (slots >= 0.0) or slots > 1e9:
        raise InputError(f"mars: grid of {slots} temperatures is not usable")
    return int(slots) + 1


def mars_grid_temp(p: MarsParams, k: int) -> float:
    """solvers.cpp:50-52."""
    return p.t_min + float(k) * p.t_step


def mars_run_count(params: MarsParams, requested_runs: int) -> int:
    """solvers.cpp:202-213."""
    out = np.zeros(1, np.int64)
    _check(lib.mars_run_count(C.byref(params._c()), int(requested_runs), ptr(out)))
    return int(out[0])


@dataclass
class MarsRunPlan:
    """solvers.hpp:133-137."""
    skipped: bool
    start_temp: float
    seed: int


def mars_run_plan(params: MarsParams, base_seed: int, index: int) -> MarsRunPlan:
    """solvers.cpp:215-227."""
    sk = np.zeros(1, np.int32)
    t = np.zeros(1, np.float64)
    s = np.zeros(1, np.uint64)
    _check(lib.mars_run_plan(C.byref(params._c()), int(base_seed), int(index), ptr(sk), ptr(t), ptr(s)))
    return MarsRunPlan(bool(sk[0]), float(t[0]), int(s[0]))


def initial_state(seed: int, n: int) -> np.ndarray:
    """The descent's initial state (solvers.cpp:184-187), fp64 as drawn."""
    s = np.zeros(n, np.float64)
    _check(lib.mars_initial_state(int(seed), int(n), ptr(s)))
    return s


def splitmix64(x: int) -> int:
    return int(lib.mars_splitmix64(int(x)))


def sub_seed(base_seed: int, run_index: int) -> int:
    return int(lib.mars_sub_seed(int(base_seed), int(run_index)))


# ------------------------------------------------------------ problem (model.hpp:29-101)

_KERNELS = {"auto": N.MARS_KERNEL_AUTO, "dense_simt": N.MARS_KERNEL_DENSE_SIMT,
            "csr": N.MARS_KERNEL_CSR, "dense_umma": N.MARS_KERNEL_DENSE_UMMA}
_KERNEL_NAMES = {v: k for k, v in _KERNELS.items()}


class IsingProblem:
    """Immutable Ising instance resident on one GPU (model.hpp:29-101).

    Storage follows the reference: dense row-major for dense instances, CSR below
    kSparseDensityThreshold = 5% edge density (model.hpp:31, model.cpp:91).
    """
    kSparseDensityThreshold = 0.05

    def __init__(self, handle, n: int):
        self._h = C.c_void_p(handle)
        info = N.mars_problem_info_t()
        _check(lib.mars_problem_info(self._h, C.byref(info)))
        self._n = n
        self._info = info

    def __del__(self):
        h = getattr(self, "_h", None)
        if h is not None and h.value:
            lib.mars_problem_destroy(h)
            self._h = None

    @staticmethod
    def dense(n: int, couplings, field=None, device: int = 0, kernel: str = "auto") -> "IsingProblem":
        """IsingProblem::dense (model.cpp:47-72)."""
        J = np.ascontiguousarray(np.asarray(couplings, np.float64).reshape(-1))
        if n <= 0:
            raise InputError("problem size must be positive")
        if J.size != n * n:
            raise InputError("coupling matrix must be n*n")
        h = None
        if field is not None and len(field):
            h = np.ascontiguousarray(field, np.float64)
            if h.size != n:
                raise InputError("field length must equal n")
        out = C.c_void_p()
        _check(lib.mars_problem_dense(n, ptr(J), ptr(h), device, _KERNELS[kernel], C.byref(out)))
        return IsingProblem(out.value, n)

    @staticmethod
    def from_edges(n: int, edges, field=None, device: int = 0, kernel: str = "auto") -> "IsingProblem":
        """IsingProblem::from_edges (model.cpp:74-131); ``edges`` = [(u, v, w), ...] or (u, v, w) arrays."""
        if isinstance(edges, tuple) and len(edges) == 3 and hasattr(edges[0], "__len__"):
            u, v, w = edges
        else:
            e = list(edges)
            u = [x[0] for x in e]
            v = [x[1] for x in e]
            w = [x[2] for x in e]
        u = np.ascontiguousarray(u, np.int32)
        v = np.ascontiguousarray(v, np.int32)
        w = np.ascontiguousarray(w, np.float64)
        if n <= 0:
            raise InputError("problem size must be positive")
        h = None
        if field is not None and len(field):
            h = np.ascontiguousarray(field, np.float64)
            if h.size != n:
                raise InputError("field length must equal n")
        out = C.c_void_p()
        _check(lib.mars_problem_from_edges(n, len(u), ptr(u), ptr(v), ptr(w), ptr(h), device,
                                           _KERNELS[kernel], C.byref(out)))
        return IsingProblem(out.value, n)

    def replicate(self, device: int) -> "IsingProblem":
        """The same problem stored on another device (mars_problem_replicate): the replicas
        run_batch_multi shards a batch over."""
        out = C.c_void_p()
        _check(lib.mars_problem_replicate(self._h, int(device), C.byref(out)))
        return IsingProblem(out.value, self.size())

    def size(self) -> int:
        return self._n

    def uses_adjacency(self) -> bool:
        return bool(self._info.uses_adjacency)

    def integral(self) -> bool:
        return bool(self._info.integral)

    def has_field(self) -> bool:
        return bool(self._info.has_field)

    def coupling_sum(self) -> float:
        return float(self._info.coupling_sum)

    def nonzeros(self) -> int:
        return int(self._info.nonzeros)

    def device(self) -> int:
        return int(self._info.device)

    def kernel(self) -> str:
        return _KERNEL_NAMES[int(self._info.kernel)]

    def levels(self) -> int:
        """Gauss-Seidel levels of one sweep in the sparse layouts (0 for dense kernels)."""
        return int(self._info.levels)

    def energy_equality_tolerance(self) -> float:
        """model.hpp:82."""
        return 0.0 if self.integral() else 1e-9


def _spins(p: IsingProblem, spins) -> np.ndarray:
    s = np.ascontiguousarray(spins, np.int8)
    if s.size != p.size():
        raise InputError(f"spin configuration length {s.size} does not match problem size {p.size()}")
    return s


def energy(p: IsingProblem, spins) -> float:
    """energy (model.cpp:220-225), evaluated on the device in the reference's exact order."""
    e = np.zeros(1)
    _check(lib.mars_energy(p._h, ptr(_spins(p, spins)), ptr(e), None))
    return float(e[0])


def cut_value(p: IsingProblem, spins) -> float:
    """cut_value (model.cpp:227-229)."""
    c = np.zeros(1)
    _check(lib.mars_energy(p._h, ptr(_spins(p, spins)), None, ptr(c)))
    return float(c[0])


@dataclass
class GroundState:
    """model.hpp:131-134."""
    energy: float
    spins: np.ndarray


def brute_force_ground_state(p: IsingProblem, max_n: int = 26) -> GroundState:
    """brute_force_ground_state (model.cpp:296-324) on the device: exhaustive Gray-code scan,
    ties toward the lexicographically smallest spins; exact for integer couplings."""
    spins = np.zeros(p.size(), np.int8)
    e = np.zeros(1)
    _check(lib.mars_brute_force(p._h, int(max_n), ptr(e), ptr(spins)))
    return GroundState(float(e[0]), spins)


def round_spins(state) -> np.ndarray:
    """model.cpp:245-249 (host helper for tests/callers; the kernels round on device)."""
    s = np.asarray(state, np.float64)
    return np.where(s < 0.0, -1, 1).astype(np.int8)


# ------------------------------------------------------------ results (solvers.hpp:95-106)

@dataclass
class RunResult:
    status: RunStatus = RunStatus.Ok
    energy: float = 0.0
    cut: float = 0.0
    spins: Optional[np.ndarray] = None
    start_temp: float = 0.0
    descent_iters: int = 0
    elapsed_seconds: float = 0.0
    error: str = ""


@dataclass
class Records:
    """Struct-of-arrays form of ``std::vector<RunResult>`` (one entry per run index)."""
    status: np.ndarray
    energy: np.ndarray
    cut: np.ndarray
    start_temp: np.ndarray
    descent_iters: np.ndarray
    elapsed_seconds: np.ndarray
    spins: Optional[np.ndarray] = None   # [runs, n] int8 when requested
    fail_temp: Optional[np.ndarray] = None  # level temperature of Diverged runs (their message)

    @staticmethod
    def empty(count: int, n: int, with_spins: bool) -> "Records":
        return Records(np.zeros(count, np.uint8), np.zeros(count), np.zeros(count),
                       np.zeros(count), np.zeros(count, np.int64), np.zeros(count),
                       np.zeros((count, n), np.int8) if with_spins else None, np.zeros(count))

    def c(self) -> N.mars_records_t:
        return N.mars_records_t(ptr(self.status), ptr(self.energy), ptr(self.cut),
                                ptr(self.start_temp), ptr(self.descent_iters),
                                ptr(self.elapsed_seconds), ptr(self.spins), ptr(self.fail_temp))

    def error(self, k: int) -> str:
        """RunResult::error of a Diverged run: DivergedError's message (solvers.cpp:169,
        std::to_string(t) == printf("%f", t))."""
        if self.status[k] != RunStatus.Diverged:
            return ""
        t = float(self.fail_temp[k]) if self.fail_temp is not None else 0.0
        return "relaxation exceeded the sweep cap at T = " + ("%f" % t)

    def result(self, k: int) -> RunResult:
        st = RunStatus(int(self.status[k]))
        return RunResult(st, float(self.energy[k]), float(self.cut[k]),
                         None if self.spins is None or st == RunStatus.Skipped else self.spins[k].copy(),
                         float(self.start_temp[k]), int(self.descent_iters[k]),
                         float(self.elapsed_seconds[k]), self.error(k))


@dataclass
class BatchSpec:
    """runner.hpp:19-24.  ``workers`` is accepted for interface parity; the device decides."""
    params: MarsParams = field(default_factory=MarsParams)
    runs: int = 1
    base_seed: int = 0
    workers: int = 0
    keep_spins: bool = False   # also return every run's spins (R x N bytes)


@dataclass
class BatchStats:
    """runner.hpp:29-44."""
    best_energy: float = 0.0
    mean_energy: float = 0.0
    best_cut: float = 0.0
    mean_cut: float = 0.0
    hit_count: int = 0
    success_probability: float = 0.0
    total_seconds: float = 0.0
    mean_seconds_per_run: float = 0.0
    best_result: RunResult = field(default_factory=RunResult)
    energies: np.ndarray = field(default_factory=lambda: np.zeros(0))
    completed_runs: int = 0
    skipped_runs: int = 0
    failed_runs: int = 0
    records: Optional[Records] = None
    best_index: int = -1

    @property
    def runs(self) -> list:
        """Every slot as RunResult, including skipped/failed (materialised on demand)."""
        if self.records is None:
            return []
        return [self.records.result(k) for k in range(len(self.records.status))]


ProgressFn = Callable[[int, float], None]


def aggregate(records: Records, tolerance: float, total_seconds: float) -> BatchStats:
    """runner.cpp:126-167 via the native ``mars_aggregate``; raises Error when no run completed."""
    st = N.mars_stats_t()
    rc = lib.mars_aggregate(len(records.status), ptr(records.status), ptr(records.energy),
                            ptr(records.cut), ptr(records.elapsed_seconds), float(tolerance),
                            float(total_seconds), C.byref(st))
    _check(rc)
    stats = BatchStats(st.best_energy, st.mean_energy, st.best_cut, st.mean_cut, st.hit_count,
                       st.success_probability, st.total_seconds, st.mean_seconds_per_run)
    stats.completed_runs, stats.skipped_runs, stats.failed_runs = (
        st.completed_runs, st.skipped_runs, st.failed_runs)
    stats.best_index = int(st.best_index)
    ok = records.status == RunStatus.Ok
    stats.energies = records.energy[ok].copy()
    stats.records = records
    stats.best_result = records.result(stats.best_index)
    return stats


# ------------------------------------------------------------------ the batch seam

def _dist():
    try:
        import torch.distributed as dist
    except Exception:  # pragma: no cover - torch is part of the image
        return None
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        return dist
    return None


def shard_range(runs: int, rank: int, world: int) -> tuple:
    """Contiguous shard of run indices for one rank."""
    base, extra = divmod(runs, world)
    first = rank * base + min(rank, extra)
    return first, base + (1 if rank < extra else 0)


def run_shard(problem: IsingProblem, spec: BatchSpec, first: int, count: int) -> Records:
    """Run indices [first, first+count) of the batch on the problem's GPU."""
    rec = Records.empty(count, problem.size(), spec.keep_spins)
    c = rec.c()
    _check(lib.mars_run_shard(problem._h, C.byref(spec.params._c()), int(spec.runs),
                              int(spec.base_seed), int(first), int(count), C.byref(c)))
    return rec


def gather_records(dist, local: Records, runs: int, n: int, keep_spins: bool) -> Records:
    """all_gather of every rank's shard records, reassembled in run-index order."""
    import torch
    world = dist.get_world_size()
    backend = dist.get_backend()
    dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    out = Records.empty(runs, n, keep_spins)
    fields = ["status", "energy", "cut", "start_temp", "descent_iters", "elapsed_seconds", "fail_temp"]
    cap = max(shard_range(runs, r, world)[1] for r in range(world))
    for name in fields:
        arr = getattr(local, name)
        buf = np.zeros(cap, arr.dtype)
        buf[:len(arr)] = arr
        t = torch.from_numpy(buf.view(np.uint8).copy()).to(dev)
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        dst = getattr(out, name)
        for r in range(world):
            f, c = shard_range(runs, r, world)
            dst[f:f + c] = parts[r].cpu().numpy().view(arr.dtype)[:c]
    if keep_spins:
        buf = np.zeros((cap, n), np.int8)
        buf[:len(local.spins)] = local.spins
        t = torch.from_numpy(buf).to(dev)
        parts = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(parts, t)
        for r in range(world):
            f, c = shard_range(runs, r, world)
            out.spins[f:f + c] = parts[r].cpu().numpy()[:c]
    return out


def broadcast_best_spins(dist, local: Records, first: int, best_index: int, n: int,
                         owner: int) -> np.ndarray:
    """NCCL/gloo broadcast of the winning run's spins from the rank that owns it."""
    import torch
    dev = (torch.device("cuda", torch.cuda.current_device()) if dist.get_backend() == "nccl"
           else torch.device("cpu"))
    if dist.get_rank() == owner:
        t = torch.from_numpy(np.ascontiguousarray(local.spins[best_index - first])).to(dev)
    else:
        t = torch.zeros(n, dtype=torch.int8, device=dev)
    dist.broadcast(t, src=owner)
    return t.cpu().numpy()


def distributed_batch(dist, runs: int, n: int, tolerance: float, local_fn, keep_spins: bool):
    """Shard -> run -> gather -> aggregate -> broadcast best spins.

    ``local_fn(first, count) -> Records`` runs this rank's shard (records WITH spins).
    Every rank returns identical BatchStats (index-order aggregation after the gather).
    """
    t0 = time.perf_counter()
    rank, world = dist.get_rank(), dist.get_world_size()
    first, count = shard_range(runs, rank, world)
    local = local_fn(first, count)
    full = gather_records(dist, local, runs, n, keep_spins)
    stats = aggregate(full, tolerance, time.perf_counter() - t0)
    owner = next(r for r in range(world)
                 if shard_range(runs, r, world)[0] <= stats.best_index
                 < sum(shard_range(runs, r, world)))
    best = broadcast_best_spins(dist, local, first, stats.best_index, n, owner)
    stats.best_result.spins = best
    if not keep_spins:
        full.spins = None
    stats.total_seconds = time.perf_counter() - t0
    return stats


def run_batch(problem: IsingProblem, spec: BatchSpec, progress: Optional[ProgressFn] = None) -> BatchStats:
    """run_batch (runner.hpp:55-56, runner.cpp:170-178).

    Validates first (InputError before any run), runs every index on the GPU(s), and
    aggregates in run-index order exactly like the reference.  ``progress(index, best_so_far)``
    is invoked once per run while the batch runs, in completion order with a non-increasing
    best (runner.cpp:107-113; mars_run_batch_progress); under torch.distributed it is replayed
    in index order after the gather.
    """
    validate(spec.params)
    if isinstance(spec.params, (NmfaParams, SimCimParams)):
        stats = _run_sync_batch(problem, spec)
        if progress is not None:
            _replay_progress(stats, progress)
        return stats
    runs = mars_run_count(spec.params, spec.runs)
    n = problem.size()
    dist = _dist()
    if dist is not None:
        def local(first, count):
            return run_shard(problem, BatchSpec(spec.params, spec.runs, spec.base_seed,
                                                spec.workers, True), first, count)
        stats = distributed_batch(dist, runs, n, problem.energy_equality_tolerance(), local,
                                  spec.keep_spins)
    else:
        rec = Records.empty(runs, n, spec.keep_spins)
        c = rec.c()
        st = N.mars_stats_t()
        best = np.zeros(n, np.int8)
        if progress is None:
            _check(lib.mars_run_batch(problem._h, C.byref(spec.params._c()), int(spec.runs),
                                      int(spec.base_seed), C.byref(c), C.byref(st), ptr(best)))
        else:
            # called from this thread while the batch runs (mars_run_batch_progress)
            cb = N.PROGRESS_FN(lambda idx, best_so_far, _user: progress(int(idx), float(best_so_far)))
            _check(lib.mars_run_batch_progress(problem._h, C.byref(spec.params._c()), int(spec.runs),
                                               int(spec.base_seed), C.byref(c), C.byref(st), ptr(best), cb, None))
        stats = aggregate(rec, problem.energy_equality_tolerance(), st.total_seconds)
        stats.best_result.spins = best
        return stats
    if progress is not None:
        _replay_progress(stats, progress)
    return stats


def run_batch_multi(problems: list, spec: BatchSpec) -> BatchStats:
    """run_batch over several GPUs in ONE native call (mars_run_batch_multi): ``problems`` are
    replicas of one problem on distinct devices (IsingProblem.replicate); contiguous shards of
    the run indices run concurrently, one host thread per device, and the records / best spins
    are exchanged over NCCL (AllReduce-min of the best energy and index, Broadcast of the
    winning spins, AllGather of the records).  Identical results to run_batch on one device."""
    validate(spec.params)
    runs = mars_run_count(spec.params, spec.runs)
    n = problems[0].size()
    rec = Records.empty(runs, n, spec.keep_spins)
    c = rec.c()
    st = N.mars_stats_t()
    best = np.zeros(n, np.int8)
    handles = (C.c_void_p * len(problems))(*[p._h.value for p in problems])
    _check(lib.mars_run_batch_multi(handles, len(problems), C.byref(spec.params._c()), int(spec.runs),
                                    int(spec.base_seed), C.byref(c), C.byref(st), ptr(best)))
    stats = aggregate(rec, problems[0].energy_equality_tolerance(), st.total_seconds)
    stats.best_result.spins = best
    return stats


def debug_exchange(ranks: int, records: Records, tolerance: float):
    """TEST-ONLY: mars_run_batch_multi's shard / exchange logic on host memory (host threads as
    ranks) over given full-batch records; returns (merged Records, BatchStats, best spins)."""
    total, n = records.spins.shape
    out = Records.empty(total, n, False)
    c = out.c()
    st = N.mars_stats_t()
    best = np.zeros(n, np.int8)
    it = np.ascontiguousarray(records.descent_iters, np.int64)
    _check(lib.mars_debug_exchange(int(ranks), total, n, ptr(records.status), ptr(records.energy),
                                   ptr(records.cut), ptr(it), ptr(records.elapsed_seconds),
                                   ptr(records.spins), float(tolerance), C.byref(c), C.byref(st), ptr(best)))
    return out, st, best


def debug_choose_split(start_temps, params: MarsParams, pairs: int, resident=(74, 33, 15), num_sms: int = 148,
                       np_: int = 16384, forced: int = 0):
    """TEST-ONLY: the tcgen05 kernel's large-N split-K choice on host data -> (split, tiles)."""
    t = np.ascontiguousarray(start_temps, np.float64)
    res = np.ascontiguousarray(resident, np.int32)
    sp, tl = C.c_int32(0), C.c_int32(0)
    _check(lib.mars_debug_choose_split(ptr(t), len(t), C.byref(params._c()), int(pairs), ptr(res), int(num_sms),
                                       int(np_), int(forced), C.byref(sp), C.byref(tl)))
    return sp.value, tl.value


def _replay_progress(stats: "BatchStats", progress: ProgressFn) -> None:
    best_so_far = float("inf")
    for k in range(len(stats.records.status)):
        if stats.records.status[k] == RunStatus.Ok:
            best_so_far = min(best_so_far, float(stats.records.energy[k]))
        progress(k, best_so_far)


def _run_sync_batch(problem: IsingProblem, spec: BatchSpec) -> "BatchStats":
    """run_batch for NmfaParams / SimCimParams on the GPU (mars_run_batch_nmfa/_simcim)."""
    if spec.runs < 1:
        raise InputError("batch needs runs >= 1")
    n = problem.size()
    rec = Records.empty(int(spec.runs), n, spec.keep_spins)
    c = rec.c()
    st = N.mars_stats_t()
    best = np.zeros(n, np.int8)
    prm = spec.params._c()
    fn = lib.mars_run_batch_nmfa if isinstance(spec.params, NmfaParams) else lib.mars_run_batch_simcim
    _check(fn(problem._h, C.byref(prm), int(spec.runs), int(spec.base_seed), C.byref(c), C.byref(st), ptr(best)))
    stats = aggregate(rec, problem.energy_equality_tolerance(), st.total_seconds)
    stats.best_result.spins = best
    return stats


def run_batch_with(problem_n: int, run: Callable[[int], RunResult], runs: int, workers: int = 0,
                   progress: Optional[ProgressFn] = None, tolerance: float = 0.0) -> BatchStats:
    """runner.hpp:60-62 -- drive the aggregation with an arbitrary per-index run function
    (synthetic runs for tests); exceptions become Diverged records (runner.cpp:100-105)."""
    if runs < 1:
        raise InputError("batch needs runs >= 1")
    t0 = time.perf_counter()
    rec = Records.empty(runs, problem_n, True)
    best_so_far = float("inf")
    for k in range(runs):
        try:
            r = run(k)
        except Exception as e:  # noqa: BLE001 - mirrors catch (const std::exception&)
            r = RunResult(status=RunStatus.Diverged, error=str(e))
        rec.status[k] = int(r.status)
        rec.energy[k] = r.energy
        rec.cut[k] = r.cut
        rec.start_temp[k] = r.start_temp
        rec.descent_iters[k] = r.descent_iters
        rec.elapsed_seconds[k] = r.elapsed_seconds
        if r.spins is not None:
            rec.spins[k] = r.spins
        if progress is not None:
            if r.status == RunStatus.Ok and r.energy < best_so_far:
                best_so_far = r.energy
            progress(k, best_so_far)
    return aggregate(rec, tolerance, time.perf_counter() - t0)


def mars_sweep(p: IsingProblem, params: MarsParams, seed: int, runs: int = 1) -> list:
    """solvers.hpp:129-130 -- the per-run results of a batch, in index order."""
    stats = run_batch(p, BatchSpec(params, runs, seed, keep_spins=True))
    return stats.runs


# ------------------------------------------------------------- instances

def gen_sk_gaussian(n: int, seed: int) -> np.ndarray:
    """generate_sk's couplings (io.cpp:151-163)."""
    J = np.zeros((n, n), np.float64)
    lib.mars_gen_sk_gaussian(n, seed, ptr(J))
    return J


def gen_sk_pm1(n: int, seed: int) -> np.ndarray:
    J = np.zeros((n, n), np.float64)
    lib.mars_gen_sk_pm1(n, seed, ptr(J))
    return J


def gen_er(n: int, prob: float, seed: int):
    m = lib.mars_gen_er(n, prob, seed, None, None, None)
    u, v, w = np.zeros(m, np.int32), np.zeros(m, np.int32), np.zeros(m)
    lib.mars_gen_er(n, prob, seed, ptr(u), ptr(v), ptr(w))
    return u, v, w


def gen_ea(L: int, dims: int, seed: int):
    m = lib.mars_gen_ea(L, dims, seed, None, None, None)
    u, v, w = np.zeros(m, np.int32), np.zeros(m, np.int32), np.zeros(m)
    lib.mars_gen_ea(L, dims, seed, ptr(u), ptr(v), ptr(w))
    return u, v, w


def generate_sk(n: int, seed: int, device: int = 0, kernel: str = "auto") -> IsingProblem:
    """generate_sk (io.cpp:151-163): Gaussian SK instance on the device."""
    if n < 2:
        raise InputError("SK instance needs n >= 2")
    return IsingProblem.dense(n, gen_sk_gaussian(n, seed), device=device, kernel=kernel)


# ------------------------------------------------------------- staged batch (bench/timing)

class DeviceBatch:
    """A batch whose buffers persist across executions (mars_batch_* C-ABI): plan + H2D
    (``upload``), device-only work (``execute`` -> timing dict), D2H (``fetch``)."""

    def __init__(self, problem: IsingProblem, spec: BatchSpec, first: int = 0, count: Optional[int] = None):
        self.problem = problem
        self.spec = spec
        total = mars_run_count(spec.params, spec.runs)
        self.first = first
        self.count = total - first if count is None else count
        h = C.c_void_p()
        _check(lib.mars_batch_create(problem._h, C.byref(spec.params._c()), int(spec.runs),
                                     int(spec.base_seed), int(first), int(self.count), C.byref(h)))
        self._b = h

    def __del__(self):
        b = getattr(self, "_b", None)
        if b is not None and b.value:
            lib.mars_batch_destroy(b)
            self._b = None

    def upload(self):
        _check(lib.mars_batch_upload(self._b))

    def execute(self) -> dict:
        t = N.mars_timing_t()
        _check(lib.mars_batch_execute(self._b, C.byref(t)))
        return {k: getattr(t, k) for k, _ in N.mars_timing_t._fields_}

    def fetch(self, with_spins: bool = False) -> tuple:
        rec = Records.empty(self.count, self.problem.size(), with_spins)
        c = rec.c()
        best = np.zeros(1, np.int64)
        spins = np.zeros(self.problem.size(), np.int8)
        _check(lib.mars_batch_fetch(self._b, C.byref(c), ptr(best), ptr(spins)))
        return rec, int(best[0]), spins

    def finish_seconds(self) -> np.ndarray:
        """Per run: seconds from the launch's first descent start to the run's retirement
        (device %globaltimer of the last ``execute``; 0 for skipped runs)."""
        out = np.zeros(self.count, np.float64)
        _check(lib.mars_batch_fetch_finish(self._b, ptr(out)))
        return out


def debug_sweep(problem: IsingProblem, states, temps, sweeps: int = 1) -> tuple:
    """TEST-ONLY: ``sweeps`` in-order Gauss-Seidel sweeps (mars_relax_sweep,
    solvers.cpp:150-161) at fixed temperatures through the handle's dense device kernel, from
    the given fp32 states ([count, n]).  Returns (final states [count, n] fp32, kernel name)."""
    st = np.ascontiguousarray(states, dtype=np.float32)
    if st.ndim == 1:
        st = st[None, :]
    tt = np.ascontiguousarray(np.broadcast_to(np.asarray(temps, np.float64), (st.shape[0],)))
    out = np.zeros_like(st)
    used = C.c_int32(0)
    _check(lib.mars_debug_sweeps(problem._h, st.shape[0], ptr(st), ptr(tt), int(sweeps), ptr(out),
                                 C.byref(used)))
    return out, {1: "dense_simt", 2: "csr", 3: "dense_umma", 4: "dense_small"}.get(used.value, "?")
