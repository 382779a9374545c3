"""ctypes front end for the TEST-ONLY CPU checkers in oracle/ (never the product path).

``Oracle("ref")`` loads oracle/_ref/libmars_ref.so -- the reference's own C++ sources
compiled by oracle/Makefile -- and ``Oracle("port")`` loads oracle/libmars_oracle.so, the
plain-C restatement.  Both expose the identical interface declared in
oracle/mars_oracle.h, so every parity test can run against either.

Only tests/, __graft_entry__.smoke() and bench.py's CPU-baseline legs import this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIBS = {
    "ref": os.path.join(HERE, "_ref", "libmars_ref.so"),
    "port": os.path.join(HERE, "libmars_oracle.so"),
}
PREFIX = {"ref": "ref_", "port": "orc_"}


class OracleParams(C.Structure):
    _fields_ = [("t_min", C.c_double), ("t_max", C.c_double), ("t_step", C.c_double),
                ("c_step", C.c_double), ("d_min", C.c_double), ("start_mode", C.c_int32),
                ("pad_", C.c_int32)]


class OracleRecords(C.Structure):
    _fields_ = [("status", C.c_void_p), ("energy", C.c_void_p), ("cut", C.c_void_p),
                ("start_temp", C.c_void_p), ("descent_iters", C.c_void_p),
                ("elapsed_seconds", C.c_void_p), ("spins", C.c_void_p)]


class OracleStats(C.Structure):
    _fields_ = [("best_energy", C.c_double), ("mean_energy", C.c_double),
                ("best_cut", C.c_double), ("mean_cut", C.c_double), ("hit_count", C.c_int64),
                ("success_probability", C.c_double), ("total_seconds", C.c_double),
                ("mean_seconds_per_run", C.c_double), ("best_index", C.c_int64),
                ("completed_runs", C.c_int64), ("skipped_runs", C.c_int64),
                ("failed_runs", C.c_int64)]


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


@dataclass
class OracleBatch:
    status: np.ndarray
    energy: np.ndarray
    cut: np.ndarray
    start_temp: np.ndarray
    descent_iters: np.ndarray
    elapsed_seconds: np.ndarray
    spins: np.ndarray | None
    stats: dict


class OracleError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code


def params(t_min=0.0, t_max=30.0, t_step=1.0, c_step=1.0, d_min=1e-4, uniform=False):
    return OracleParams(t_min, t_max, t_step, c_step, d_min, 1 if uniform else 0, 0)


class Oracle:
    """One of the two CPU checkers (``kind`` = "ref" or "port")."""

    def __init__(self, kind: str = "ref"):
        path = LIBS[kind]
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (run `make -C oracle`)")
        self.kind = kind
        self.lib = C.CDLL(path)
        p = PREFIX[kind]
        L = self.lib
        def f(name, res, *args):
            fn = getattr(L, p + name)
            fn.restype = res
            fn.argtypes = list(args)
            return fn
        vp, i32, i64, u64, dbl = C.c_void_p, C.c_int, C.c_int64, C.c_uint64, C.c_double
        self._splitmix = f("splitmix64", u64, u64)
        self._sub_seed = f("sub_seed", u64, u64, u64)
        self._draws = f("rng_draws", None, u64, i32, u64, i64, vp, vp)
        self._dense = f("problem_dense", vp, i32, vp, vp, C.c_char_p, i32)
        self._edges = f("problem_edges", vp, i32, i64, vp, vp, vp, vp, C.c_char_p, i32)
        self._free = f("problem_free", None, vp)
        self._info = f("problem_info", None, vp, vp, vp, vp, vp, vp)
        self._energy = f("energy", dbl, vp, vp)
        self._cut = f("cut_value", dbl, vp, vp)
        self._coupling = f("coupling_term", dbl, vp, vp)
        self._tanh = f("tanh_trial", dbl, dbl, dbl)
        self._sweep = f("relax_sweep", dbl, vp, vp, dbl)
        self._relax = f("relax_to_fixed_point", i32, vp, vp, dbl, dbl, vp, vp)
        self._validate = f("validate", i32, C.POINTER(OracleParams), C.c_char_p, i32)
        self._count = f("run_count", i32, C.POINTER(OracleParams), i64, vp, C.c_char_p, i32)
        self._plan = f("run_plan", None, C.POINTER(OracleParams), u64, i64, vp, vp, vp)
        self._init = f("initial_state", None, u64, i32, vp)
        self._descent = f("descent", i32, vp, dbl, C.POINTER(OracleParams), u64, vp, vp, vp, vp,
                          vp, C.c_char_p, i32)
        self._batch = f("run_batch", i32, vp, C.POINTER(OracleParams), i64, u64, i32,
                        C.POINTER(OracleRecords), C.POINTER(OracleStats), C.c_char_p, i32)
        self._gen_sk = f("gen_sk_gaussian", None, i32, u64, vp)
        self._gen_pm1 = f("gen_sk_pm1", None, i32, u64, vp)
        self._gen_er = f("gen_er", i64, i32, dbl, u64, vp, vp, vp)
        self._gen_ea = f("gen_ea", i64, i32, i32, u64, vp, vp, vp)
        if kind == "ref":
            for nm in ("ref_run_batch_nmfa", "ref_run_batch_simcim"):
                fn = getattr(L, nm)
                fn.restype = i32
                fn.argtypes = [vp, dbl, dbl, i64, vp, i64, i64, u64, i32, C.POINTER(OracleRecords),
                               C.POINTER(OracleStats), C.c_char_p, i32]
            self._nmfa = L.ref_run_batch_nmfa
            self._simcim = L.ref_run_batch_simcim
        if kind == "port":
            self._sweep32 = L.orc_relax_sweep_f32
            self._sweep32.restype = dbl
            self._sweep32.argtypes = [vp, vp, dbl]
            self._replay = L.orc_replay_batch_f32
            self._replay.restype = i32
            self._replay.argtypes = [vp, C.POINTER(OracleParams), i64, u64, i32, i32, vp, vp, vp]
            self._set_cap = L.orc_set_sweep_cap
            self._set_cap.restype = None
            self._set_cap.argtypes = [i64]

    def set_sweep_cap(self, cap: int):
        """Port-only test knob: override kMarsSweepCap (0 restores 10^6)."""
        self._set_cap(int(cap))

    # ---- rng.hpp
    def splitmix64(self, x: int) -> int:
        return self._splitmix(x)

    def sub_seed(self, base: int, idx: int) -> int:
        return self._sub_seed(base, idx)

    def draws(self, seed: int, kind: int, count: int, arg: int = 0) -> np.ndarray:
        if kind in (0, 5):
            out = np.zeros(count, np.uint64)
            self._draws(seed, kind, arg, count, _ptr(out), None)
        else:
            out = np.zeros(count, np.float64)
            self._draws(seed, kind, arg, count, None, _ptr(out))
        return out

    # ---- model.hpp
    def problem_dense(self, J: np.ndarray, h: np.ndarray | None = None) -> "OracleProblem":
        J = np.ascontiguousarray(J, np.float64)
        n = J.shape[0]
        h = None if h is None else np.ascontiguousarray(h, np.float64)
        err = C.create_string_buffer(256)
        p = self._dense(n, _ptr(J), _ptr(h), err, 256)
        if not p:
            raise OracleError(1, err.value.decode())
        return OracleProblem(self, p)

    def problem_edges(self, n, u, v, w, h=None) -> "OracleProblem":
        u = np.ascontiguousarray(u, np.int32)
        v = np.ascontiguousarray(v, np.int32)
        w = np.ascontiguousarray(w, np.float64)
        h = None if h is None else np.ascontiguousarray(h, np.float64)
        err = C.create_string_buffer(256)
        p = self._edges(n, len(u), _ptr(u), _ptr(v), _ptr(w), _ptr(h), err, 256)
        if not p:
            raise OracleError(1, err.value.decode())
        return OracleProblem(self, p)

    def tanh_trial(self, phi: float, t: float) -> float:
        return self._tanh(phi, t)

    # ---- solvers.hpp
    def validate(self, prm: OracleParams):
        err = C.create_string_buffer(256)
        if self._validate(C.byref(prm), err, 256):
            raise OracleError(1, err.value.decode())

    def run_count(self, prm: OracleParams, requested: int) -> int:
        out = np.zeros(1, np.int64)
        err = C.create_string_buffer(256)
        if self._count(C.byref(prm), requested, _ptr(out), err, 256):
            raise OracleError(1, err.value.decode())
        return int(out[0])

    def run_plan(self, prm: OracleParams, base_seed: int, index: int):
        sk = np.zeros(1, np.int32)
        t = np.zeros(1, np.float64)
        s = np.zeros(1, np.uint64)
        self._plan(C.byref(prm), base_seed, index, _ptr(sk), _ptr(t), _ptr(s))
        return bool(sk[0]), float(t[0]), int(s[0])

    def initial_state(self, seed: int, n: int) -> np.ndarray:
        s = np.zeros(n, np.float64)
        self._init(seed, n, _ptr(s))
        return s

    # ---- generators
    def gen_sk_gaussian(self, n: int, seed: int) -> np.ndarray:
        J = np.zeros((n, n), np.float64)
        self._gen_sk(n, seed, _ptr(J))
        return J

    def gen_sk_pm1(self, n: int, seed: int) -> np.ndarray:
        J = np.zeros((n, n), np.float64)
        self._gen_pm1(n, seed, _ptr(J))
        return J

    def gen_er(self, n: int, prob: float, seed: int):
        m = self._gen_er(n, prob, seed, None, None, None)
        u, v, w = np.zeros(m, np.int32), np.zeros(m, np.int32), np.zeros(m, np.float64)
        self._gen_er(n, prob, seed, _ptr(u), _ptr(v), _ptr(w))
        return u, v, w

    def gen_ea(self, L: int, dims: int, seed: int):
        m = self._gen_ea(L, dims, seed, None, None, None)
        u, v, w = np.zeros(m, np.int32), np.zeros(m, np.int32), np.zeros(m, np.float64)
        self._gen_ea(L, dims, seed, _ptr(u), _ptr(v), _ptr(w))
        return u, v, w


class OracleProblem:
    def __init__(self, orc: Oracle, handle):
        self.orc = orc
        self.h = handle
        n, adj, integ = np.zeros(1, np.int32), np.zeros(1, np.int32), np.zeros(1, np.int32)
        cs, nnz = np.zeros(1, np.float64), np.zeros(1, np.int64)
        orc._info(handle, _ptr(n), _ptr(adj), _ptr(integ), _ptr(cs), _ptr(nnz))
        self.n = int(n[0])
        self.uses_adjacency = bool(adj[0])
        self.integral = bool(integ[0])
        self.coupling_sum = float(cs[0])
        self.nonzeros = int(nnz[0])

    def __del__(self):
        try:
            self.orc._free(self.h)
        except Exception:
            pass

    def energy(self, spins: np.ndarray) -> float:
        s = np.ascontiguousarray(spins, np.int8)
        return self.orc._energy(self.h, _ptr(s))

    def cut_value(self, spins: np.ndarray) -> float:
        s = np.ascontiguousarray(spins, np.int8)
        return self.orc._cut(self.h, _ptr(s))

    def coupling_term(self, spins: np.ndarray) -> float:
        s = np.ascontiguousarray(spins, np.int8)
        return self.orc._coupling(self.h, _ptr(s))

    def relax_sweep(self, s: np.ndarray, t: float) -> float:
        assert s.dtype == np.float64 and s.flags.c_contiguous
        return self.orc._sweep(self.h, _ptr(s), t)

    def relax_to_fixed_point(self, s: np.ndarray, t: float, d_min: float, budget: int):
        b = np.array([budget], np.int64)
        sw = np.zeros(1, np.int64)
        rc = self.orc._relax(self.h, _ptr(s), t, d_min, _ptr(b), _ptr(sw))
        return rc, int(sw[0]), int(b[0])

    def descent(self, start_temp: float, prm: OracleParams, seed: int):
        st = np.zeros(1, np.uint8)
        e, c = np.zeros(1, np.float64), np.zeros(1, np.float64)
        it = np.zeros(1, np.int64)
        sp = np.zeros(self.n, np.int8)
        err = C.create_string_buffer(256)
        rc = self.orc._descent(self.h, start_temp, C.byref(prm), seed, _ptr(st), _ptr(e), _ptr(c),
                               _ptr(it), _ptr(sp), err, 256)
        if rc == 1:
            raise OracleError(1, err.value.decode())
        return dict(status=int(st[0]), energy=float(e[0]), cut=float(c[0]),
                    descent_iters=int(it[0]), spins=sp)

    def relax_sweep_f32(self, s: np.ndarray, t: float) -> float:
        """Port only (TEST-ONLY): one in-order sweep in fp32 (the fp32 floor), in place."""
        assert s.dtype == np.float32 and s.flags.c_contiguous
        return self.orc._sweep32(self.h, _ptr(s), t)

    def run_sync(self, solver: str, a: float, b: float, iters: int, schedule, runs: int, base_seed: int,
                 workers: int = 0) -> OracleBatch:
        """Reference only: run_batch with NmfaParams (a = noise_sigma, b = alpha) or SimCimParams
        (a = step_size, b = noise_sigma) -- the checker of the device's synchronous baselines."""
        sched = np.ascontiguousarray(schedule, np.float64)
        status = np.zeros(runs, np.uint8)
        energy, cut = np.zeros(runs), np.zeros(runs)
        t0, el = np.zeros(runs), np.zeros(runs)
        iters_out = np.zeros(runs, np.int64)
        sp = np.zeros((runs, self.n), np.int8)
        rec = OracleRecords(_ptr(status), _ptr(energy), _ptr(cut), _ptr(t0), _ptr(iters_out), _ptr(el), _ptr(sp))
        st = OracleStats()
        err = C.create_string_buffer(256)
        fn = self.orc._nmfa if solver == "nmfa" else self.orc._simcim
        rc = fn(self.h, a, b, iters, _ptr(sched), len(sched), runs, base_seed, workers, C.byref(rec),
                C.byref(st), err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        stats = {k: getattr(st, k) for k, _ in OracleStats._fields_}
        return OracleBatch(status, energy, cut, t0, iters_out, el, sp, stats)

    def replay_f32(self, prm: OracleParams, runs: int, base_seed: int, workers: int = 0, mode: int = 0):
        """Port only (TEST-ONLY measurement tool): the first `runs` descents replayed with fp32
        state/fields/tanh (mode 0) or additionally J rounded to one fp16 plane (mode 1).
        Returns (status, descent_iters, spins)."""
        status = np.zeros(runs, np.uint8)
        iters = np.zeros(runs, np.int64)
        sp = np.zeros((runs, self.n), np.int8)
        if self.orc._replay(self.h, C.byref(prm), runs, base_seed, workers, mode, _ptr(status), _ptr(iters), _ptr(sp)):
            raise OracleError(1, "replay_f32 needs a dense problem")
        return status, iters, sp

    def run_batch(self, prm: OracleParams, runs: int, base_seed: int, workers: int = 0,
                  spins: bool = True) -> OracleBatch:
        count = self.orc.run_count(prm, runs)
        status = np.zeros(count, np.uint8)
        energy, cut = np.zeros(count), np.zeros(count)
        t0, el = np.zeros(count), np.zeros(count)
        iters = np.zeros(count, np.int64)
        sp = np.zeros((count, self.n), np.int8) if spins else None
        rec = OracleRecords(_ptr(status), _ptr(energy), _ptr(cut), _ptr(t0), _ptr(iters),
                            _ptr(el), _ptr(sp))
        st = OracleStats()
        err = C.create_string_buffer(256)
        rc = self.orc._batch(self.h, C.byref(prm), runs, base_seed, workers, C.byref(rec),
                             C.byref(st), err, 256)
        if rc:
            raise OracleError(rc, err.value.decode())
        stats = {k: getattr(st, k) for k, _ in OracleStats._fields_}
        return OracleBatch(status, energy, cut, t0, iters, el, sp, stats)
